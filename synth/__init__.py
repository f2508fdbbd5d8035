"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no reduction, no offsets,
no partition): it only draws inputs.  It is the one module both `oracle/`
(through the tests) and the product path (through `bench.py` / the GPU tests)
may use, per the input recipe in DESIGN.md §3 (SURVEY.md §8(d) "Synthetic
inputs").

Host side (numpy) here; the device side is the same counter-based generator
re-implemented in `synth/csrc/synth.cu` (loaded by `synth.device`), checked
bit-for-bit against this file by `tests/test_synth.py`/`tests/test_gpu_*.py`.

Recipe:
  * segment lengths: numpy PCG64 `default_rng(seed)`;
      - "powerlaw": Lomax (Pareto II) alpha=2: u = 1 - rng.random(S),
        w = u**(-1/alpha) - 1, lengths = largest-remainder apportionment of E
        proportional to w (ties -> lower segment id), so sum(lengths) == E;
      - "uniform": E // S each, the first E % S segments get +1.
  * values: h = splitmix64(seed * 0x9E3779B97F4A7C15 + e * F + f) with the
    GLOBAL edge id e (so shards regenerate the same global input):
      - "real"   fp32: (h >> 40) * 2**-24               in [0, 1)
      - "signed" fp32: (h >> 40) * 2**-23 - 1           in [-1, 1), never -0.0
      - "real"   bf16: (h >> 56) * 2**-8                in [0, 1), exact in bf16
      - "signed" bf16: (h >> 56) * 2**-7 - 1            in [-1, 1), exact in bf16
      - "int"  (both): (h mod 17) - 8                   integers in [-8, 8]
  * fused source index: src_idx[e] = splitmix64(seed2 + e) mod V
    (uniform iid, worst-case locality).
  * edge weights (weighted fused form): "real" mode with seed3, as fp32.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15

MODES = ("real", "signed", "int")
DTYPES = ("f32", "bf16")
DISTS = ("powerlaw", "uniform")


# ----------------------------------------------------------------------------
# splitmix64 (Steele, Lea, Flood 2014) — vectorised over numpy uint64
# ----------------------------------------------------------------------------
def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def value_seed_base(seed: int) -> int:
    return (int(seed) * GOLDEN) & MASK64


def _values_from_h(h: np.ndarray, dtype: str, mode: str) -> np.ndarray:
    """Map 64-bit hashes to float32 values exactly representable in `dtype`."""
    if mode == "int":
        return ((h % np.uint64(17)).astype(np.int64) - 8).astype(np.float32)
    if dtype == "f32":
        k = (h >> np.uint64(40)).astype(np.float64)
        if mode == "real":
            return (k * 2.0 ** -24).astype(np.float32)
        return (k * 2.0 ** -23 - 1.0).astype(np.float32)
    if dtype == "bf16":
        k = (h >> np.uint64(56)).astype(np.float64)
        if mode == "real":
            return (k * 2.0 ** -8).astype(np.float32)
        return (k * 2.0 ** -7 - 1.0).astype(np.float32)
    raise ValueError(dtype)


def values_f32(seed: int, e_begin: int, n_rows: int, F: int, dtype: str = "f32",
               mode: str = "real", rows: np.ndarray | None = None) -> np.ndarray:
    """Values of rows [e_begin, e_begin+n_rows) (or the explicit global `rows`)
    as an (n, F) float32 array holding values exact in `dtype`."""
    if rows is None:
        rows = np.arange(e_begin, e_begin + n_rows, dtype=np.uint64)
    else:
        rows = np.asarray(rows, dtype=np.uint64)
    base = np.uint64(value_seed_base(seed))
    with np.errstate(over="ignore"):
        ctr = base + rows[:, None] * np.uint64(F) + np.arange(F, dtype=np.uint64)[None, :]
    return _values_from_h(splitmix64(ctr), dtype, mode)


def f32_to_bf16_bits(v: np.ndarray) -> np.ndarray:
    """Exact conversion for values already representable in bf16 (truncation)."""
    b = np.ascontiguousarray(v, dtype=np.float32).view(np.uint32)
    return (b >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def values(seed: int, e_begin: int, n_rows: int, F: int, dtype: str = "f32",
           mode: str = "real", rows: np.ndarray | None = None) -> np.ndarray:
    """Values in storage form: float32 array for f32, uint16 bit array for bf16."""
    v = values_f32(seed, e_begin, n_rows, F, dtype, mode, rows)
    return v if dtype == "f32" else f32_to_bf16_bits(v)


def src_index(seed2: int, e_begin: int, n: int, V: int) -> np.ndarray:
    """Fused-form source index: splitmix64(seed2 + e) mod V, int64."""
    e = np.arange(e_begin, e_begin + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(seed2 & MASK64) + e)
    return (h % np.uint64(V)).astype(np.int64)


def weights(seed3: int, e_begin: int, n: int) -> np.ndarray:
    """Edge weights for the weighted fused form: 'real' fp32 values, F=1."""
    return values_f32(seed3, e_begin, n, 1, "f32", "real")[:, 0].copy()


# ----------------------------------------------------------------------------
# segment lengths
# ----------------------------------------------------------------------------
def apportion(E: int, w: np.ndarray) -> np.ndarray:
    """Largest-remainder apportionment of E units proportional to w >= 0.
    Remainders go to the largest fractional parts; ties to the lower id."""
    w = np.asarray(w, dtype=np.float64)
    S = w.shape[0]
    if S == 0:
        return np.zeros(0, dtype=np.int64)
    tot = w.sum()
    if E == 0:
        return np.zeros(S, dtype=np.int64)
    if tot <= 0:
        w = np.ones(S)
        tot = float(S)
    q = w * (E / tot)
    L = np.floor(q).astype(np.int64)
    rem = E - int(L.sum())
    if rem > 0:
        frac = q - L
        order = np.lexsort((np.arange(S), -frac))  # largest frac first, then lower id
        L[order[:rem]] += 1
    elif rem < 0:  # float rounding pushed the floors over E: take back from the smallest fracs
        frac = q - L
        order = np.lexsort((np.arange(S), frac))
        take = order[L[order] > 0][:(-rem)]
        L[take] -= 1
    assert int(L.sum()) == E
    return L


def segment_lengths(E: int, S: int, dist: str = "powerlaw", seed: int = 0,
                    alpha: float = 2.0) -> np.ndarray:
    if S == 0:
        if E:
            raise ValueError("E > 0 edges need S > 0 segments")
        return np.zeros(0, dtype=np.int64)
    if dist == "uniform":
        L = np.full(S, E // S, dtype=np.int64)
        L[: E % S] += 1
        return L
    if dist == "powerlaw":
        rng = np.random.default_rng(seed)
        u = 1.0 - rng.random(S)
        w = u ** (-1.0 / alpha) - 1.0
        return apportion(E, w)
    raise ValueError(dist)


def lengths_to_index(L: np.ndarray, itype: str = "i32") -> np.ndarray:
    """Sorted destination index: segment s repeated L[s] times."""
    dt = np.int32 if itype == "i32" else np.int64
    return np.repeat(np.arange(L.shape[0], dtype=dt), L)


def lengths_to_bounds(L: np.ndarray) -> np.ndarray:
    """Cumulative row bounds (int64, S+1) used only to EXPAND the generated
    lengths into an index on the device (the generator's own bookkeeping)."""
    b = np.zeros(L.shape[0] + 1, dtype=np.int64)
    np.cumsum(L, out=b[1:])
    return b


# ----------------------------------------------------------------------------
# stress index families
# ----------------------------------------------------------------------------
def stress_lengths(kind: str, E: int, S: int, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    if kind == "single":           # one segment holds every edge
        L = np.zeros(S, dtype=np.int64)
        if S:
            L[rng.integers(S)] = E
        return L
    if kind == "singletons":       # all-singleton prefix, rest empty
        L = np.zeros(S, dtype=np.int64)
        L[: min(E, S)] = 1
        if E > S:
            L[-1] += E - S
        return L
    if kind == "alternating":      # runs of 1 and long runs, gaps between
        w = np.where(np.arange(S) % 3 == 0, 0.0, np.where(np.arange(S) % 3 == 1, 1.0, 37.0))
        return apportion(E, w)
    if kind == "gaps":             # many empty segments, incl. leading and trailing
        w = rng.random(S) * (rng.random(S) < 0.3)
        if S > 2:
            w[0] = 0.0
            w[-1] = 0.0
        return apportion(E, w)
    if kind == "powerlaw15":
        return segment_lengths(E, S, "powerlaw", seed, alpha=1.5)
    if kind in DISTS:
        return segment_lengths(E, S, kind, seed)
    raise ValueError(kind)


STRESS_KINDS = ("single", "singletons", "alternating", "gaps", "powerlaw15", "powerlaw", "uniform")


# ----------------------------------------------------------------------------
# named workloads (BASELINE.json configs; SURVEY.md §8(d) table "Configs")
# ----------------------------------------------------------------------------
WORKLOADS = {
    # id: (E, S, F, dtype, dist, seed)
    "cora": dict(E=10_556, S=2_708, F=32, dtype="f32", dist="powerlaw", seed=1),
    "arxiv": dict(E=1_166_243, S=169_343, F=128, dtype="f32", dist="powerlaw", seed=2),
    "reddit": dict(E=114_615_892, S=232_965, F=64, dtype="f32", dist="powerlaw", seed=3, V=232_965),
    "products": dict(E=61_859_140, S=2_449_029, F=128, dtype="bf16", dist="powerlaw", seed=4),
    "sweep": dict(E=1 << 24, S=1 << 20, F=64, dtype="f32", dist="powerlaw", seed=5),
}


def workload(name: str, **over) -> dict:
    w = dict(WORKLOADS[name])
    w.update(over)
    w.setdefault("seed2", w["seed"] + 1000)
    w.setdefault("seed3", w["seed"] + 2000)
    w["name"] = name
    return w


# ----------------------------------------------------------------------------
# worked examples W1 / W2 (instance of the paper's Fig. 1(a)
# shape "4 nodes and 5 edges", PAPER.md:27-33 — the figure's values are absent)
# ----------------------------------------------------------------------------
W_X = np.array([[1, 2], [3, 4], [5, 6], [7, 8]], dtype=np.float32)
W1 = dict(dst=np.array([0, 0, 1, 2, 3]), src=np.array([1, 3, 0, 1, 2]), x=W_X, S=4)
W2 = dict(dst=np.array([0, 0, 1, 1, 3]), src=np.array([1, 2, 0, 3, 2]), x=W_X, S=4)

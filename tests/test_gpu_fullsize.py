"""Parity at BASELINE.json's full sizes (products-, Reddit-shaped and the
width/skew sweep), in the default (selector) launch configuration: inputs are
generated on the device, and a sample of output segments is re-derived on the
host (host generator, keyed by global edge id) and checked against the oracle
one by one.  Sample = random segments + the longest ones + every segment that
contains an agent/tile boundary of the kernels' edge splits (the carry paths)."""
import numpy as np
import pytest

import oracle
import synth
from parity_helpers import check, from_torch_vals

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def geot():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_03019_b200 as g
    return g


def sample_segments(L, E, rng, n_random=4000, n_long=50):
    S = L.shape[0]
    bounds = synth.lengths_to_bounds(L)
    picks = set(rng.choice(S, size=min(n_random, S), replace=False).tolist())
    picks |= set(np.argsort(L)[-n_long:].tolist())
    nsm = torch.cuda.get_device_properties(0).multi_processor_count if torch.cuda.is_available() else 148
    # agent splits of the narrow kernel: NA = SMs x CTAs/SM x warps (8, or 12 for fp32 F=1),
    # boundaries ((k*E)/NA) rounded down to ITEMS rows (narrow.cuh agent_lo)
    for NA in sorted({nsm * c * w for c in (1, 2) for w in (8, 12)} | {nsm * 32, nsm * 64}):
        k = np.arange(1, NA, dtype=np.int64)
        for items in (1, 8, 16, 32):
            e = (k * E) // NA // items * items
            picks.update((np.searchsorted(bounds, e, side="right") - 1).tolist())
    for NA in (2368, 4736, 9472, 18944):  # stream kernel: L = ceil(E/NA) rounded up to RS rows per agent
        for RS in (4, 6, 12):
            Lr = (-(-E // NA) + RS - 1) // RS * RS
            e = np.arange(Lr, E, Lr)
            picks.update((np.searchsorted(bounds, e, side="right") - 1).tolist())
    for tile in (256, 1024, 4096):  # edge-tile kernel tiles (a subset)
        for e in range(tile, E, max(tile, E // 3000)):
            picks.add(int(np.searchsorted(bounds, e, side="right") - 1))
    segs = np.array(sorted(s for s in picks if 0 <= s < S), dtype=np.int64)
    return segs, bounds


def sub_problem(segs, bounds):
    """Global edge ids of the sampled segments and their local (renumbered) index."""
    lens = bounds[segs + 1] - bounds[segs]
    rows = np.concatenate([np.arange(bounds[s], bounds[s + 1]) for s in segs]) if len(segs) else np.zeros(0, np.int64)
    loc = np.repeat(np.arange(len(segs)), lens)
    return rows, loc, lens


def run_full(geot, name, F=None, op="sum", mode="real", itype=torch.int32):
    import synth.device as sd
    w = synth.workload(name, **({"F": F} if F else {}))
    E, S, F = w["E"], w["S"], w["F"]
    tdt = torch.float32 if w["dtype"] == "f32" else torch.bfloat16
    L = synth.segment_lengths(E, S, w["dist"], w["seed"])
    idx = sd.index_from_lengths(L, itype)
    if "V" in w:  # fused gather form
        V = w["V"]
        x = sd.values(V, F, w["seed"], dtype=tdt, mode=mode)
        src = sd.src_index(E, V, w["seed2"], itype=itype)
        y = geot.geot_gather_segment_reduce(x, src, idx, S, op)
        del src
    else:
        X = sd.values(E, F, w["seed"], dtype=tdt, mode=mode)
        y = geot.geot_segment_reduce(X, idx, S, op)
        del X
    torch.cuda.synchronize()
    return w, L, y


@pytest.mark.parametrize("op", ["sum", "max"])
def test_products_shaped_bf16(geot, op):
    w, L, y = run_full(geot, "products", op=op, mode="real" if op == "sum" else "signed")
    rng = np.random.default_rng(1)
    segs, bounds = sample_segments(L, w["E"], rng)
    rows, loc, lens = sub_problem(segs, bounds)
    X = synth.values(w["seed"], 0, 0, w["F"], "bf16", "real" if op == "sum" else "signed", rows=rows)
    ref = oracle.segment_reduce(X, loc, len(segs), op, nthreads=oracle.default_threads())
    got = from_torch_vals(y[torch.from_numpy(segs).cuda()])
    check(got, ref, op, "bf16", "real", counts=lens, what=f"products {op}")


def test_reddit_shaped_fused(geot):
    w, L, y = run_full(geot, "reddit")
    rng = np.random.default_rng(2)
    segs, bounds = sample_segments(L, w["E"], rng, n_random=2000)
    rows, loc, lens = sub_problem(segs, bounds)
    # src_idx of the sampled edges, regenerated on the host (counter-based)
    src = np.empty(rows.shape[0], dtype=np.int64)
    with np.errstate(over="ignore"):
        h = synth.splitmix64(np.uint64(w["seed2"]) + rows.astype(np.uint64))
    src[:] = (h % np.uint64(w["V"])).astype(np.int64)
    x = synth.values_f32(w["seed"], 0, w["V"], w["F"], "f32", "real")
    ref = oracle.gather_segment_reduce(x, src, loc, len(segs), "sum", nthreads=oracle.default_threads())
    got = y[torch.from_numpy(segs).cuda()].cpu().numpy()
    check(got, ref, "sum", "f32", "real", counts=lens, what="reddit fused")


@pytest.mark.parametrize("F", [1, 4, 16, 64, 256, 1024])
@pytest.mark.parametrize("mode", ["real", "int"])
def test_sweep_widths_full(geot, F, mode):
    w, L, y = run_full(geot, "sweep", F=F, op="sum", mode=mode)
    rng = np.random.default_rng(F)
    n_random = 4000 if F <= 256 else 800
    segs, bounds = sample_segments(L, w["E"], rng, n_random=n_random, n_long=10 if F == 1024 else 50)
    rows, loc, lens = sub_problem(segs, bounds)
    X = synth.values(w["seed"], 0, 0, F, "f32", mode, rows=rows)
    ref = oracle.segment_reduce(X, loc, len(segs), "sum", nthreads=oracle.default_threads())
    got = y[torch.from_numpy(segs).cuda()].cpu().numpy()
    check(got, ref, "sum", "f32", mode, counts=lens, what=f"sweep F={F}")
    del y
    torch.cuda.empty_cache()


def test_sweep_uniform_mean_int64(geot):
    w, L, y = run_full(geot, "sweep", F=4, op="mean", itype=torch.int64)
    assert y.shape == (w["S"], 4)
    rng = np.random.default_rng(7)
    segs, bounds = sample_segments(L, w["E"], rng, n_random=3000)
    rows, loc, lens = sub_problem(segs, bounds)
    X = synth.values(w["seed"], 0, 0, 4, "f32", "real", rows=rows)
    ref = oracle.segment_reduce(X, loc, len(segs), "mean")
    check(y[torch.from_numpy(segs).cuda()].cpu().numpy(), ref, "mean", "f32", "real", counts=lens, what="sweep mean")

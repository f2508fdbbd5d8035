"""Pins for the CPU oracle (oracle/geot_oracle.c) against things other than
itself: hand constants (tests/golden/, cited), a pure-Python brute-force double
loop, closed forms / library routines (numpy), exact integer-mode
arithmetic, and the invariants of SURVEY.md §8(c).  No GPU needed."""
import itertools

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.filterwarnings("ignore")


# ---------------------------------------------------------------- brute force
def brute_force(X, idx, S, op, src=None, w=None):
    """SPEC.md:61 'independent double-loop accumulator': for every output row s
    scan ALL edges e and fold those with idx[e] == s.  Python floats (fp64)."""
    X = np.asarray(X, dtype=np.float64)
    F = X.shape[1]
    Y = [[0.0] * F for _ in range(S)]
    for s in range(S):
        for f in range(F):
            acc, n, have = 0.0, 0, False
            for e in range(len(idx)):
                if int(idx[e]) != s:
                    continue
                v = float(X[int(src[e]) if src is not None else e, f])
                if w is not None:
                    v = float(w[e]) * v
                n += 1
                if op == "max":
                    acc = v if not have else (v if v > acc else acc)
                    have = True
                else:
                    acc += v
            if n == 0:
                Y[s][f] = 0.0
            elif op == "mean":
                Y[s][f] = acc / n
            else:
                Y[s][f] = acc
    return np.array(Y, dtype=np.float64).reshape(S, F)


def rand_case(rng, E, S, F, mode="real"):
    idx = np.sort(rng.integers(0, S, size=E)) if S else np.zeros(0, dtype=np.int64)
    if mode == "int":
        X = rng.integers(-8, 9, size=(E, F)).astype(np.float32)
    else:
        X = rng.random((E, F)).astype(np.float32)
    return idx, X


# ------------------------------------------------------------ worked examples
@pytest.mark.parametrize("name", ["W1", "W2"])
@pytest.mark.parametrize("op", ["sum", "mean", "max"])
def test_worked_examples(golden, name, op):
    g = golden["worked_examples"]
    x = np.array(g["x"], dtype=np.float32)
    c = g[name]
    dst, src, S = np.array(c["dst"]), np.array(c["src"]), c["S"]
    want = np.array(c[op], dtype=np.float64)
    # fused form
    r = oracle.gather_segment_reduce(x, src, dst, S, op)
    np.testing.assert_array_equal(r.y64, want)
    np.testing.assert_array_equal(r.rounded, want.astype(np.float32))
    # unfused form on the materialised messages msg = x[src]
    msg = x[src]
    if "msg_unfused" in c:
        np.testing.assert_array_equal(msg, np.array(c["msg_unfused"], dtype=np.float32))
    r2 = oracle.segment_reduce(msg, dst, S, op)
    np.testing.assert_array_equal(r2.y64, want)
    # int32 and int64 indices agree
    r3 = oracle.segment_reduce(msg, dst.astype(np.int32), S, op)
    np.testing.assert_array_equal(r3.y64, want)


@pytest.mark.parametrize("name", ["W1", "W2"])
def test_worked_offsets_counts_partition(golden, name):
    c = golden["worked_examples"][name]
    off = oracle.offsets(np.array(c["dst"]), c["S"])
    np.testing.assert_array_equal(off, c["offsets"])
    if "counts" in c:
        np.testing.assert_array_equal(np.diff(off), c["counts"])
    for P, b in c.get("partition", {}).items():
        sb, eb = oracle.partition(np.array(c["dst"]), c["S"], int(P))
        np.testing.assert_array_equal(sb, b["seg"])
        np.testing.assert_array_equal(eb, b["edge"])


def test_spec_hand_cases(golden):
    for c in golden["spec_cases"]["cases"]:
        r = oracle.segment_reduce(np.array(c["x"], dtype=np.float32), np.array(c["idx"]), c["S"], c["op"])
        np.testing.assert_array_equal(r.y64, np.array(c["y"], dtype=np.float64), err_msg=c["cite"])


def test_spec_pr_group_sums(golden):
    g = golden["spec_cases"]["pr_group"]
    keys = np.array(g["keys"])
    vals = np.array(g["values"], dtype=np.float32)[:, None]
    r = oracle.segment_reduce(vals, keys, 4, "sum")
    assert {str(k): int(v) for k, v in enumerate(r.y64[:, 0])} == {k: v for k, v in g["commits"].items()}


# --------------------------------------------------------------- brute force
@pytest.mark.parametrize("op", ["sum", "mean", "max"])
def test_brute_force_random_tiny(op):
    rng = np.random.default_rng(7)
    for trial in range(120):
        E = int(rng.integers(0, 40))
        S = int(rng.integers(1, 12))
        F = int(rng.integers(1, 5))
        idx, X = rand_case(rng, E, S, F, mode="real" if trial % 2 else "int")
        if op == "max":
            X = (X * 2 - 1).astype(np.float32)
        r = oracle.segment_reduce(X, idx, S, op)
        bf = brute_force(X, idx, S, op)
        # same fp64 ascending-e accumulation order => bitwise identical
        np.testing.assert_array_equal(r.y64, bf)


@pytest.mark.parametrize("op", ["sum", "mean", "max"])
def test_brute_force_fused_and_weighted(op):
    rng = np.random.default_rng(8)
    for trial in range(80):
        E = int(rng.integers(0, 30))
        S = int(rng.integers(1, 9))
        V = int(rng.integers(1, 9))
        F = int(rng.integers(1, 4))
        dst = np.sort(rng.integers(0, S, size=E))
        src = rng.integers(0, V, size=E)
        x = rng.random((V, F)).astype(np.float32)
        r = oracle.gather_segment_reduce(x, src, dst, S, op)
        np.testing.assert_array_equal(r.y64, brute_force(x, dst, S, op, src=src))
        if op == "sum":
            w = rng.random(E).astype(np.float32)
            rw = oracle.gather_segment_reduce(x, src, dst, S, op, weight=w)
            np.testing.assert_array_equal(rw.y64, brute_force(x, dst, S, op, src=src, w=w))


def test_brute_force_bf16_inputs():
    rng = np.random.default_rng(9)
    for _ in range(30):
        E, S, F = int(rng.integers(1, 30)), int(rng.integers(1, 7)), int(rng.integers(1, 4))
        idx = np.sort(rng.integers(0, S, size=E))
        v = (rng.integers(0, 256, size=(E, F)) / 256.0).astype(np.float32)  # exact in bf16
        bits = synth.f32_to_bf16_bits(v)
        for op in ("sum", "mean", "max"):
            r = oracle.segment_reduce(bits, idx, S, op)
            np.testing.assert_array_equal(r.y64, brute_force(v, idx, S, op))
            assert r.rounded.dtype == np.uint16


# ------------------------------------------------------------- closed forms
def test_identity_index_gives_X():
    """idx = arange(E), S = E  =>  Y = X."""
    rng = np.random.default_rng(1)
    X = rng.random((50, 7)).astype(np.float32)
    for op in ("sum", "mean", "max"):
        r = oracle.segment_reduce(X, np.arange(50), 50, op)
        np.testing.assert_array_equal(r.rounded, X)


def test_single_segment_is_column_sum():
    """One segment => numpy column sums / max / mean (library routines, fp64)."""
    rng = np.random.default_rng(2)
    X = rng.random((1000, 5)).astype(np.float32)
    idx = np.full(1000, 3)
    r = oracle.segment_reduce(X, idx, 6, "sum")
    np.testing.assert_allclose(r.y64[3], X.astype(np.float64).sum(axis=0), rtol=1e-13)
    assert np.all(r.y64[[0, 1, 2, 4, 5]] == 0)
    np.testing.assert_array_equal(oracle.segment_reduce(X, idx, 6, "max").y64[3], X.max(axis=0))
    np.testing.assert_allclose(oracle.segment_reduce(X, idx, 6, "mean").y64[3],
                               X.astype(np.float64).mean(axis=0), rtol=1e-13)


def test_fused_identity_src_equals_unfused():
    """src = identity => fused == unfused, bitwise."""
    rng = np.random.default_rng(3)
    idx, X = rand_case(rng, 300, 40, 6)
    for op in ("sum", "mean", "max"):
        a = oracle.segment_reduce(X, idx, 40, op)
        b = oracle.gather_segment_reduce(X, np.arange(300), idx, 40, op)
        np.testing.assert_array_equal(a.y64, b.y64)


def test_fused_equals_gather_then_reduce():
    """fused == segment_reduce(dst, x[src]) bitwise."""
    rng = np.random.default_rng(4)
    V, E, S, F = 30, 400, 25, 9
    x = rng.random((V, F)).astype(np.float32)
    src = rng.integers(0, V, size=E)
    dst = np.sort(rng.integers(0, S, size=E))
    for op in ("sum", "mean", "max"):
        np.testing.assert_array_equal(oracle.gather_segment_reduce(x, src, dst, S, op).y64,
                                      oracle.segment_reduce(x[src], dst, S, op).y64)


def test_fused_on_adjacency_is_dense_matmul():
    """fused sum on a 0/1 adjacency (Cora-shaped sizes) == numpy A @ x."""
    w = synth.workload("cora")
    L = synth.segment_lengths(w["E"], w["S"], "powerlaw", w["seed"])
    dst = synth.lengths_to_index(L, "i64")
    # unique (dst, src) pairs so A is 0/1
    rng = np.random.default_rng(5)
    src = np.empty_like(dst)
    off = synth.lengths_to_bounds(L)
    for s in range(w["S"]):
        n = int(L[s])
        if n:
            src[off[s]:off[s + 1]] = rng.choice(w["S"], size=n, replace=False)
    x = synth.values_f32(11, 0, w["S"], 8)
    A = np.zeros((w["S"], w["S"]))
    A[dst, src] = 1.0
    r = oracle.gather_segment_reduce(x, src, dst, w["S"], "sum")
    np.testing.assert_allclose(r.y64, A @ x.astype(np.float64), rtol=1e-12, atol=1e-12)


def test_weighted_is_dense_matmul():
    """8x8 random sparse (nnz=20) times 8x4 dense == numpy W @ X."""
    rng = np.random.default_rng(6)
    flat = np.sort(rng.choice(64, size=20, replace=False))
    dst, src = flat // 8, flat % 8
    wv = rng.random(20).astype(np.float32)
    x = rng.random((8, 4)).astype(np.float32)
    W = np.zeros((8, 8))
    W[dst, src] = wv
    r = oracle.gather_segment_reduce(x, src, dst, 8, "sum", weight=wv)
    np.testing.assert_allclose(r.y64, W @ x.astype(np.float64), rtol=1e-12)
    r0 = oracle.gather_segment_reduce(x, src, dst, 8, "sum", weight=np.zeros(20, np.float32))
    assert np.all(r0.y64 == 0)
    r1 = oracle.gather_segment_reduce(x, src, dst, 8, "sum", weight=np.ones(20, np.float32))
    np.testing.assert_array_equal(r1.y64, oracle.gather_segment_reduce(x, src, dst, 8, "sum").y64)


# ----------------------------------------------------------------- invariants
def test_invariants_random():
    rng = np.random.default_rng(10)
    for kind in synth.STRESS_KINDS:
        L = synth.stress_lengths(kind, 3000, 200, seed=3)
        idx = synth.lengths_to_index(L)
        X = synth.values_f32(4, 0, 3000, 3, "f32", "int")
        s = oracle.segment_reduce(X, idx, 200, "sum")
        m = oracle.segment_reduce(X, idx, 200, "mean")
        mx = oracle.segment_reduce(X, idx, 200, "max")
        counts = np.diff(oracle.offsets(idx, 200))
        np.testing.assert_array_equal(counts, L)
        # conservation (exact in integer mode)
        np.testing.assert_array_equal(s.y64.sum(axis=0), X.astype(np.float64).sum(axis=0))
        # empty -> 0 for all ops
        empty = counts == 0
        for r in (s, m, mx):
            assert np.all(r.y64[empty] == 0) and not np.any(np.signbit(r.y64[empty]))
        # mean * count == sum
        np.testing.assert_allclose(m.y64 * counts[:, None], s.y64, rtol=1e-14, atol=0)
        # max >= every member and equals one member
        for seg in np.nonzero(~empty)[0][:50]:
            rows = X[idx == seg]
            assert np.all(mx.y64[seg] >= rows.max(axis=0)) and np.all(mx.y64[seg] == rows.max(axis=0))
        # permuting rows inside each segment leaves the result unchanged (integers: exact)
        perm = np.arange(3000)
        off = synth.lengths_to_bounds(L)
        for seg in range(200):
            a, b = off[seg], off[seg + 1]
            perm[a:b] = a + rng.permutation(b - a)
        np.testing.assert_array_equal(oracle.segment_reduce(X[perm], idx, 200, "sum").y64, s.y64)


def test_integer_mode_exact_long_segment():
    """Integer mode: every partial sum is an exact integer."""
    E = 200_000
    X = synth.values_f32(3, 0, E, 2, "f32", "int")
    idx = np.zeros(E, dtype=np.int32)
    r = oracle.segment_reduce(X, idx, 1, "sum")
    exact = X.astype(np.int64).sum(axis=0)
    np.testing.assert_array_equal(r.y64[0], exact.astype(np.float64))
    np.testing.assert_array_equal(r.rounded[0], exact.astype(np.float32))


def test_threads_do_not_change_result():
    w = synth.workload("cora")
    L = synth.segment_lengths(w["E"], w["S"], "powerlaw", w["seed"])
    idx = synth.lengths_to_index(L)
    X = synth.values_f32(w["seed"], 0, w["E"], w["F"])
    a = oracle.segment_reduce(X, idx, w["S"], "sum", nthreads=1)
    b = oracle.segment_reduce(X, idx, w["S"], "sum", nthreads=7)
    np.testing.assert_array_equal(a.y64, b.y64)


# ------------------------------------------------------------------ rounding
def test_rounding_to_dtype_matches_torch():
    """R5/R6: fp32 = one RN of the fp64 value; bf16 = RNE_bf16(RN_fp32(y)).
    Pinned against torch's CPU dtype conversions (library routines)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(12)
    idx = np.sort(rng.integers(0, 50, size=800))
    X = rng.random((800, 4)).astype(np.float32)
    bits = synth.f32_to_bf16_bits(synth.bf16_bits_to_f32(synth.f32_to_bf16_bits(X)))
    for op in ("sum", "mean", "max"):
        r = oracle.segment_reduce(X, idx, 50, op)
        np.testing.assert_array_equal(r.rounded, torch.tensor(r.y64).float().numpy())
        rb = oracle.segment_reduce(bits, idx, 50, op)
        want = torch.tensor(rb.y64).float().bfloat16().view(torch.int16).numpy().view(np.uint16)
        np.testing.assert_array_equal(rb.rounded, want)


def test_bf16_rne_ties_oracle():
    """R5: the oracle's bf16 output is round-to-nearest-EVEN of the fp32 value.
    Segments of exactly representable bf16 inputs whose sums fall exactly on a
    bf16 tie (or just above one), with the expected bf16 values written by hand
    (bf16 keeps 8 significant bits: the spacing just above 1.0 is 2^-7)."""
    vals = [[1.0], [2 ** -8],                    # seg 0: 1 + 2^-8, tie -> 1.0 (even)
            [1.0 + 2 ** -7], [2 ** -8],          # seg 1: 1 + 3*2^-8, tie -> 1 + 2^-6 (even)
            [1.0], [2 ** -8], [2 ** -20],        # seg 2: just above the tie -> 1 + 2^-7
            [-1.0], [-(2 ** -8)],                # seg 3: -(1 + 2^-8), tie -> -1.0
            [3.0], [2 ** -7]]                    # seg 4: 3 + 2^-7, tie between 3 and 3 + 2^-6 -> 3.0
    idx = np.array([0, 0, 1, 1, 2, 2, 2, 3, 3, 4, 4])
    bits = synth.f32_to_bf16_bits(np.array(vals, np.float32))
    assert np.array_equal(synth.bf16_bits_to_f32(bits), np.array(vals, np.float32))  # inputs exact in bf16
    r = oracle.segment_reduce(bits, idx, 5, "sum")
    got = synth.bf16_bits_to_f32(r.rounded)[:, 0]
    np.testing.assert_array_equal(got, np.array([1.0, 1.0 + 2 ** -6, 1.0 + 2 ** -7, -1.0, 3.0], np.float32))
    np.testing.assert_array_equal(r.y64[:, 0], [1 + 2 ** -8, 1 + 3 * 2 ** -8, 1 + 2 ** -8 + 2 ** -20,
                                                 -(1 + 2 ** -8), 3 + 2 ** -7])


# ------------------------------------------------------------ offsets / part.
def test_offsets_match_searchsorted():
    rng = np.random.default_rng(13)
    for _ in range(50):
        S = int(rng.integers(1, 60))
        idx = np.sort(rng.integers(0, S, size=int(rng.integers(0, 300))))
        off = oracle.offsets(idx, S)
        np.testing.assert_array_equal(off, np.searchsorted(idx, np.arange(S + 1), side="left"))
        assert off[0] == 0 and off[-1] == len(idx) and np.all(np.diff(off) >= 0)


def test_partition_invariants():
    rng = np.random.default_rng(14)
    for _ in range(1500):
        S = int(rng.integers(1, 30))
        E = int(rng.integers(0, 80))
        idx = np.sort(rng.integers(0, S, size=E))
        P = int(rng.integers(1, 10))
        sb, eb = oracle.partition(idx, S, P)
        off = np.searchsorted(idx, np.arange(S + 1))
        assert sb[0] == 0 and sb[-1] == S and eb[0] == 0 and eb[-1] == E
        assert np.all(np.diff(sb) >= 0) and np.all(np.diff(eb) >= 0)
        np.testing.assert_array_equal(eb, off[sb])          # e_p = offsets[s_p]
        maxlen = int(np.diff(off).max()) if S else 0
        bound = -(-E // P) + max(maxlen - 1, 0)
        assert np.all(np.diff(eb) <= bound)                  # balance bound (R18)
        # every edge's segment lies in its owner's segment range
        for p in range(P):
            seg = idx[eb[p]:eb[p + 1]]
            assert np.all((seg >= sb[p]) & (seg < sb[p + 1]))


def test_validate_bits():
    ok = np.array([0, 0, 1, 3])
    assert oracle.validate(ok, 4) == 0
    assert oracle.validate(np.array([0, 2, 1]), 4) == oracle.BAD_UNSORTED
    assert oracle.validate(np.array([0, 1, 4]), 4) == oracle.BAD_IDX_RANGE
    assert oracle.validate(np.array([-1, 0]), 4) == oracle.BAD_IDX_RANGE
    assert oracle.validate(ok, 4, src_idx=np.array([0, 1, 2, 5]), num_x_rows=5) == oracle.BAD_SRC_RANGE
    assert oracle.validate(np.array([3, 1]), 3, src_idx=np.array([0, 9]), num_x_rows=5) == 7


def test_empty_inputs():
    r = oracle.segment_reduce(np.zeros((0, 3), np.float32), np.zeros(0, np.int64), 5, "max")
    assert r.y64.shape == (5, 3) and np.all(r.y64 == 0)
    r = oracle.segment_reduce(np.zeros((0, 3), np.float32), np.zeros(0, np.int64), 0, "sum")
    assert r.y64.shape == (0, 3)
    sb, eb = oracle.partition(np.zeros(0, np.int64), 5, 3)
    np.testing.assert_array_equal(sb, [0, 0, 0, 5])
    np.testing.assert_array_equal(eb, [0, 0, 0, 0])


def test_exhaustive_length8_keys_group_sums():
    """all 6435 non-decreasing length-8 key sequences over 8 symbols:
    the oracle's per-key sums equal the exact integer sums."""
    n = 0
    vals = np.arange(1, 9, dtype=np.float32)[:, None]
    for keys in itertools.combinations_with_replacement(range(8), 8):
        k = np.array(keys)
        r = oracle.segment_reduce(vals, k, 8, "sum")
        want = np.bincount(k, weights=np.arange(1, 9), minlength=8)
        assert np.array_equal(r.y64[:, 0], want)
        n += 1
    assert n == 6435


# ------------------------------------------------------- absum (tolerance A)
# A[s,f] = sum_{e in segment s} |X[e,f]| is the denominator of every real-mode
# sum/mean parity tolerance (R14; SURVEY.md §8(c) step 3 and the
# "Parity rule").  It is pinned here against things other than the oracle: a
# numpy column sum of |X|, the identity A == Y for non-negative inputs, a
# pure-Python double loop, and the weighted/fused forms' |w * x[src]|.
def _brute_absum(X, idx, S, src=None, w=None):
    X = np.asarray(X, dtype=np.float64)
    F = X.shape[1]
    A = [[0.0] * F for _ in range(S)]
    for s in range(S):
        for e in range(len(idx)):
            if int(idx[e]) != s:
                continue
            for f in range(F):
                v = float(X[int(src[e]) if src is not None else e, f])
                if w is not None:
                    v = float(w[e]) * v
                A[s][f] += abs(v)
    return np.array(A, dtype=np.float64).reshape(S, F)


def test_absum_single_segment_is_numpy_abs_column_sum():
    """One segment among empties: A[3] = numpy |X|.sum(axis=0); empties 0."""
    rng = np.random.default_rng(31)
    X = (rng.random((1500, 6)) * 2 - 1).astype(np.float32)
    idx = np.full(1500, 3)
    for op in ("sum", "mean", "max"):  # A does not depend on the op
        r = oracle.segment_reduce(X, idx, 7, op)
        np.testing.assert_allclose(r.absum[3], np.abs(X.astype(np.float64)).sum(axis=0), rtol=1e-13)
        assert np.all(r.absum[[0, 1, 2, 4, 5, 6]] == 0)


def test_absum_equals_sum_for_nonnegative_inputs():
    """X >= 0 => |x| = x, accumulated in the same order: A == Y64 bitwise, for
    every segment (a missing per-segment reset would carry the previous
    segment's total into A)."""
    for kind in ("powerlaw", "gaps", "alternating", "singletons"):
        L = synth.stress_lengths(kind, 4000, 300, seed=5)
        idx = synth.lengths_to_index(L)
        X = synth.values_f32(9, 0, 4000, 5, "f32", "real")  # U[0,1)
        r = oracle.segment_reduce(X, idx, 300, "sum")
        np.testing.assert_array_equal(r.absum, r.y64)
        m = oracle.segment_reduce(X, idx, 300, "mean")
        np.testing.assert_array_equal(m.absum, r.y64)


def test_absum_signed_brute_force():
    """Signed values, random sorted index with empty segments: A equals the
    Python double loop (same fp64 ascending-e order => bitwise)."""
    rng = np.random.default_rng(32)
    for trial in range(60):
        E, S, F = int(rng.integers(0, 50)), int(rng.integers(1, 10)), int(rng.integers(1, 4))
        idx = np.sort(rng.integers(0, S, size=E))
        X = (rng.random((E, F)) * 2 - 1).astype(np.float32)
        for op in ("sum", "mean", "max"):
            np.testing.assert_array_equal(oracle.segment_reduce(X, idx, S, op).absum, _brute_absum(X, idx, S))
        # bf16 inputs: A from the bf16-valued inputs
        bits = synth.f32_to_bf16_bits(X)
        np.testing.assert_array_equal(oracle.segment_reduce(bits, idx, S, "sum").absum,
                                      _brute_absum(synth.bf16_bits_to_f32(bits), idx, S))


def test_absum_fused_and_weighted():
    """Fused form: A = sum |x[src[e]]|; weighted: A = sum |w[e] * x[src[e]]|
    (signed weights, so |w x| != w |x|)."""
    rng = np.random.default_rng(33)
    for trial in range(40):
        E, S, V, F = int(rng.integers(0, 40)), int(rng.integers(1, 8)), int(rng.integers(1, 9)), int(rng.integers(1, 4))
        dst = np.sort(rng.integers(0, S, size=E))
        src = rng.integers(0, V, size=E)
        x = (rng.random((V, F)) * 2 - 1).astype(np.float32)
        w = (rng.random(E) * 2 - 1).astype(np.float32)
        r = oracle.gather_segment_reduce(x, src, dst, S, "sum")
        np.testing.assert_array_equal(r.absum, _brute_absum(x, dst, S, src=src))
        rw = oracle.gather_segment_reduce(x, src, dst, S, "sum", weight=w)
        np.testing.assert_array_equal(rw.absum, _brute_absum(x, dst, S, src=src, w=w))
        assert np.all(rw.absum >= np.abs(rw.y64))  # triangle inequality


def test_absum_bounds_sum_and_empty_rows_zero():
    """|Y| <= A everywhere (triangle inequality), and empty segments have A = 0."""
    L = synth.stress_lengths("gaps", 5000, 400, seed=6)
    idx = synth.lengths_to_index(L)
    X = synth.values_f32(10, 0, 5000, 4, "f32", "signed")
    r = oracle.segment_reduce(X, idx, 400, "sum")
    assert np.all(r.absum >= np.abs(r.y64))
    assert np.all(r.absum[L == 0] == 0) and np.any(L == 0)
    assert np.all(r.absum[L > 0] > 0)


# ------------------------------------------------------ exact split (R21)
@pytest.mark.parametrize("name", ["W1", "W2"])
def test_partition_exact_worked(golden, name):
    """Hand constants (tests/golden/worked_examples.json) of the exact edge
    split, SURVEY.md §8(e) 'Alternative partition', R21."""
    c = golden["worked_examples"][name]
    for P, b in c["partition_exact"].items():
        sb, eb, keys = oracle.partition_exact(np.array(c["dst"]), c["S"], int(P))
        np.testing.assert_array_equal(sb, b["seg"])
        np.testing.assert_array_equal(eb, b["edge"])
        np.testing.assert_array_equal(keys, b["keys"])


def test_partition_exact_invariants():
    """Edge bounds are exactly floor(pE/P) (balance within one edge); row
    bounds are monotone, cover [0, S), and every segment's row lies in the part
    holding its first edge; the keys are the edges on both sides of each split."""
    rng = np.random.default_rng(15)
    for _ in range(800):
        S = int(rng.integers(1, 25))
        E = int(rng.integers(0, 70))
        idx = np.sort(rng.integers(0, S, size=E))
        P = int(rng.integers(1, 10))
        sb, eb, keys = oracle.partition_exact(idx, S, P)
        np.testing.assert_array_equal(eb, [(p * E) // P for p in range(P + 1)])
        assert sb[0] == 0 and sb[-1] == S and np.all(np.diff(sb) >= 0)
        for p in range(P + 1):
            assert keys[p, 0] == (idx[eb[p] - 1] if eb[p] > 0 else -1)
            assert keys[p, 1] == (idx[eb[p]] if eb[p] < E else -1)
        first = np.searchsorted(idx, np.arange(S))  # first edge of every segment (E if empty)
        for s in range(S):
            if first[s] < E and idx[first[s]] == s:
                owner = int(np.searchsorted(eb, first[s], side="right") - 1)
                while eb[owner] == eb[owner + 1]:  # skip empty parts
                    owner += 1
                assert sb[owner] <= s < sb[owner + 1], (s, owner, sb, eb)

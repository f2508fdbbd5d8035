"""The warp segmented scan of the narrow kernel (narrow.cuh warp_segscan — the
shfl doubling loop of Alg. 1) run on the GPU through the
self-test hook geot_selftest_warp_segscan, against a brute force:

  * SPEC.md:79 / :457 — every one of the 6,435 non-decreasing length-8 key
    sequences over 8 symbols (4 independent sequences per warp, lanes 8j..8j+7);
  * 10,000 random non-decreasing 16-lane and 32-lane sequences each.

Per lane the scan must return the fold (sum / max) of the values from its
segment's first lane through itself and, for mean, that first lane's index.
Integer values: sums are exact, so the comparison is bit-exact."""
import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def geot():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_03019_b200 as g
    return g


def run_scan(geot, keys, vals, op):
    from paper_2404_03019_b200 import _lib
    n = keys.size
    assert n % 32 == 0
    k = torch.from_numpy(keys.astype(np.int32)).cuda()
    v = torch.from_numpy(vals.astype(np.float32)).cuda()
    ov = torch.empty(n, dtype=torch.float32, device="cuda")
    of = torch.empty(n, dtype=torch.int32, device="cuda")
    op_ = torch.empty(n, dtype=torch.int64, device="cuda")
    opc = {"sum": 0, "mean": 1, "max": 2}[op]
    import ctypes
    st = _lib.load().geot_selftest_warp_segscan(ctypes.c_void_p(k.data_ptr()), ctypes.c_void_p(v.data_ptr()), n // 32,
                                                opc, ctypes.c_void_p(ov.data_ptr()), ctypes.c_void_p(of.data_ptr()),
                                                ctypes.c_void_p(op_.data_ptr()),
                                                ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    _lib.check(st, "geot_selftest_warp_segscan")
    torch.cuda.synchronize()
    return ov.cpu().numpy(), of.cpu().numpy(), op_.cpu().numpy()


def brute(keys, vals, op):
    """Per lane, walking the lanes in order (vectorised over warps only): the
    segment's first lane, and the fold of its values up to this lane."""
    k = keys.reshape(-1, 32)
    v = vals.reshape(-1, 32).astype(np.float64)
    start = np.zeros_like(k)
    out = v.copy()
    for lane in range(1, 32):
        same = k[:, lane] == k[:, lane - 1]
        start[:, lane] = np.where(same, start[:, lane - 1], lane)
        prev = out[:, lane - 1]
        out[:, lane] = np.where(same, np.maximum(prev, v[:, lane]) if op == "max" else prev + v[:, lane], v[:, lane])
    return out.reshape(-1), start.reshape(-1)


def check(geot, keys, vals):
    for op in ("sum", "mean", "max"):
        v, f, p = run_scan(geot, keys, vals, op)
        want, start = brute(keys, vals, op)
        np.testing.assert_array_equal(v.astype(np.float64), want)
        assert np.all(f == 1)
        if op == "mean":
            np.testing.assert_array_equal(p, start)


def test_exhaustive_length8_sequences(geot):
    seqs = list(itertools.combinations_with_replacement(range(8), 8))
    assert len(seqs) == 6435
    seqs += [(0,) * 8] * ((-len(seqs)) % 4)  # pad to whole warps
    keys = np.array([[k + 8 * (j % 4) for k in s] for j, s in enumerate(seqs)], dtype=np.int64).reshape(-1)
    rng = np.random.default_rng(79)
    vals = rng.integers(-9, 10, size=keys.size).astype(np.float32)
    check(geot, keys, vals)
    # the values 1..8 of S:79 (each position's own index + 1)
    check(geot, keys, np.tile(np.arange(1, 9, dtype=np.float32), keys.size // 8))


@pytest.mark.parametrize("group", [16, 32])
def test_random_sequences(geot, group):
    rng = np.random.default_rng(457 + group)
    n_seq = 10_000
    per_warp = 32 // group
    n_seq += (-n_seq) % per_warp
    keys = np.sort(rng.integers(0, group // 2 + 1, size=(n_seq, group)), axis=1)
    keys += (np.arange(n_seq) % per_warp)[:, None] * (group + 1)  # independent sequences within a warp
    vals = rng.integers(-100, 101, size=keys.size).astype(np.float32)
    check(geot, keys.reshape(-1), vals)

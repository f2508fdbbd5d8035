"""CPU oracle for GeoT's segment-reduction hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this package.  It shares no code with the
CUDA path (`paper_2404_03019_b200/`); the C source it wraps is
`oracle/geot_oracle.c` (fp64 accumulation, the plain definitions of PAPER.md
§II-B; see that file's header for citations and pins).

Numpy in / numpy out.  Values may be given as float32 (fp32) or as uint16 bf16
bit patterns (bf16); indices as int32 or int64.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "geot_oracle.c")
_LIB = os.path.join(_HERE, "libgeot_oracle.so")

SUM, MEAN, MAX = 0, 1, 2
OPS = {"sum": SUM, "mean": MEAN, "max": MAX}
BAD_UNSORTED, BAD_IDX_RANGE, BAD_SRC_RANGE = 1, 2, 4

_lib = None


def build(force: bool = False, src: str = _SRC, out: str = _LIB) -> str:
    """gcc -O2 (no -ffast-math) the oracle into oracle/libgeot_oracle.so.
    (`src`/`out` other than the defaults: the mutation tests build deliberately
    broken copies to show that the pins catch them.)"""
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-fno-fast-math",
                               "-o", tmp, src, "-lpthread", "-lm"])
        os.replace(tmp, out)
    return out


def _load(path):
    L = ctypes.CDLL(path)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    L.oracle_validate.argtypes = [vp, i32, i64, i64, vp, i64]
    L.oracle_validate.restype = i32
    L.oracle_offsets.argtypes = [vp, i32, i64, i64, vp]
    L.oracle_offsets.restype = None
    L.oracle_segment_reduce.argtypes = [vp, i32, vp, i32, i64, i64, i64, i32, vp, vp, vp, i32]
    L.oracle_segment_reduce.restype = i32
    L.oracle_gather_segment_reduce.argtypes = [vp, i32, i64, vp, vp, i32, vp, i64, i64, i64, i32,
                                               vp, vp, vp, i32]
    L.oracle_gather_segment_reduce.restype = i32
    L.oracle_partition.argtypes = [vp, i32, i64, i64, i32, vp, vp]
    L.oracle_partition.restype = i32
    L.oracle_partition_exact.argtypes = [vp, i32, i64, i64, i32, vp, vp, vp]
    L.oracle_partition_exact.restype = i32
    L.oracle_segment_reduce_backward.argtypes = [vp, vp, i32, vp, i32, i64, i64, i64, i32, vp]
    L.oracle_segment_reduce_backward.restype = i32
    L.oracle_gather_segment_reduce_backward.argtypes = [vp, vp, i64, vp, vp, i32, vp, i64, i64, i64, i32, vp,
                                                        vp]
    L.oracle_gather_segment_reduce_backward.restype = i32
    return L


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = _load(_LIB)
    return _lib


class use_library:
    """Context manager: route every oracle call through another build of the
    C source (mutation tests only)."""

    def __init__(self, path):
        self.path = path

    def __enter__(self):
        global _lib
        self.saved, _lib = lib(), _load(self.path)
        return self

    def __exit__(self, *a):
        global _lib
        _lib = self.saved


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _index(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.int32:
        return a, 0
    return np.ascontiguousarray(a, dtype=np.int64), 1


def _vals(X):
    X = np.ascontiguousarray(X)
    if X.dtype == np.uint16:
        return X, 1
    return np.ascontiguousarray(X, dtype=np.float32), 0


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class Result:
    """y64: fp64 result; absum: per-element sum |x| (tolerance denominator);
    rounded: the result rounded to the input dtype (float32, or uint16 bf16 bits)."""

    def __init__(self, y64, absum, rounded):
        self.y64, self.absum, self.rounded = y64, absum, rounded


def validate(idx, S, src_idx=None, num_x_rows=0) -> int:
    idx, it = _index(idx)
    if src_idx is not None:
        src_idx = np.ascontiguousarray(src_idx, dtype=idx.dtype)
    return int(lib().oracle_validate(_ptr(idx), it, idx.shape[0], S, _ptr(src_idx), num_x_rows))


def offsets(idx, S) -> np.ndarray:
    idx, it = _index(idx)
    out = np.zeros(S + 1, dtype=np.int64)
    lib().oracle_offsets(_ptr(idx), it, idx.shape[0], S, _ptr(out))
    return out


def segment_reduce(X, idx, S, op="sum", nthreads=1) -> Result:
    """Y[s,:] = op over {X[e,:] : idx[e] == s}."""
    X, dt = _vals(X)
    idx, it = _index(idx)
    E = idx.shape[0]
    if X.ndim != 2 or X.shape[0] != E:
        raise ValueError("X must be [nnz, F]")
    F = X.shape[1]
    y = np.zeros((S, F), dtype=np.float64)
    a = np.zeros((S, F), dtype=np.float64)
    r = np.zeros((S, F), dtype=X.dtype)
    rc = lib().oracle_segment_reduce(_ptr(X), dt, _ptr(idx), it, E, S, F, OPS[op], _ptr(y), _ptr(a),
                                     _ptr(r), nthreads)
    if rc:
        raise ValueError("oracle_segment_reduce rejected its arguments")
    return Result(y, a, r)


def gather_segment_reduce(x, src_idx, dst_idx, S, op="sum", weight=None, nthreads=1) -> Result:
    """Fused form, P:293 / P:330: Y[s,:] = op over {w[e] * x[src[e],:] : dst[e] == s}."""
    x, dt = _vals(x)
    dst_idx, it = _index(dst_idx)
    src_idx = np.ascontiguousarray(src_idx, dtype=dst_idx.dtype)
    E = dst_idx.shape[0]
    V, F = x.shape
    w = None if weight is None else np.ascontiguousarray(weight, dtype=np.float32)
    y = np.zeros((S, F), dtype=np.float64)
    a = np.zeros((S, F), dtype=np.float64)
    r = np.zeros((S, F), dtype=x.dtype)
    rc = lib().oracle_gather_segment_reduce(_ptr(x), dt, V, _ptr(src_idx), _ptr(dst_idx), it, _ptr(w),
                                            E, S, F, OPS[op], _ptr(y), _ptr(a), _ptr(r), nthreads)
    if rc:
        raise ValueError("oracle_gather_segment_reduce rejected its arguments")
    return Result(y, a, r)


def segment_reduce_backward(dY, X, idx, op="sum"):
    """VJP of segment_reduce w.r.t. X (fp64): dX[e] = g * dY[idx[e]] (see the C header)."""
    X, dt = _vals(X)
    idx, it = _index(idx)
    dY = np.ascontiguousarray(dY, dtype=np.float64)
    S, F = dY.shape
    dX = np.zeros((idx.shape[0], F), dtype=np.float64)
    rc = lib().oracle_segment_reduce_backward(_ptr(dY), _ptr(X), dt, _ptr(idx), it, idx.shape[0], S, F, OPS[op],
                                              _ptr(dX))
    if rc:
        raise ValueError("oracle_segment_reduce_backward rejected its arguments")
    return dX


def gather_segment_reduce_backward(dY, x, src_idx, dst_idx, op="sum", weight=None):
    """(dx, dw) of the (weighted) fused form, fp64; x fp32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    dst_idx, it = _index(dst_idx)
    src_idx = np.ascontiguousarray(src_idx, dtype=dst_idx.dtype)
    dY = np.ascontiguousarray(dY, dtype=np.float64)
    S, F = dY.shape
    V = x.shape[0]
    E = dst_idx.shape[0]
    w = None if weight is None else np.ascontiguousarray(weight, dtype=np.float32)
    dx = np.zeros((V, F), dtype=np.float64)
    dw = np.zeros(E, dtype=np.float64)
    rc = lib().oracle_gather_segment_reduce_backward(_ptr(dY), _ptr(x), V, _ptr(src_idx), _ptr(dst_idx), it, _ptr(w),
                                                     E, S, F, OPS[op], _ptr(dx), _ptr(dw))
    if rc:
        raise ValueError("oracle_gather_segment_reduce_backward rejected its arguments")
    return dx, dw


def partition(idx, S, nparts):
    idx, it = _index(idx)
    sb = np.zeros(nparts + 1, dtype=np.int64)
    eb = np.zeros(nparts + 1, dtype=np.int64)
    rc = lib().oracle_partition(_ptr(idx), it, idx.shape[0], S, nparts, _ptr(sb), _ptr(eb))
    if rc:
        raise ValueError("oracle_partition rejected its arguments")
    return sb, eb


def partition_exact(idx, S, nparts):
    """Exact edge split (R21): (seg_bounds, edge_bounds, boundary_keys [nparts+1, 2])."""
    idx, it = _index(idx)
    sb = np.zeros(nparts + 1, dtype=np.int64)
    eb = np.zeros(nparts + 1, dtype=np.int64)
    keys = np.zeros((nparts + 1, 2), dtype=np.int64)
    rc = lib().oracle_partition_exact(_ptr(idx), it, idx.shape[0], S, nparts, _ptr(sb), _ptr(eb), _ptr(keys))
    if rc:
        raise ValueError("oracle_partition_exact rejected its arguments")
    return sb, eb, keys

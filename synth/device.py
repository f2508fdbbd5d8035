"""Device side of the shared input generator (synth/csrc/synth.cu via ctypes).

Generates the same values as the host generator in synth/__init__.py directly
in device memory (large workloads never touch the host), keyed by GLOBAL edge
id so every shard of a multi-GPU run sees the same global input.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

import synth

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgeot_synth.so")
_lib = None
_MODE = {"real": 0, "signed": 1, "int": 2}


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} missing: run `python tools/build.py`")
        L = ctypes.CDLL(_LIB)
        vp, ll, i32, u64 = ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_uint64
        L.synth_fill_values.argtypes = [vp, i32, u64, ll, ll, ll, i32, vp]
        L.synth_expand_index.argtypes = [vp, ll, ll, ll, vp, i32, ll, vp]
        L.synth_src_index.argtypes = [vp, i32, u64, ll, ll, ll, vp]
        for f in (L.synth_fill_values, L.synth_expand_index, L.synth_src_index):
            f.restype = i32
        _lib = L
    return _lib


def _st(dev):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _chk(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what}: cudaError {rc}")


def fill_values(out: torch.Tensor, seed: int, e_begin: int, mode: str = "real"):
    """out: [n, F] float32/bfloat16 CUDA tensor, rows = global edges e_begin.."""
    n, F = out.shape
    dt = 0 if out.dtype == torch.float32 else 1
    with torch.cuda.device(out.device):
        _chk(lib().synth_fill_values(ctypes.c_void_p(out.data_ptr()), dt, seed & synth.MASK64, e_begin, n, F,
                                     _MODE[mode], _st(out.device)), "synth_fill_values")
    return out


def values(n, F, seed, e_begin=0, dtype=torch.float32, mode="real", device="cuda"):
    return fill_values(torch.empty((n, F), dtype=dtype, device=device), seed, e_begin, mode)


def expand_index(bounds_dev: torch.Tensor, e_begin: int, n: int, itype=torch.int32, key_offset: int = 0):
    """idx for global edges [e_begin, e_begin+n) from device bounds (int64, S+1)."""
    S = bounds_dev.numel() - 1
    out = torch.empty(n, dtype=itype, device=bounds_dev.device)
    with torch.cuda.device(out.device):
        _chk(lib().synth_expand_index(ctypes.c_void_p(bounds_dev.data_ptr()), S, e_begin, n,
                                      ctypes.c_void_p(out.data_ptr()), 0 if itype == torch.int32 else 1,
                                      key_offset, _st(out.device)), "synth_expand_index")
    return out


def src_index(n, V, seed2, e_begin=0, itype=torch.int32, device="cuda"):
    out = torch.empty(n, dtype=itype, device=device)
    with torch.cuda.device(out.device):
        _chk(lib().synth_src_index(ctypes.c_void_p(out.data_ptr()), 0 if itype == torch.int32 else 1,
                                   seed2 & synth.MASK64, e_begin, n, V, _st(out.device)), "synth_src_index")
    return out


def index_from_lengths(L: np.ndarray, itype=torch.int32, device="cuda"):
    b = torch.from_numpy(synth.lengths_to_bounds(L)).to(device)
    return expand_index(b, 0, int(L.sum()), itype)

"""ctypes loader of libgeot.so (the C ABI declared in include/geot.h).

No fallback of any kind: if the library is missing or fails to load, this
module raises, so the product path fails loudly instead of silently running
something else.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# GEOT_LIB_OVERRIDE: an alternative build of the same library (kernel A/B experiments only)
LIB_PATH = os.environ.get("GEOT_LIB_OVERRIDE") or os.path.join(_HERE, "libgeot.so")

SUM, MEAN, MAX = 0, 1, 2
F32, BF16 = 0, 1
I32, I64 = 0, 1
VARIANT_AUTO, VARIANT_EDGE_TILE, VARIANT_NARROW = 0, 1, 2

STATUS = {
    0: "GEOT_OK", 1: "GEOT_ERR_INVALID_VALUE", 2: "GEOT_ERR_UNSUPPORTED", 3: "GEOT_ERR_WORKSPACE_TOO_SMALL",
    4: "GEOT_ERR_UNSORTED_INDEX", 5: "GEOT_ERR_INDEX_OUT_OF_RANGE", 6: "GEOT_ERR_SRC_OUT_OF_RANGE",
    7: "GEOT_ERR_CUDA",
}


class GeotConfig(ctypes.Structure):
    """Mirror of `geot_config` (include/geot.h)."""
    _fields_ = [("variant", ctypes.c_int32), ("vec_elems", ctypes.c_int32), ("lanes_per_row", ctypes.c_int32),
                ("vecs_per_lane", ctypes.c_int32), ("rows_per_group", ctypes.c_int32),
                ("warps_per_cta", ctypes.c_int32), ("ctas_per_sm", ctypes.c_int32), ("stages", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class GeotError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)}")


# exported symbol -> (argtypes, restype); the single source of truth for the
# ABI as seen from Python (tests check it against include/geot.h).
_vp, _i64, _i32, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
_cfgp = ctypes.POINTER(GeotConfig)
SIGNATURES = {
    "geot_status_string": ([_i32], ctypes.c_char_p),
    "geot_abi_version": ([], _i32),
    "geot_last_cuda_error": ([], ctypes.c_char_p),
    "geot_launch_count": ([], ctypes.c_uint64),
    "geot_profile_events": ([_vp, _vp], None),
    "geot_select_config": ([_i64, _i64, _i64, _i32, _i32, _i32, _i32, _cfgp], _i32),
    "geot_workspace_size": ([_i64, _i64, _i64, _i32, _i32, _i32, _i32, _cfgp], _sz),
    "geot_workspace_init": ([_vp, _sz, _vp], _i32),
    "geot_workspace_status": ([_vp, _sz, _vp, ctypes.POINTER(ctypes.c_int32)], _i32),
    "geot_select_config_ex": ([_i64, _i64, _i64, _i32, _i32, _i32, _i32, ctypes.c_double, _cfgp], _i32),
    "geot_select_hand_rules": ([_i64, _i64, _i64, _i32, _i32, _cfgp], _i32),
    "geot_select_tree": ([ctypes.c_double] * 7 + [ctypes.POINTER(ctypes.c_int32)], None),
    "geot_selector_provenance": ([], ctypes.c_char_p),
    "geot_segment_reduce": ([_vp, _vp, _i64, _i64, _i64, _i32, _i32, _i32, _vp, _vp, _sz, _vp], _i32),
    "geot_segment_reduce_ex": ([_vp, _vp, _i64, _i64, _i64, _i64, _i32, _i32, _i32, _vp, _vp, _sz, _cfgp, _vp],
                               _i32),
    "geot_segment_reduce_allgather": ([_vp, _vp, _i64, _i64, _i64, _i64, _i32, _i32, _i32, ctypes.POINTER(_vp), _i32,
                                       _vp, _sz, _cfgp, _vp], _i32),
    "geot_segment_reduce_multicast": ([_vp, _vp, _i64, _i64, _i64, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _sz, _cfgp,
                                       _vp], _i32),
    "geot_gather_segment_reduce": ([_vp, _i64, _vp, _vp, _i64, _i64, _i64, _i32, _i32, _i32, _vp, _vp, _sz, _vp],
                                   _i32),
    "geot_gather_weight_segment_reduce": ([_vp, _i64, _vp, _vp, _vp, _i64, _i64, _i64, _i32, _i32, _vp, _vp, _sz,
                                           _vp], _i32),
    "geot_gather_segment_reduce_ex": ([_vp, _i64, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i32, _i32, _i32, _vp,
                                       _vp, _sz, _cfgp, _vp], _i32),
    "geot_segment_offsets": ([_vp, _i32, _i64, _i64, _vp, _vp], _i32),
    "geot_segment_reduce_backward": ([_vp, _vp, _i64, _i64, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp],
                                     _i32),
    "geot_gather_segment_reduce_backward": ([_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i32, _i32, _vp, _vp, _vp,
                                             _vp, _vp], _i32),
    "geot_validate_index": ([_vp, _i32, _i64, _i64, _vp, _i64, _vp, _vp], _i32),
    "geot_partition": ([_vp, _i32, _i64, _i64, _i32, _vp, _vp, _vp], _i32),
    "geot_partition_exact": ([_vp, _i32, _i64, _i64, _i32, _vp, _vp, _vp, _vp], _i32),
    "geot_split_workspace_size": ([_i64, _i64, _i64, _i32, _i32, _i32, _cfgp], _sz),
    "geot_segment_reduce_split": ([_vp, _vp, _i64, _i64, _i64, _i64, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp,
                                   _vp, _sz, _cfgp, _vp], _i32),
    "geot_selftest_warp_segscan": ([_vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp], _i32),
    "geot_combine_partials": ([_vp, _vp, ctypes.POINTER(ctypes.c_int32), _i32, _i64, _i32, _i32, _vp, _vp], _i32),
}

_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python tools/build.py` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(status: int, where: str) -> None:
    if status != 0:
        if status == 7 and _lib is not None:
            where = f"{where} ({_lib.geot_last_cuda_error().decode()})"
        raise GeotError(status, where)

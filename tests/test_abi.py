"""C-ABI checks that need no GPU: libgeot.so loads, exports every symbol that
include/geot.h declares, and its pure-host entry points (selection, workspace
sizing, argument validation that returns before any CUDA call) behave."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "geot.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(geot_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2404_03019_b200 import _lib
    return _lib.load()


def test_library_exports_every_declared_symbol(L):
    names = header_functions()
    assert len(names) >= 13
    from paper_2404_03019_b200 import _lib
    for n in names:
        assert hasattr(L, n), f"libgeot.so does not export {n}"
        assert n in _lib.SIGNATURES, f"python binding has no signature for {n}"


def test_abi_version_and_status_strings(L):
    assert L.geot_abi_version() == 1
    for s in range(8):
        assert L.geot_status_string(s).startswith(b"GEOT_")


def test_select_config_pure_host(L):
    from paper_2404_03019_b200._lib import GeotConfig
    c = GeotConfig()
    assert L.geot_select_config(1_166_243, 169_343, 128, 0, 0, 0, 0, ctypes.byref(c)) == 0
    assert c.variant >= 1 and c.vec_elems == 4 and c.lanes_per_row == 32 and c.rows_per_group >= 1
    assert L.geot_select_config(10, 5, 3, 0, 0, 0, 0, ctypes.byref(c)) == 0
    assert c.vec_elems == 1 and c.lanes_per_row == 4
    assert L.geot_select_config(10, 5, 0, 0, 0, 0, 0, ctypes.byref(c)) == 1  # F < 1
    assert L.geot_select_config(10, 5, 8, 9, 0, 0, 0, ctypes.byref(c)) == 1  # bad op
    assert L.geot_select_config(10, 5, 8, 0, 0, 0, 0, None) == 1


def test_workspace_size(L):
    assert L.geot_workspace_size(0, 10, 8, 0, 0, 0, 0, None) == 0
    n = L.geot_workspace_size(1_166_243, 169_343, 128, 0, 0, 0, 0, None)
    assert 0 < n < 64 << 20
    assert L.geot_workspace_size(10, 5, 8, 0, 0, 0, 0, None) == 0  # one tile: no carries


def test_argument_errors_return_before_cuda(L):
    # nnz < 0, F < 1, bad enums, S == 0 (no-op): all answered on the host
    p = ctypes.c_void_p(16)
    assert L.geot_segment_reduce(p, p, -1, 4, 8, 0, 0, 0, p, None, 0, None) == 1
    assert L.geot_segment_reduce(p, p, 10, 4, 0, 0, 0, 0, p, None, 0, None) == 1
    assert L.geot_segment_reduce(p, p, 10, 4, 8, 5, 0, 0, p, None, 0, None) == 1
    assert L.geot_segment_reduce(p, p, 10, 0, 8, 0, 0, 0, p, None, 0, None) == 0
    assert L.geot_segment_reduce(None, None, 10, 4, 8, 0, 0, 0, p, None, 0, None) == 1
    assert L.geot_gather_segment_reduce_ex(p, 4, p, p, p, 10, 0, 4, 8, 2, 0, 0, p, None, 0, None, None) == 2
    assert L.geot_partition(p, 0, 10, 4, 0, p, p, None) == 1
    assert L.geot_segment_offsets(p, 0, -1, 4, p, None) == 1
    # too-small workspace is refused on the host
    n = L.geot_workspace_size(1_000_000, 1000, 64, 0, 0, 0, 0, None)
    assert n > 0
    assert L.geot_segment_reduce(ctypes.c_void_p(256), ctypes.c_void_p(256), 1_000_000, 1000, 64, 0, 0, 0,
                                 ctypes.c_void_p(256), ctypes.c_void_p(256), 100, None) == 3


def test_synth_library_loads():
    import synth.device as sd
    lib = sd.lib()
    for n in ("synth_fill_values", "synth_expand_index", "synth_src_index"):
        assert hasattr(lib, n)

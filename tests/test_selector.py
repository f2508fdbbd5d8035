"""Selector (H2) checks on the CPU: the generated if/else (select_tree.inc,
compiled into libgeot) agrees with the exported tree on random features and at
every exact threshold ('<=' goes left), and geot_select_config(_ex)
always returns a configuration the library compiled for the input (any skew
hint, any op)."""
import ctypes
import json
import math
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TREE = os.path.join(ROOT, "tools", "selector_tree.json")


@pytest.fixture(scope="module")
def L():
    from paper_2404_03019_b200 import _lib
    return _lib.load()


def interp(tree, x):
    feats = tree["features"]
    n = 0
    while "leaf" not in tree["nodes"][n]:
        node = tree["nodes"][n]
        n = node["left"] if x[feats.index(node["feature"])] <= node["threshold"] else node["right"]
    return tree["nodes"][n]["leaf"]


def c_tree(L, x):
    out = (ctypes.c_int32 * 4)()
    L.geot_select_tree(*[float(v) for v in x], out)
    return list(out)


@pytest.mark.skipif(not os.path.exists(TREE), reason="no refit tree exported yet")
def test_codegen_matches_tree(L):
    tree = json.load(open(TREE))
    rng = np.random.default_rng(0)
    xs = []
    for _ in range(1000):
        xs.append([rng.uniform(10, 28), rng.uniform(1, 200), float(rng.choice([-1.0, rng.uniform(0, 14)])),
                   float(rng.choice([1, 2, 3, 4, 8, 16, 31, 32, 64, 96, 128, 256, 512, 1024])),
                   float(rng.integers(0, 2)), float(rng.integers(0, 2)), float(rng.integers(0, 3))])
    # exact thresholds and their neighbours
    feats = tree["features"]
    for node in tree["nodes"]:
        if "leaf" in node:
            continue
        for delta in (0.0, -1e-9, 1e-9):
            base = [20.0, 7.0, 5.0, 128.0, 0.0, 0.0, 0.0]
            base[feats.index(node["feature"])] = node["threshold"] + delta
            xs.append(base)
    for x in xs:
        assert c_tree(L, x) == interp(tree, x), x
    assert L.geot_selector_provenance().startswith(b"B200 refit")


# compiled stream pipelines (warps, rows per stage, stages) per vectors per lane (launch.cuh);
# stages 1 = the LDG register pipeline
STREAM_PIPES = {1: {(16, 6, 4), (8, 6, 8), (16, 3, 8), (8, 8, 6), (8, 4, 1), (8, 8, 1)},
                2: {(16, 3, 4), (8, 3, 8), (8, 4, 1)}, 4: {(8, 3, 4), (8, 2, 1)},
                8: {(8, 1, 4), (8, 1, 6), (8, 1, 1)}}
STREAM_PIPES_LPR4 = {(16, 4, 4), (8, 4, 8), (8, 4, 1)}  # 64-byte rows: RS <= 4


def test_select_config_always_valid(L):
    from paper_2404_03019_b200._lib import GeotConfig
    c = GeotConfig()
    for F in (1, 2, 3, 4, 8, 16, 31, 32, 64, 96, 128, 200, 256, 512, 1024, 2048):
        for dt in (0, 1):
            for nnz in (10, 10_000, 1 << 17, 1 << 22, 1 << 26):
                for avg in (1, 3, 7, 16, 100):
                    for fused in (0, 1):
                        S = max(1, nnz // avg)
                        skew = float([0.0, 1.0, 30.0, 3000.0][(nnz + F + avg) % 4])
                        op = (F + avg) % 3
                        assert L.geot_select_config_ex(nnz, S, F, op, dt, 0, fused, skew, ctypes.byref(c)) == 0
                        wide = 4 if dt == 0 else 8
                        if c.variant == 3:  # 16-byte lane vectors, 8/16/32 lanes per row
                            assert c.vec_elems == wide and c.lanes_per_row >= 4
                            lpr = c.lanes_per_row
                            fused_pipes = {(16, min(6, lpr), 4)} | ({(16, 8, 3)} if lpr >= 8 else set()) | \
                                ({(16, 12, 2)} if lpr >= 16 else set())
                            assert not fused or (c.vecs_per_lane == 1 and (c.warps_per_cta, c.rows_per_group, c.stages)
                                                 in fused_pipes)
                            assert F // wide <= c.lanes_per_row * c.vecs_per_lane
                            pipes = STREAM_PIPES_LPR4 if c.lanes_per_row == 4 else set(STREAM_PIPES[c.vecs_per_lane])
                            if c.vecs_per_lane == 1 and lpr >= 16:  # deeper stages for 256/512-byte rows
                                pipes |= {(16, 12, 2), (16, 8, 3)}
                            assert fused or (c.warps_per_cta, c.rows_per_group, c.stages) in pipes
                        elif c.variant == 2:
                            # one lane per row (4..32-byte rows) or lane groups (64 / 128-byte rows)
                            assert not fused and (F in (1, 2, 4, 8, 16, 32) or (dt == 1 and F == 64))
                        else:
                            assert c.variant == 1 and 1 <= c.rows_per_group <= 1024
                            assert c.vec_elems in (1, wide) and F % c.vec_elems == 0
                            assert c.lanes_per_row & (c.lanes_per_row - 1) == 0
                        assert math.isfinite(c.rows_per_group)


def test_select_config_ex_arguments(L):
    from paper_2404_03019_b200._lib import GeotConfig
    c = GeotConfig()
    assert L.geot_select_config_ex(1 << 20, 1 << 16, 64, 0, 0, 0, 0, float("nan"), ctypes.byref(c)) == 1
    assert L.geot_select_config_ex(1 << 20, 1 << 16, 64, 0, 0, 0, 0, -1.0, ctypes.byref(c)) == 0
    d = GeotConfig()
    assert L.geot_select_config(1 << 20, 1 << 16, 64, 0, 0, 0, 0, ctypes.byref(d)) == 0
    assert c.as_dict() == d.as_dict()  # unknown skew == the plain call

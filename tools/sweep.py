"""Configuration sweep on the GPU -> performance database (JSONL).

The B200 analog of the paper's offline benchmarking (PAPER.md P:301-309,
Fig. 5: "we explore a comprehensive range of configurations ... and benchmark
the outcomes offline on GPUs"; key = features + config, value = throughput).

    python tools/sweep.py --out gpurun_out/perfdb.jsonl [--quick] [--grid NAME]

Every record: workload features (E, S, avg, F, dtype, op, fused, dist,
max_len), the config tuple, median/min kernel time (CUDA events over the
launching stream, inputs > L2 or L2 flushed), GB/s (algorithmic bytes) and
e*F/s.  Inputs come from the device generator (synth.device).
"""
from __future__ import annotations

import argparse
import itertools
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_03019_b200 as geot  # noqa: E402
import synth  # noqa: E402
import synth.device as sd  # noqa: E402

L2_BYTES = 126 * 1024 * 1024


def time_call(fn, reps, flush=None, min_ms=0.0):
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    t_total = 0.0
    for i in range(reps):
        if flush is not None:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
        t_total += ts[-1]
        if i >= 4 and t_total > 2000:
            break
    return statistics.median(ts), min(ts)


def make_inputs(E, S, F, dtype, dist, seed, fused=False, V=None, itype=torch.int32):
    if dist == "powerlaw15":  # the heavier-tailed degree distribution (Lomax alpha = 1.5)
        L = synth.segment_lengths(E, S, "powerlaw", seed, alpha=1.5)
    else:
        L = synth.segment_lengths(E, S, dist, seed)
    idx = sd.index_from_lengths(L, itype)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    if fused:
        x = sd.values(V, F, seed, dtype=tdt)
        src = sd.src_index(E, V, seed + 1000, itype=itype)
        return L, idx, x, src
    X = sd.values(E, F, seed, dtype=tdt)
    return L, idx, X, None


# compiled stream pipelines per vectors per lane — launch.cuh
STREAM_PIPES = {1: [(16, 6, 4), (8, 6, 8), (16, 3, 8), (8, 8, 6), (8, 4, 1), (8, 8, 1)],
                2: [(16, 3, 4), (8, 3, 8), (8, 4, 1)], 4: [(8, 3, 4), (8, 2, 1)],
                8: [(8, 1, 4), (8, 1, 6), (8, 1, 1)]}


def stream_lane_shape(F, dtype):
    """(lanes per row, vectors per lane) of the stream kernel for F, or None (select.cpp)."""
    wide = 4 if dtype == "f32" else 8
    if F % wide or F // wide < 4:
        return None
    nv = F // wide
    lpr = 4
    while lpr < nv and lpr < 32:
        lpr *= 2
    v = 1
    while lpr * v < nv:
        v *= 2
    return (lpr, v) if v <= (8 if dtype == "f32" else 4) else None


def candidate_configs(E, S, F, dtype, fused, quick=False):
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    base = geot.geot_select_config(E, S, F, "sum", tdt, torch.int32, fused)
    out = []
    Rs = ([2, 4] if E < 100_000 else []) + ([8, 16, 32, 64] if not quick else [16, 64])
    ctas = [0] if not quick else [0]
    for R, c in itertools.product(Rs, ctas):
        out.append({"variant": 1, "rows_per_group": R, "ctas_per_sm": c})
    # eligibility from the input alone (not from the current selection)
    esz = 4 if dtype == "f32" else 2
    # one lane per row (4..32-byte rows) or lane groups (64 / 128-byte rows): select.cpp narrow_eligible
    narrow_ok = (not fused) and E >= 65536 and (F in (1, 2, 4, 8, 16, 32) or (dtype == "bf16" and F == 64))
    shape = stream_lane_shape(F, dtype)
    stream_ok = E >= 65536 and shape is not None and (not fused or shape[1] == 1)
    if narrow_ok:
        out.append({"variant": 2})
    if stream_ok:
        pipes = [(16, 4, 4), (8, 4, 8), (8, 4, 1)] if shape[0] == 4 else list(STREAM_PIPES[shape[1]])
        if shape in ((16, 1), (32, 1)):  # the deeper-stage 256/512-byte-row pipelines (launch.cuh)
            pipes += [(16, 12, 2), (16, 8, 3)]
        if fused:  # the gather form's compiled pipelines (launch.cuh launch_stream_gather)
            pipes = [(16, min(6, shape[0]), 4)] + ([(16, 8, 3)] if shape[0] >= 8 else []) + \
                ([(16, 12, 2)] if shape[0] >= 16 else [])
        for (w, rs, ns) in pipes:
            if rs <= shape[0]:
                out.append({"variant": 3, "warps_per_cta": w, "rows_per_group": rs, "stages": ns})
    return base, out


def run(args):
    torch.cuda.init()
    dev = torch.device("cuda", 0)
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    f = open(args.out, "a")
    grid = GRIDS[args.grid]
    for (E, S, F, dtype, dist, op, fused) in grid:
        seed = 7
        # fused: x has >= 2^18 rows (a Reddit-sized feature matrix) so a high mean
        # degree does not make x trivially cache-resident (V is not a selector feature)
        V = max(S, 1 << 18) if fused else S
        L, idx, X, src = make_inputs(E, S, F, dtype, dist, seed, fused, V)
        esz = 4 if dtype == "f32" else 2
        B = E * F * esz + E * 4 * (2 if fused else 1) + S * F * esz
        small = B < 4 * L2_BYTES
        out = torch.empty((S, F), dtype=X.dtype, device=dev)
        base, cands = candidate_configs(E, S, F, dtype, fused, args.quick)
        maxlen = int(L.max())
        for cfg in cands:
            if fused:
                fn = lambda: geot.geot_gather_segment_reduce(X, src, idx, S, op, out=out, cfg=cfg)  # noqa: E731
            else:
                fn = lambda: geot.geot_segment_reduce(X, idx, S, op, out=out, cfg=cfg)  # noqa: E731
            try:
                med, mn = time_call(fn, args.reps, flush if small else None)
            except Exception as e:  # unsupported config
                print("skip", cfg, e, file=sys.stderr)
                continue
            rec = {"E": E, "S": S, "avg": E / S, "F": F, "dtype": dtype, "op": op, "fused": int(fused), "dist": dist,
                   "max_len": maxlen, "cfg": {**base.as_dict(), **cfg}, "ms_median": med, "ms_min": mn,
                   "gbs": B / (med * 1e-3) / 1e9, "efs": E * F / (med * 1e-3), "bytes": B, "l2_flushed": small}
            f.write(json.dumps(rec) + "\n")
            f.flush()
            print(f"E={E} S={S} F={F} {dtype} {dist} {op} fused={int(fused)} {cfg} -> {med * 1e3:.1f} us "
                  f"{rec['gbs']:.0f} GB/s", flush=True)
        del X, idx, out, src
        torch.cuda.empty_cache()


ARXIV = (1_166_243, 169_343)


def selector_grid():
    """Training/evaluation workloads of the selector refit (the B200 analog of the
    paper's 51 datasets x augmentation): widths x sizes x mean degree."""
    g = []
    for F in (1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024):
        for logE in (18, 21, 24):
            E = 1 << logE
            if E * F * 4 > (6 << 30):
                continue
            for avg in (3, 16, 64):
                g.append((E, max(1, E // avg), F, "f32", "powerlaw", "sum", False))
    for F in (8, 16, 32, 64, 128, 256):
        for logE in (20, 23):
            g.append((1 << logE, (1 << logE) // 16, F, "bf16", "powerlaw", "sum", False))
    for F in (4, 64, 128):
        g.append((1 << 22, (1 << 22) // 16, F, "f32", "uniform", "sum", False))
    for F in (16, 32, 64, 128):
        for avg in (8, 64, 492):
            g.append((1 << 23, (1 << 23) // avg, F, "f32", "powerlaw", "sum", True))
    for F in (64, 128):
        for avg in (8, 64):
            g.append((1 << 23, (1 << 23) // avg, F, "bf16", "powerlaw", "sum", True))
    for avg in (16, 492):
        g.append((1 << 25, (1 << 25) // avg, 64, "f32", "powerlaw", "sum", True))
    # small graphs (Cora/Citeseer/PubMed-sized) and arxiv-sized ones
    for F in (8, 16, 32, 64, 128):
        for E in (4096, 10_556, 40_000):
            for avg in (3, 8):
                g.append((E, max(1, E // avg), F, "f32", "powerlaw", "sum", False))
    for F in (64, 128, 256):
        for E in (600_000, 1_166_243, 2_500_000):
            for avg in (4, 7, 20):
                g.append((E, E // avg, F, "f32", "powerlaw", "sum", False))
    return g


def selector_grid_large():
    """Large bf16 / fp32 streams (products-shaped and beyond)."""
    g = []
    for F in (64, 128):
        for E in (1 << 24, 1 << 25, 61_859_140):
            g.append((E, E // 25, F, "bf16", "powerlaw", "sum", False))
    for F in (128, 256):
        g.append((1 << 25, (1 << 25) // 25, F, "f32", "powerlaw", "sum", False))
    return g


def selector_grid_fused():
    return [w for w in selector_grid() if w[6]]


# the paper's evaluation datasets (PAPER.md tab:dataset_stats):
# (nodes, edges) — the base set the r2 grid augments
PAPER_DATASETS = {"citeseer": (3_327, 9_104), "cora": (2_708, 10_556), "ppi": (2_245, 61_318),
                  "pubmed": (19_717, 88_648), "amazon_photo": (7_650, 238_162), "flickr": (89_250, 899_756),
                  "arxiv": (169_343, 1_166_243), "collab": (235_868, 1_285_465), "reddit2": (232_965, 23_213_838)}


def selector_grid_r2():
    """Round-2 performance database: the paper's procedure ("51 valid
    datasets ... noising and scaling ... 3060 datasets") on synthetic shapes —
    the Table's nine datasets (plus products- and sweep-sized graphs) SCALED
    (x1, x16: nodes and edges together, mean degree kept) and NOISED (the
    degree distribution: Lomax alpha 2 / alpha 1.5 / uniform), at the feature
    widths of the sweep; bf16, mean/max and the fused form on subsets."""
    g = []
    bases = list(PAPER_DATASETS.values()) + [(2_449_029 // 4, 61_859_140 // 4), (1 << 20, 1 << 24)]
    for (V, E0) in bases:
        for scale in (1, 16):
            E, S = E0 * scale, V * scale
            for dist in ("powerlaw", "powerlaw15", "uniform"):
                for F in (1, 4, 16, 32, 64, 128, 256):
                    if E * F * 4 > (3 << 30) or E * F < 4096:
                        continue
                    g.append((E, S, F, "f32", dist, "sum", False))
    for (V, E0) in (PAPER_DATASETS["flickr"], PAPER_DATASETS["arxiv"], PAPER_DATASETS["reddit2"], (1 << 20, 1 << 24)):
        for F in (1, 8, 16, 32, 64, 128, 256):
            if E0 * F * 2 <= (3 << 30):
                g.append((E0, V, F, "bf16", "powerlaw", "sum", False))
        for op in ("mean", "max"):
            for F in (1, 16, 64, 128):
                if E0 * F * 4 <= (3 << 30):
                    g.append((E0, V, F, "f32", "powerlaw", op, False))
    for (V, E0) in (PAPER_DATASETS["flickr"], PAPER_DATASETS["arxiv"], PAPER_DATASETS["reddit2"]):
        for F in (16, 32, 64, 128):
            for dist in ("powerlaw", "uniform"):
                g.append((E0, V, F, "f32", dist, "sum", True))
    return g


GRIDS = {
    "selector_r2": selector_grid_r2(),
    # the 512-byte-row workloads of the r2 grid again, once the deeper-stage
    # LPR = 32 pipelines were compiled (tools/merge_perfdb.py replaces them)
    "selector_r2_lpr32": [w for w in selector_grid_r2() if stream_lane_shape(w[2], w[3]) == (32, 1)],
    # the widest rows (the sweep's F = 1024; several vectors per lane)
    "selector_r2_wide": [(E, E // avg, F, dt, "powerlaw", "sum", False)
                         for F in (512, 1024) for dt in ("f32", "bf16") for E in (1 << 20, 1 << 22, 1 << 24)
                         for avg in (16, 64) if E * F * (4 if dt == "f32" else 2) <= (68 << 30)],
    "selector": selector_grid(),
    "selector_fused": selector_grid_fused(),
    "selector_large": selector_grid_large(),
    "arxiv": [(ARXIV[0], ARXIV[1], 128, "f32", "powerlaw", "sum", False)],
    "main": [
        (ARXIV[0], ARXIV[1], 128, "f32", "powerlaw", "sum", False),
        (1 << 24, 1 << 20, 1, "f32", "powerlaw", "sum", False),
        (1 << 24, 1 << 20, 4, "f32", "powerlaw", "sum", False),
        (1 << 24, 1 << 20, 16, "f32", "powerlaw", "sum", False),
        (1 << 24, 1 << 20, 64, "f32", "powerlaw", "sum", False),
        (1 << 24, 1 << 20, 64, "f32", "uniform", "sum", False),
        (1 << 24, 1 << 20, 256, "f32", "powerlaw", "sum", False),
        (1 << 22, 1 << 18, 1024, "f32", "powerlaw", "sum", False),
        (61_859_140 // 4, 2_449_029 // 4, 128, "bf16", "powerlaw", "sum", False),
        (10_556, 2_708, 32, "f32", "powerlaw", "sum", False),
        (114_615_892 // 8, 232_965, 64, "f32", "powerlaw", "sum", True),
    ],
}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "perfdb.jsonl"))
    ap.add_argument("--grid", default="arxiv", choices=sorted(GRIDS))
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--quick", action="store_true")
    run(ap.parse_args())

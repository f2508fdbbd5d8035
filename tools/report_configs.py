"""Measure every BASELINE.json configuration with the default (selector)
configuration and write a markdown table + JSONL.

    python tools/report_configs.py --md profiles/r1_configs.md --jsonl gpurun_out/configs.jsonl

Timing: CUDA events on the launching stream around each call, median of
>= 20 reps after 5 warm-ups; inputs < 4x L2 get an L2 flush (write of 252 MB)
before every rep.  Bytes = src rows read + indices + out rows written
(fused: + the second index); the fused form is also reported as effective
logical GB/s (gathered rows counted), as SURVEY §8(d) prescribes.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2404_03019_b200 as geot  # noqa: E402
import synth  # noqa: E402
import synth.device as sd  # noqa: E402

L2 = 126 << 20
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def timed(fn, flush=None, reps=30):
    st = torch.cuda.current_stream()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), min(ts)


def graph_latency(fn, reps=200):
    """Hot latency of one call replayed from a CUDA graph (no L2 flush)."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(10):
        g.replay()
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def run_case(name, F=None, op="sum", dist=None, itype=torch.int32, flush=None, graph=False):
    over = {}
    if F:
        over["F"] = F
    if dist:
        over["dist"] = dist
    w = synth.workload(name, **over)
    E, S, F = w["E"], w["S"], w["F"]
    tdt = torch.float32 if w["dtype"] == "f32" else torch.bfloat16
    esz = 4 if w["dtype"] == "f32" else 2
    isz = 4 if itype == torch.int32 else 8
    L = synth.segment_lengths(E, S, w["dist"], w["seed"])
    idx = sd.index_from_lengths(L, itype)
    out = torch.empty((S, F), dtype=tdt, device="cuda")
    fused = "V" in w
    if fused:
        x = sd.values(w["V"], F, w["seed"], dtype=tdt)
        src = sd.src_index(E, w["V"], w["seed2"], itype=itype)
        fn = lambda: geot.geot_gather_segment_reduce(x, src, idx, S, op, out=out)  # noqa: E731
        B = w["V"] * F * esz + 2 * E * isz + S * F * esz      # HBM-minimum bytes
        B_logical = E * F * esz + 2 * E * isz + S * F * esz   # gathered rows counted
    else:
        X = sd.values(E, F, w["seed"], dtype=tdt)
        fn = lambda: geot.geot_segment_reduce(X, idx, S, op, out=out)  # noqa: E731
        B = B_logical = E * F * esz + E * isz + S * F * esz
    cfg = geot.geot_select_config(E, S, F, op, tdt, itype, fused)
    med, mn = timed(fn, flush if B < 4 * L2 else None)
    rec = {"config": name, "E": E, "S": S, "F": F, "dtype": w["dtype"], "dist": w["dist"], "op": op,
           "index": "int32" if isz == 4 else "int64", "fused": fused, "variant": cfg.variant,
           "us_median": round(med * 1e3, 2), "us_min": round(mn * 1e3, 2), "bytes": B,
           "GBps": round(B / (med * 1e-3) / 1e9, 1), "pct_peak": round(100 * B / (med * 1e-3) / 1e9 / PEAK, 1),
           "eF_per_s": E * F / (med * 1e-3), "l2_flushed": B < 4 * L2}
    if fused:
        rec["GBps_logical"] = round(B_logical / (med * 1e-3) / 1e9, 1)
    if graph:
        rec["us_graph_hot"] = round(graph_latency(fn) * 1e3, 2)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--md", default=os.path.join(ROOT, "profiles", "configs.md"))
    ap.add_argument("--jsonl", default=os.path.join(ROOT, "gpurun_out", "configs.jsonl"))
    a = ap.parse_args()
    flush = torch.empty(2 * L2 // 4, dtype=torch.float32, device="cuda")
    cases = [dict(name="cora", op=o, graph=True) for o in ("sum", "mean", "max")]
    cases += [dict(name="arxiv", op=o) for o in ("sum", "mean", "max")]
    cases += [dict(name="reddit", op="sum")]
    cases += [dict(name="products", op="sum"), dict(name="products", op="max")]
    for F in (1, 4, 16, 64, 256, 1024):
        for dist in ("powerlaw", "uniform"):
            cases.append(dict(name="sweep", F=F, dist=dist, op="sum"))
    cases += [dict(name="sweep", F=1, op="sum", itype=torch.int64), dict(name="sweep", F=4, op="sum",
                                                                       itype=torch.int64)]
    recs = []
    with open(a.jsonl, "w") as jf:
        for c in cases:
            name = c.pop("name")
            r = run_case(name, flush=flush, **c)
            recs.append(r)
            jf.write(json.dumps(r) + "\n")
            print(json.dumps(r), flush=True)
            torch.cuda.empty_cache()
    vname = {1: "edge_tile", 2: "narrow", 3: "stream"}
    with open(a.md, "w") as f:
        f.write(f"# BASELINE configurations on one B200 (default selector; peak = {PEAK} GB/s measured copy)\n\n")
        f.write("| config | E | S | F | dtype | dist | op | index | kernel | µs (median) | GB/s | % peak | e·F/s |\n")
        f.write("|---|---|---|---|---|---|---|---|---|---|---|---|---|\n")
        for r in recs:
            extra = ""
            if r.get("fused"):
                extra = f" (logical {r['GBps_logical']} GB/s)"
            if "us_graph_hot" in r:
                extra += f" (graph-replay hot {r['us_graph_hot']} µs)"
            f.write(f"| {r['config']} | {r['E']:,} | {r['S']:,} | {r['F']} | {r['dtype']} | {r['dist']} | {r['op']} | "
                    f"{r['index']} | {vname.get(r['variant'], '?')} | {r['us_median']}{extra} | {r['GBps']} | "
                    f"{r['pct_peak']} | {r['eF_per_s']:.3g} |\n")
        f.write("\nInputs smaller than 4x L2 are timed with an L2 flush before every call (cold). "
                "Fused (Reddit-shaped): GB/s counts the HBM-minimum bytes (x once + 2 indices + out); "
                "'logical' counts every gathered row.\n")


if __name__ == "__main__":
    main()

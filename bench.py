"""bench.py — GeoT segment-reduction throughput on B200 (the driver's contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload arxiv]

Metric (BASELINE.json): segment_reduce achieved HBM GB/s and % of B200 peak;
edges*F/s at 1/2/4/8 GPUs.  Workload at N=1: configs[1], the ogbn-arxiv-shaped
graph (169,343 segments, 1,166,243 sorted edges, Lomax(2) degree mix,
F=128 fp32, sum).  A step = one geot_segment_reduce call (H1 features + H2
selection on the host, H4-H7 + H5 carries on the device) over the resident
inputs.  Bytes = src rows read + indices + out rows written.
For N>1 (torchrun, one rank per GPU) the global graph is N times larger,
partitioned at segment boundaries by geot_partition (H9) once per graph, and
every rank reduces its own shard with no data-path collective (weak scaling);
value = all ranks' bytes / max-over-ranks time.

--impl reference times the CPU oracle (oracle/, fp64) on the host cores on the
same workload (rank 0 only), as the reference arm for this tier.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "segment_reduce achieved HBM GB/s and % of B200 peak; edges*F/s at 1/2/4/8 GPUs"
UNIT = "GB/s"
FALLBACK_HBM_GBS = 6650.0


# ----------------------------------------------------------------------------- helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def algorithmic_bytes(E, S, F, esz, isz, fused=False):
    """src rows read + indices + out rows written."""
    if fused:
        return E * F * esz + 2 * E * isz + S * F * esz
    return E * F * esz + E * isz + S * F * esz


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


_SAMPLER_SRC = r"""
import json, sys, threading, time
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
period = float(sys.argv[2])
stop = threading.Event()
threading.Thread(target=lambda: (sys.stdin.read(), stop.set()), daemon=True).start()
samples, masks = [], 0
print("ready", flush=True)
while not stop.is_set():
    try:
        samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        masks |= pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
    except Exception:
        pass
    time.sleep(period)
print(json.dumps({"samples": samples, "mask": masks,
                  "max": pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)}), flush=True)
"""


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region, in a
    child process (the launch loop holds the GIL, which starved an in-process thread)."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index, period=float(os.environ.get("GEOT_CLOCK_PERIOD", "0.005"))):
        self.index, self.period = index, period
        self.samples, self.reasons, self.max_mhz, self.err = [], set(), None, ""
        self.proc = None

    def __enter__(self):
        import subprocess
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER_SRC, str(self.index), str(self.period)],
                                         stdin=subprocess.PIPE, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                         text=True)
            if self.proc.stdout.readline().strip() != "ready":
                raise RuntimeError(self.proc.stderr.read()[-300:])
        except Exception as e:  # pragma: no cover
            self.err, self.proc = str(e), None
        return self

    def __exit__(self, *a):
        if not self.proc:
            return
        try:
            out, _ = self.proc.communicate(input="", timeout=30)
            d = json.loads(out.strip().splitlines()[-1])
            self.samples, self.max_mhz = d["samples"], d["max"]
            self.reasons = {name for bit, name in self.REASONS.items() if d["mask"] & bit and bit != 0x1}
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "error": self.err}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def host_workload(w, e_chunk=1 << 17):
    """Host copy of the workload for the oracle (host generator only)."""
    L = synth.segment_lengths(w["E"], w["S"], w["dist"], w["seed"])
    idx = synth.lengths_to_index(L, "i32")
    X = np.empty((w["E"], w["F"]), dtype=np.float32 if w["dtype"] == "f32" else np.uint16)
    for e0 in range(0, w["E"], e_chunk):
        n = min(e_chunk, w["E"] - e0)
        X[e0:e0 + n] = synth.values(w["seed"], e0, n, w["F"], w["dtype"], "real")
    return L, idx, X


def cpu_oracle_time(w, budget_s=10.0, op="sum"):
    """Time the oracle as it stands on the host cores, on the full workload,
    repeated until ~budget_s of CPU work.  Returns (GB/s, cores, sample, per-run s)."""
    import oracle
    L, idx, X = host_workload(w)
    cores = oracle.default_threads()
    B = algorithmic_bytes(w["E"], w["S"], w["F"], 4 if w["dtype"] == "f32" else 2, 4)
    times = []
    t_all = time.perf_counter()
    while not times or (time.perf_counter() - t_all < budget_s and len(times) < 50):
        t0 = time.perf_counter()
        oracle.segment_reduce(X, idx, w["S"], op, nthreads=cores)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return B / t / 1e9, cores, f"full {w['name']}-shaped problem, {len(times)} oracle runs (median)", t


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    w = synth.workload(args.workload)
    import oracle
    L, idx, X = host_workload(w)
    cores = oracle.default_threads()
    B = algorithmic_bytes(w["E"], w["S"], w["F"], 4 if w["dtype"] == "f32" else 2, 4)
    for _ in range(args.warmup):
        oracle.segment_reduce(X, idx, w["S"], "sum", nthreads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.segment_reduce(X, idx, w["S"], "sum", nthreads=cores)
    dt = (time.perf_counter() - t0) / args.steps
    v = B / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(w, 1),
        "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"full {w['name']}-shaped problem per step (fp64 C oracle, {cores} threads)"},
        "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(w, N):
    return {"workload": f"{w['name']}-shaped", "E": w["E"] * N, "S": w["S"] * N, "F": w["F"], "op": "sum",
            "value_dtype": w["dtype"], "index": "int32", "degree_dist": "Lomax(alpha=2) segment lengths",
            "seed": w["seed"], "parallelism": f"{N} segment-range shard(s), no data-path collective",
            "l2": "inputs larger than L2 (no flush needed)"}


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    N = ws
    if N > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if N > 1 else 0)
    torch.cuda.set_device(dev)
    import paper_2404_03019_b200 as geot
    import synth.device as sd
    from paper_2404_03019_b200 import _lib, shard

    w = synth.workload(args.workload)
    Eg, Sg, F = w["E"] * N, w["S"] * N, w["F"]
    tdt = torch.float32 if w["dtype"] == "f32" else torch.bfloat16
    esz = 4 if w["dtype"] == "f32" else 2
    # ---- global index (same on every rank), partition once per graph (H9)
    L = synth.segment_lengths(Eg, Sg, w["dist"], w["seed"])
    bounds = torch.from_numpy(synth.lengths_to_bounds(L)).to(dev)
    if N > 1:
        gidx = sd.expand_index(bounds, 0, Eg, torch.int32)
        sb, eb = [b.cpu().numpy() for b in geot.geot_partition(gidx, Sg, N)]
        e0, e1, s0, s1 = shard.shard_of(sb, eb, rank)
        idx = gidx[e0:e1].clone()
        del gidx
    else:
        e0, e1, s0, s1 = 0, Eg, 0, Sg
        idx = sd.expand_index(bounds, 0, Eg, torch.int32)
    E, S = e1 - e0, s1 - s0
    X = sd.values(E, F, w["seed"], e_begin=e0, dtype=tdt, mode="real", device=dev)
    out = torch.empty((S, F), dtype=tdt, device=dev)
    B_rank = algorithmic_bytes(E, S, F, esz, 4)
    cfg = geot.geot_select_config(E, S, F, "sum", tdt, torch.int32, False)
    user_cfg = json.loads(args.cfg) if args.cfg else None  # experiments only (selector override)
    if user_cfg:
        for k, v in user_cfg.items():
            setattr(cfg, k, int(v))
    stream = torch.cuda.current_stream(dev)

    L_ = _lib.load()
    prof = getattr(L_, "geot_profile_events", None)
    if prof is not None:
        prof.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        prof.restype = None

    def step():
        geot.geot_segment_reduce(X, idx, S, "sum", out=out, seg_base=s0, cfg=user_cfg)

    def barrier():
        if N > 1:
            torch.distributed.barrier()

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    # ---- timed region: exactly K steps
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in kev:  # materialise the underlying cudaEvent_t (torch creates it lazily on first record)
        a.record(stream)
        b.record(stream)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    launches0 = geot.geot_launch_count()
    with ClockSampler(dev.index) as clk:
        t_start.record(stream)
        for i in range(args.steps):
            if prof is not None:
                prof(ctypes.c_void_p(kev[i][0].cuda_event), ctypes.c_void_p(kev[i][1].cuda_event))
            step()
        t_end.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = geot.geot_launch_count() - launches0
    ms = t_start.elapsed_time(t_end) / args.steps
    kern_ms = None
    if prof is not None:
        kern_ms = statistics.mean(a.elapsed_time(b) for a, b in kev)
    t = [ms, kern_ms if kern_ms is not None else ms]
    if N > 1:
        t = shard.max_over_ranks(t)
        B_all, EF_all = shard.sum_over_ranks([B_rank, E * F])
    else:
        B_all, EF_all = float(B_rank), float(E * F)
    ms, kern_ms_max = float(t[0]), float(t[1])
    ag_ms = None
    if N > 1 and args.allgather:  # optional output all-gather (COLL-0), timed separately
        for _ in range(2):
            shard.allgather_rows(out, sb)
        torch.cuda.synchronize()
        barrier()
        ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ga.record(stream)
        for _ in range(5):
            shard.allgather_rows(out, sb)
        gb.record(stream)
        torch.cuda.synchronize()
        ag_ms = shard.max_over_ranks([ga.elapsed_time(gb) / 5])[0]
    value = B_all / (ms * 1e-3) / 1e9
    peak, peak_src = peaks()

    # ---- end-to-end through the public API with host buffers (pinned), N ranks
    k_e2e = max(1, min(args.steps, args.e2e_steps))
    hX = torch.empty((E, F), dtype=tdt, pin_memory=True)
    hX.copy_(X)
    hidx = torch.empty(E, dtype=torch.int32, pin_memory=True)
    hidx.copy_(idx)
    hout = torch.empty((S, F), dtype=tdt, pin_memory=True)
    dX, didx = torch.empty_like(X), torch.empty_like(idx)

    def e2e_step():
        dX.copy_(hX, non_blocking=True)
        didx.copy_(hidx, non_blocking=True)
        geot.geot_segment_reduce(dX, didx, S, "sum", out=out, seg_base=s0)
        hout.copy_(out, non_blocking=True)

    e2e_step()
    torch.cuda.synchronize()
    barrier()
    ea, eb_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    for _ in range(k_e2e):
        e2e_step()
    eb_.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([ea.elapsed_time(eb_) / k_e2e], dtype=torch.float64, device=dev)
    if N > 1:
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
    e2e_ms = float(te[0])
    h2d = E * F * esz + E * 4
    d2h = S * F * esz
    del hX, dX, didx

    if rank != 0:
        if N > 1:
            torch.distributed.destroy_process_group()
        return 0

    kern_bytes = B_rank  # per launch of the dominant kernel on rank 0's shard
    achieved = kern_bytes / (kern_ms_max * 1e-3) / 1e9 if kern_ms is not None else value / N
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(f"{w['name']}:{N}") or json.load(open(tp)).get(w["name"])
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": N, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": w["dtype"], "data": "synthetic",
        "config": workload_config(w, N),
        "pct_of_peak": round(100 * value / (N * peak), 2), "edges_F_per_s": EF_all / (ms * 1e-3),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                     "kernel": {1: "edge_tile_kernel (+ carry_fixup_kernel)", 2: "narrow_kernel",
                                3: "stream_kernel"}.get(cfg.variant, "?"),
                     "kernel_ms": round(kern_ms_max, 5) if kern_ms is not None else None,
                     "algorithmic_bytes_per_launch": kern_bytes},
        "e2e": {"value": round(B_all / (e2e_ms * 1e-3) / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": k_e2e, "ms_per_step": round(e2e_ms, 4)},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "selected_config": cfg.as_dict(),
        "allgather_ms": ag_ms,
    }
    if N == 1 and not args.no_cpu_baseline:
        v, cores, sample, _ = cpu_oracle_time(w, budget_s=args.cpu_budget)
        line["cpu_baseline"] = {"value": round(v, 3), "unit": UNIT, "cores": cores, "kind": "oracle",
                                "sample": sample}
    print(json.dumps(line), flush=True)
    if N > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="arxiv", choices=sorted(synth.WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-budget", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cfg", default="", help="JSON geot_config override (experiments; default = the selector)")
    ap.add_argument("--allgather", action="store_true", help="N>1: also time the optional output all-gather")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

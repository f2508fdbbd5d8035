"""bench.py — GeoT segment-reduction throughput on B200 (the driver's contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--workload products|arxiv|reddit|sweep|cora] [--F F] [--dist D] [--op OP] [--weighted]

Metric (BASELINE.json): segment_reduce achieved HBM GB/s and % of B200 peak;
edges*F/s at 1/2/4/8 GPUs.  Default workload: BASELINE.json configs[3], the
ogbn-products-shaped graph (2,449,029 segments, 61,859,140 sorted edges,
Lomax(2) degree mix, F=128, bf16 values, sum) — the configuration the metric's
"at 1/2/4/8 GPUs" names and the largest single-GPU segment_reduce config.
A step = one geot_segment_reduce call (H1 features + H2 selection on the host,
H4-H7 + H5 carries on the device) over inputs resident in HBM.
Bytes = src rows read + indices + out rows written.

N > 1 (torchrun, one rank per GPU): STRONG scaling of the same global graph.
Every rank builds the global index, runs geot_partition (H9, once per graph)
and reduces only its own shard [e_p, e_{p+1}) -> rows [s_p, s_{p+1}) with
seg_base = s_p; no data-path collective (NCCL carries the barrier and the
max-over-ranks time only).  value = global bytes / max-over-ranks time.

--impl reference times the CPU oracle (oracle/, fp64) on the host cores, rank
0 only, on a bounded sample (the leading segments) of the same workload.
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


def algorithmic_bytes(E, S, F, esz, isz, fused=False, weighted=False):
    """src rows read + indices + out rows written (fused: the
    logical gathered rows, both indices, and the weights when weighted)."""
    if fused:
        return E * F * esz + 2 * E * isz + S * F * esz + (4 * E if weighted else 0)
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


def l2_gather_peak():
    """Measured ceiling of L2-resident random 256-byte row gathers (tools/microbench/
    l2_gather.cu, written by tools/l2_gather_peak.py into profiles/)."""
    p = os.path.join(ROOT, "profiles", "l2_gather_peak.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            return float(d["gbs"]), f"measured (profiles/l2_gather_peak.json, {d.get('how', '')})"
        except Exception:
            pass
    return None, None


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

    def __init__(self, index, period=float(os.environ.get("GEOT_CLOCK_PERIOD", "0.002"))):
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


def make_workload(args):
    over = {}
    if args.F:
        over["F"] = args.F
    if args.dist:
        over["dist"] = args.dist
    w = synth.workload(args.workload, **over)
    w["op"] = args.op
    w["fused"] = "V" in w
    w["weighted"] = bool(args.weighted) and w["fused"]
    if w["weighted"] and args.op != "sum":
        raise SystemExit("--weighted is the sum-only SpMM form (P:330)")
    return w


def mode_of(op):
    return "signed" if op == "max" else "real"


def workload_config(w, N, e_rank_max=None):
    c = {"workload": f"{w['name']}-shaped", "E": w["E"], "S": w["S"], "F": w["F"], "op": w["op"],
         "value_dtype": w["dtype"], "index": "int32",
         "degree_dist": f"{'Lomax(alpha=2)' if w['dist'] == 'powerlaw' else 'uniform'} segment lengths",
         "seed": w["seed"],
         "parallelism": (f"{N} segment-range shards of one graph (geot_partition), no data-path collective"
                         if N > 1 else "1 GPU"),
         "l2": "inputs larger than L2 (no flush needed)"}
    if w["fused"]:
        c["form"] = "fused gather (index_weight_segment_reduce)" if w["weighted"] else \
            "fused gather (index_segment_reduce)"
        c["V"] = w["V"]
        c["l2"] = "x (the gathered rows) is L2-resident by design; index streams larger than L2 (no flush)"
    if e_rank_max is not None:
        c["edges_per_rank_max"] = int(e_rank_max)
    return c


def leading_sample(L, max_edges):
    """The leading segments of the graph holding at most max_edges edges (>= 1 segment)."""
    b = synth.lengths_to_bounds(L)
    k = int(np.searchsorted(b, max_edges, side="right") - 1)
    k = max(1, min(k, L.shape[0]))
    return k, int(b[k])


def host_sample(w, max_edges, e_chunk=1 << 17):
    """Host copy of the leading segments of the workload (host generator only)."""
    L = synth.segment_lengths(w["E"], w["S"], w["dist"], w["seed"])
    k, Es = leading_sample(L, max_edges)
    idx = synth.lengths_to_index(L[:k], "i32")
    mode = mode_of(w["op"])
    if w["fused"]:
        x = np.empty((w["V"], w["F"]), dtype=np.float32 if w["dtype"] == "f32" else np.uint16)
        for r0 in range(0, w["V"], e_chunk):
            n = min(e_chunk, w["V"] - r0)
            x[r0:r0 + n] = synth.values(w["seed"], r0, n, w["F"], w["dtype"], mode)
        src = synth.src_index(w["seed2"], 0, Es, w["V"]).astype(np.int32)
        wt = synth.weights(w["seed3"], 0, Es) if w["weighted"] else None
        return k, Es, idx, (x, src, wt)
    X = np.empty((Es, w["F"]), dtype=np.float32 if w["dtype"] == "f32" else np.uint16)
    for e0 in range(0, Es, e_chunk):
        n = min(e_chunk, Es - e0)
        X[e0:e0 + n] = synth.values(w["seed"], e0, n, w["F"], w["dtype"], mode)
    return k, Es, idx, X


def run_oracle(w, k, idx, data, cores):
    import oracle
    if w["fused"]:
        x, src, wt = data
        return oracle.gather_segment_reduce(x, src, idx, k, w["op"], weight=wt, nthreads=cores)
    return oracle.segment_reduce(data, idx, k, w["op"], nthreads=cores)


def sample_bytes(w, k, Es):
    esz = 4 if w["dtype"] == "f32" else 2
    return algorithmic_bytes(Es, k, w["F"], esz, 4, w["fused"], w["weighted"])


def cpu_oracle_time(w, k, Es, idx, data, budget_s):
    """The oracle as it stands, on the host cores, on a sample (the leading k
    segments, Es edges), repeated until ~budget_s of CPU work."""
    import oracle
    cores = oracle.default_threads()
    B = sample_bytes(w, k, Es)
    times = []
    t_all = time.perf_counter()
    while not times or (time.perf_counter() - t_all < budget_s and len(times) < 50):
        t0 = time.perf_counter()
        run_oracle(w, k, idx, data, cores)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    sample = (f"leading {k:,} segments / {Es:,} edges ({B / 1e9:.2f} GB algorithmic) of the {w['name']}-shaped "
              f"workload, fp64 C oracle on {cores} threads, median of {len(times)} runs")
    return B / t / 1e9, cores, sample


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    w = make_workload(args)
    import oracle
    cores = oracle.default_threads()
    k, Es, idx, data = host_sample(w, args.ref_sample_edges)
    B = sample_bytes(w, k, Es)
    for _ in range(args.warmup):
        run_oracle(w, k, idx, data, cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run_oracle(w, k, idx, data, cores)
    dt = (time.perf_counter() - t0) / args.steps
    v = B / dt / 1e9
    sample = (f"leading {k:,} segments / {Es:,} edges ({B / 1e9:.3f} GB algorithmic) of the {w['name']}-shaped "
              f"workload per step (fp64 C oracle, {cores} threads)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(w, 1),
        "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    N = ws
    # GEOT_BENCH_SHARED_GPU=1: every rank on cuda:0 with a gloo process group — a
    # functional check of the N > 1 path on a one-GPU box (its timings mean nothing)
    shared = os.environ.get("GEOT_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    if N > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if N > 1 else 0)
    torch.cuda.set_device(dev)
    import paper_2404_03019_b200 as geot
    import synth.device as sd
    from paper_2404_03019_b200 import _lib, shard

    w = make_workload(args)
    Eg, Sg, F, op = w["E"], w["S"], w["F"], w["op"]
    tdt = torch.float32 if w["dtype"] == "f32" else torch.bfloat16
    esz = 4 if w["dtype"] == "f32" else 2
    mode = mode_of(op)
    # ---- global index (identical on every rank); partition once per graph (H9)
    L = synth.segment_lengths(Eg, Sg, w["dist"], w["seed"])
    bounds = torch.from_numpy(synth.lengths_to_bounds(L)).to(dev)
    gidx = sd.expand_index(bounds, 0, Eg, torch.int32)
    sb_t, eb_t = geot.geot_partition(gidx, Sg, N)
    sb, eb = sb_t.cpu().numpy(), eb_t.cpu().numpy()
    e0, e1, s0, s1 = shard.shard_of(sb, eb, rank)
    E, S = e1 - e0, s1 - s0
    idx = gidx[e0:e1].clone() if N > 1 else gidx
    del gidx
    if w["fused"]:  # x replicated on every rank; src (and weights) sliced like dst
        V = w["V"]
        x = sd.values(V, F, w["seed"], dtype=tdt, mode=mode, device=dev)
        src = sd.src_index(E, V, w["seed2"], e_begin=e0, device=dev)
        wt = sd.values(E, 1, w["seed3"], e_begin=e0, dtype=torch.float32, device=dev)[:, 0].contiguous() \
            if w["weighted"] else None
    else:
        X = sd.values(E, F, w["seed"], e_begin=e0, dtype=tdt, mode=mode, device=dev)
    out = torch.empty((S, F), dtype=tdt, device=dev)
    B_rank = algorithmic_bytes(E, S, F, esz, 4, w["fused"], w["weighted"])
    cfg = geot.geot_select_config(E, S, F, op, tdt, torch.int32, w["fused"])
    user_cfg = json.loads(args.cfg) if args.cfg else None  # experiments only (selector override)
    if user_cfg:
        for k_, v_ in user_cfg.items():
            setattr(cfg, k_, int(v_))
    stream = torch.cuda.current_stream(dev)

    L_ = _lib.load()
    prof = getattr(L_, "geot_profile_events", None)

    if w["fused"]:
        def call(xx, ss, ii, ww):
            geot.geot_gather_segment_reduce(xx, ss, ii, S, op, weight=ww, out=out, seg_base=s0, cfg=user_cfg)

        def step():
            call(x, src, idx, wt)
    else:
        def call(xx, ii):
            geot.geot_segment_reduce(xx, ii, S, op, out=out, seg_base=s0, cfg=user_cfg)

        def step():
            call(X, idx)

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
    torch.cuda.synchronize()
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
    kern_ms = statistics.mean(a.elapsed_time(b) for a, b in kev) if prof is not None else None
    t = [ms, kern_ms if kern_ms is not None else ms]
    if N > 1:
        t = shard.max_over_ranks(t)
        B_all, EF_all, E_max = shard.sum_over_ranks([B_rank, E * F, 0])[0], float(Eg * F), \
            shard.max_over_ranks([E])[0]
    else:
        B_all, EF_all, E_max = float(B_rank), float(E * F), E
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

    # ---- end-to-end through the public API with host buffers (pinned), N ranks:
    # every step copies its inputs host->device, reduces, and reads the result back
    k_e2e = max(1, min(args.steps, args.e2e_steps))

    def pinned_like(t_):
        try:
            h = torch.empty(t_.shape, dtype=t_.dtype, pin_memory=True)
        except RuntimeError:  # pinning refused (host memory limits): pageable staging
            h = torch.empty(t_.shape, dtype=t_.dtype)
        h.copy_(t_)
        return h

    if w["fused"]:
        h_in = [pinned_like(x), pinned_like(src), pinned_like(idx)] + ([pinned_like(wt)] if w["weighted"] else [])
    else:
        h_in = [pinned_like(X), pinned_like(idx)]
    d_in = [torch.empty_like(h, device=dev) for h in h_in]
    hout = torch.empty((S, F), dtype=tdt, pin_memory=True)

    def e2e_step():
        for h, d in zip(h_in, d_in):
            d.copy_(h, non_blocking=True)
        if w["fused"]:
            call(d_in[0], d_in[1], d_in[2], d_in[3] if w["weighted"] else None)
        else:
            call(d_in[0], d_in[1])
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
    e2e_ms = ea.elapsed_time(eb_) / k_e2e
    if N > 1:
        e2e_ms = shard.max_over_ranks([e2e_ms])[0]
    h2d = sum(h.numel() * h.element_size() for h in h_in)
    d2h = S * F * esz
    del h_in, d_in

    if rank != 0:
        if N > 1:
            torch.distributed.destroy_process_group()
        return 0

    kern_bytes = B_rank  # per launch of the dominant kernel on rank 0's shard
    achieved = kern_bytes / (kern_ms_max * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    tkey = f"{w['name']}:F{F}:{w['dtype']}:{op}:{w['dist']}" + (":w" if w["weighted"] else "")
    if os.path.exists(tp):
        try:
            d = json.load(open(tp))
            traffic = d.get(f"{tkey}:N{N}") or (d.get(tkey) if N == 1 else None)
        except Exception:
            traffic = None
    kname = {1: "edge_tile_kernel (+ carry_fixup_kernel)", 2: "narrow_kernel", 3: "stream_kernel"}.get(cfg.variant, "?")
    if w["fused"]:
        hbm_min = V * F * esz + (2 * E) * 4 + S * F * esz + (4 * E if w["weighted"] else 0)
        l2p, l2src = l2_gather_peak()
        roof = {"bound": "l2_gather", "achieved": round(achieved, 1), "peak": l2p, "unit": "GB/s",
                "frac": round(achieved / l2p, 4) if l2p else None, "traffic": traffic, "peak_source": l2src,
                "hbm_min_bytes_per_launch": hbm_min,
                "hbm_min_frac": round(hbm_min / (kern_ms_max * 1e-3) / 1e9 / peak, 4)}
    else:
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src}
    roof.update({"kernel": kname, "kernel_ms": round(kern_ms_max, 5), "algorithmic_bytes_per_launch": kern_bytes})
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": N, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": w["dtype"], "data": "synthetic",
        "config": workload_config(w, N, E_max if N > 1 else None),
        "pct_of_peak": round(100 * value / (N * peak), 2), "edges_F_per_s": EF_all / (ms * 1e-3),
        "roofline": roof,
        "e2e": {"value": round(B_all / (e2e_ms * 1e-3) / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": k_e2e, "ms_per_step": round(e2e_ms, 4)},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "selected_config": cfg.as_dict(),
        "allgather_ms": ag_ms,
    }
    if N == 1 and not args.no_cpu_baseline:
        # bounded sample: the leading segments, copied from the device-resident inputs
        k, Es = leading_sample(L, args.cpu_sample_edges)
        hidx = idx[:Es].cpu().numpy()
        if w["fused"]:
            data = (_host_vals(x), src[:Es].cpu().numpy(), wt[:Es].cpu().numpy() if w["weighted"] else None)
        else:
            data = _host_vals(X[:Es])
        v, cores, sample = cpu_oracle_time(w, k, Es, hidx, data, args.cpu_budget)
        line["cpu_baseline"] = {"value": round(v, 3), "unit": UNIT, "cores": cores, "kind": "oracle",
                                "sample": sample}
    print(json.dumps(line), flush=True)
    if N > 1:
        torch.distributed.destroy_process_group()
    return 0


def _host_vals(t):
    import torch
    t = t.cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="products", choices=sorted(synth.WORKLOADS))
    ap.add_argument("--F", type=int, default=0, help="feature width override (the width/skew sweep)")
    ap.add_argument("--dist", default="", choices=["", "powerlaw", "uniform"], help="segment-length distribution")
    ap.add_argument("--op", default="sum", choices=["sum", "mean", "max"])
    ap.add_argument("--weighted", action="store_true", help="fused workloads: index_weight_segment_reduce (P:330)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--cpu-sample-edges", type=int, default=4_000_000)
    ap.add_argument("--ref-sample-edges", type=int, default=1_000_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cfg", default="", help="JSON geot_config override (experiments; default = the selector)")
    ap.add_argument("--allgather", action="store_true", help="N>1: also time the optional output all-gather")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

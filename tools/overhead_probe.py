"""Where does a step's time go beyond the kernel?  For one workload: host time
per call (no sync), event-timed steps with and without the kernel-bracketing
profile events, a CUDA-graph replay of the same call, and the kernel alone.
python tools/overhead_probe.py [workload] [F]"""
import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_03019_b200 as geot  # noqa: E402
import synth  # noqa: E402
import synth.device as sd  # noqa: E402
from paper_2404_03019_b200 import _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "arxiv"
over = {"F": int(sys.argv[2])} if len(sys.argv) > 2 else {}
w = synth.workload(name, **over)
tdt = torch.float32 if w["dtype"] == "f32" else torch.bfloat16
L = synth.segment_lengths(w["E"], w["S"], w["dist"], w["seed"])
idx = sd.index_from_lengths(L)
X = sd.values(w["E"], w["F"], w["seed"], dtype=tdt)
out = torch.empty((w["S"], w["F"]), dtype=tdt, device="cuda")
S = w["S"]
N = 200


def call():
    geot.geot_segment_reduce(X, idx, S, "sum", out=out)


for _ in range(20):
    call()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(N):
    call()
t_host = (time.perf_counter() - t0) / N
torch.cuda.synchronize()
st = torch.cuda.current_stream()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(N):
    call()
b.record(st)
torch.cuda.synchronize()
t_ev = a.elapsed_time(b) / N
prof = _lib.load().geot_profile_events
kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
for x, y in kev:
    x.record(st)
    y.record(st)
torch.cuda.synchronize()
a.record(st)
for i in range(N):
    prof(ctypes.c_void_p(kev[i][0].cuda_event), ctypes.c_void_p(kev[i][1].cuda_event))
    call()
b.record(st)
torch.cuda.synchronize()
t_ev_prof = a.elapsed_time(b) / N
t_kern = statistics.mean(x.elapsed_time(y) for x, y in kev)
# CUDA graph of one call, replayed
g = torch.cuda.CUDAGraph()
s2 = torch.cuda.Stream()
s2.wait_stream(st)
with torch.cuda.stream(s2):
    call()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s2):
        call()
torch.cuda.synchronize()
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
a.record(st)
for _ in range(N):
    g.replay()
b.record(st)
torch.cuda.synchronize()
t_graph = a.elapsed_time(b) / N
B = w["E"] * w["F"] * (4 if w["dtype"] == "f32" else 2) + w["E"] * 4 + S * w["F"] * (4 if w["dtype"] == "f32" else 2)
print(f"{name} F={w['F']}: host {t_host * 1e6:.1f} us/call | events {t_ev * 1e3:.1f} us/step | events+prof "
      f"{t_ev_prof * 1e3:.1f} us/step, kernel {t_kern * 1e3:.1f} us | graph replay {t_graph * 1e3:.1f} us/step | "
      f"GB/s: step {B / t_ev / 1e6:.0f}, kernel {B / t_kern / 1e6:.0f}, graph {B / t_graph / 1e6:.0f}")

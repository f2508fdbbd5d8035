"""Per-CTA / per-agent timeline of one stream-kernel launch, from a -DGEOT_TRACE build:
    python tools/build_variant.py v_trace inst_stream.cu -DGEOT_TRACE
    GEOT_LIB_OVERRIDE=scratch/v_trace/libgeot.so python tools/trace_stream.py arxiv   (or products)
Prints CTA start/end, the spread of agent loop ends, per-SM / per-warp-index / per-position means."""
import ctypes, json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_03019_b200 as geot
from paper_2404_03019_b200 import _lib
import synth
wl = sys.argv[1] if len(sys.argv) > 1 else "arxiv"
w = synth.WORKLOADS[wl]
E, S, F = w["E"], w["S"], w["F"]
L = synth.segment_lengths(E, S, "powerlaw", 2)
idx = torch.from_numpy(synth.lengths_to_index(L, "i32")).cuda()
dt = torch.bfloat16 if w.get("dtype", "f32") == "bf16" else torch.float32
X = torch.randn(E, F, device="cuda").to(dt)
for _ in range(5):
    y = geot.geot_segment_reduce(X, idx, S, "sum")
torch.cuda.synchronize()
fl = torch.empty(256 << 20, device="cuda")
res = []
for rep in range(3):
    fl.add_(1.0)
    torch.cuda.synchronize()
    y = geot.geot_segment_reduce(X, idx, S, "sum")
    torch.cuda.synchronize()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    cta = (ctypes.c_ulonglong * (4096 * 4))()
    ag = (ctypes.c_ulonglong * 65536)()
    assert lib.geot_debug_trace(cta, 4096 * 4, ag, 65536) == 0
    c = np.array(cta, dtype=np.int64).reshape(-1, 4)
    n = int((c[:, 0] > 0).sum())
    c = c[:n]
    t0 = c[:, 0].min()
    st, en, sm = (c[:, 0] - t0) / 1e3, (c[:, 1] - t0) / 1e3, c[:, 2]
    a = np.array(ag, dtype=np.int64)
    a = a[a > 0]
    aw = (a - t0) / 1e3
    print(f"rep {rep}: ctas {n} start us min/med/max {st.min():.1f}/{np.median(st):.1f}/{st.max():.1f}  end {en.min():.1f}/{np.median(en):.1f}/{en.max():.1f}")
    print(f"   agent loop end us min/p10/med/p90/max {np.percentile(aw,[0,10,50,90,100]).round(1).tolist()}")
    order = np.argsort(en)
    print("   slowest CTAs (ticket, sm, start, end):", [(int(i), int(sm[i]), round(st[i],1), round(en[i],1)) for i in order[-6:]])
    print("   fastest CTAs:", [(int(i), int(sm[i]), round(st[i],1), round(en[i],1)) for i in order[:6]])
    # per-SM end time grouped by smid//2 (TPC) and smid range
    ends = {int(sm[i]): float(en[i]) for i in range(n)}
    arr = np.array([ends.get(k, np.nan) for k in range(max(ends) + 1)])
    print("   end by smid (blocks of 16):", [round(float(np.nanmean(arr[i:i+16])), 1) for i in range(0, len(arr), 16)])
    G = 1 if F * X.element_size() >= 512 else 512 // (F * X.element_size())
    ag_all = np.array(ag, dtype=np.int64)
    na = int((ag_all > 0).sum())
    ae = (ag_all[:na] - t0) / 1e3
    warp = (np.arange(na) // G) % 16
    print("   agent end by warp index:", [round(float(ae[warp == w].mean()), 1) for w in range(16)])
    tick = np.arange(na) // (16 * G)
    print("   agent end std within CTA (mean over CTAs):", round(float(np.mean([ae[tick == t].std() for t in range(n)])), 1),
          " std of CTA means:", round(float(np.std([ae[tick == t].mean() for t in range(n)])), 1))
    print("   agent end vs position (deciles of agent id):", [round(float(x.mean()), 1) for x in np.array_split(ae, 10)])

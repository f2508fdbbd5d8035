"""Time one workload under several configurations (kernel-design experiments):
python tools/time_cfgs.py E S F dtype dist [fused] -- 'json-cfg' ['json-cfg' ...]   ('' = selector default)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_03019_b200 as geot  # noqa: E402
from tools.sweep import make_inputs, time_call  # noqa: E402

sep = sys.argv.index("--")
head, cfgs = sys.argv[1:sep], sys.argv[sep + 1:]
E, S, F, dt, dist = int(head[0]), int(head[1]), int(head[2]), head[3], head[4]
fused = len(head) > 5 and head[5] == "fused"
inp = make_inputs(E, S, F, dt, dist, 5, fused=fused, V=S if fused else None)
esz = 4 if dt == "f32" else 2
B = E * F * esz + E * 4 * (2 if fused else 1) + S * F * esz
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for c in cfgs:
    cfg = json.loads(c) if c else None
    try:
        if fused:
            L, idx, x, src = inp
            fn = lambda: geot.geot_gather_segment_reduce(x, src, idx, S, "sum", cfg=cfg)  # noqa: E731
        else:
            L, idx, X, _ = inp
            fn = lambda: geot.geot_segment_reduce(X, idx, S, "sum", cfg=cfg)  # noqa: E731
        med, mn = time_call(fn, 30, flush if B < 4 * (126 << 20) else None)
        print(json.dumps({"E": E, "F": F, "dtype": dt, "dist": dist, "fused": fused, "cfg": c, "us": round(med * 1e3, 1),
                          "GBps": round(B / (med * 1e-3) / 1e9)}), flush=True)
    except Exception as ex:  # noqa: BLE001
        print(json.dumps({"cfg": c, "error": str(ex)[:200]}), flush=True)

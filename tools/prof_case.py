"""Run one configuration a few times (for ncu):
python tools/prof_case.py E S F dtype dist [cfg-json|-] [fused|weighted|-] [op] [mode]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_03019_b200 as geot  # noqa: E402
import synth  # noqa: E402
import synth.device as sd  # noqa: E402

E, S, F = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dt, dist = sys.argv[4], sys.argv[5]
cfg = json.loads(sys.argv[6]) if len(sys.argv) > 6 and sys.argv[6] not in ("", "-") else None
fused = len(sys.argv) > 7 and sys.argv[7] in ("fused", "weighted")
weighted = len(sys.argv) > 7 and sys.argv[7] == "weighted"
op = sys.argv[8] if len(sys.argv) > 8 else "sum"
mode = sys.argv[9] if len(sys.argv) > 9 else ("signed" if op == "max" else "real")
tdt = torch.float32 if dt == "f32" else torch.bfloat16
L = synth.segment_lengths(E, S, dist, 5)
idx = sd.index_from_lengths(L)
if fused:
    x = sd.values(S, F, 5, dtype=tdt, mode=mode)
    src = sd.src_index(E, S, 1005)
    w = sd.values(E, 1, 7, dtype=torch.float32)[:, 0].contiguous() if weighted else None
    run = lambda: geot.geot_gather_segment_reduce(x, src, idx, S, op, weight=w, cfg=cfg)  # noqa: E731
else:
    X = sd.values(E, F, 5, dtype=tdt, mode=mode)
    run = lambda: geot.geot_segment_reduce(X, idx, S, op, cfg=cfg)  # noqa: E731
for _ in range(6):
    run()
torch.cuda.synchronize()
print("ok")

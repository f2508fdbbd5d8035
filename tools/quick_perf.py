"""Quick timing of the default configuration on a few workloads (tooling)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_03019_b200 as geot  # noqa: E402
import synth  # noqa: E402
import synth.device as sd  # noqa: E402
from tools.sweep import time_call  # noqa: E402

CASES = [(1 << 24, 1 << 20, F, "f32", d) for F in (1, 2, 4, 8, 16, 32, 64) for d in ("powerlaw", "uniform")]
CASES += [(1 << 24, 1 << 20, F, "bf16", "powerlaw") for F in (1, 4, 16)]
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for (E, S, F, dt, dist) in CASES:
    L = synth.segment_lengths(E, S, dist, 5)
    idx = sd.index_from_lengths(L)
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    X = sd.values(E, F, 5, dtype=tdt)
    out = torch.empty((S, F), dtype=tdt, device="cuda")
    esz = 4 if dt == "f32" else 2
    B = E * F * esz + E * 4 + S * F * esz
    c = geot.geot_select_config(E, S, F, "sum", tdt)
    med, mn = time_call(lambda: geot.geot_segment_reduce(X, idx, S, "sum", out=out), 20,
                        flush if B < 4 * (126 << 20) else None)
    print(json.dumps({"E": E, "F": F, "dtype": dt, "dist": dist, "variant": c.variant, "us": round(med * 1e3, 1),
                      "GBps": round(B / (med * 1e-3) / 1e9)}), flush=True)

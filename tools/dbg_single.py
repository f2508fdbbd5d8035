import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch, numpy as np
import paper_2404_03019_b200 as geot
from parity_helpers import make_case, to_torch_vals
L, idx, X = make_case(100_000, 9_000, 128, "f32", "int", "single", 2)
xt, it = to_torch_vals(X), torch.from_numpy(idx).to(torch.int32).cuda()
for op in ("sum", "mean", "max"):
    for rs in (3, 0):
        try:
            y = geot.geot_segment_reduce(xt, it, 9000, op, cfg={"variant": 3, "rows_per_group": rs})
            torch.cuda.synchronize()
            print(op, rs, "ok", float(y.sum()))
        except Exception as e:
            print(op, rs, "ERR", e)
            raise

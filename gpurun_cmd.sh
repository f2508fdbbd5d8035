timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "bf16 or max or stream or products" 2>&1 | tail -2
for op in sum max; do timeout 120 python - <<PY
import sys; sys.path.insert(0,'.')
import torch, json
import paper_2404_03019_b200 as geot
from tools.sweep import make_inputs, time_call
L, idx, X, _ = make_inputs(61859140, 2449029, 128, "bf16", "powerlaw", 5)
if "$op" == "max":
    import synth.device as sd
    X = sd.values(61859140, 128, 5, dtype=torch.bfloat16, mode="signed")
med, mn = time_call(lambda: geot.geot_segment_reduce(X, idx, 2449029, "$op"), 20)
B = 61859140*128*2 + 61859140*4 + 2449029*128*2
print("products $op", round(med*1e3,1), "us", round(B/(med*1e-3)/1e9), "GB/s")
PY
done

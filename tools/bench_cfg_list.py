"""Run bench.py under a list of configurations (selector experiments):
python tools/bench_cfg_list.py WORKLOAD 'json-cfg' ['json-cfg' ...]   ('' = default)"""
import json
import subprocess
import sys

w = sys.argv[1]
for c in sys.argv[2:]:
    r = subprocess.run([sys.executable, "bench.py", "--workload", w, "--steps", "200", "--warmup", "20",
                        "--no-cpu-baseline", "--e2e-steps", "1", "--cfg", c], capture_output=True, text=True)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        print(w, c or "default", d["value"], d["roofline"]["kernel_ms"], d["roofline"]["frac"], flush=True)
    except Exception:
        print(w, c, "FAILED", r.stderr[-400:], flush=True)

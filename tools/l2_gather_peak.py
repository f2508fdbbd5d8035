"""Build and run tools/microbench/l2_gather.cu on the GPU box and record the
measured ceiling of L2-resident random 256-byte row gathers in
profiles/l2_gather_peak.json (repo-written; the roofline bench.py reports the
fused Reddit-shaped path against)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(ROOT, "tools", "microbench", "l2_gather.cu")
exe = os.path.join(ROOT, "tools", "microbench", "l2_gather")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe, src])
out = subprocess.run([exe] + sys.argv[1:], capture_output=True, text=True, check=True).stdout
rows = [json.loads(line) for line in out.splitlines() if line.startswith("{")]
print(out)
best = rows[-1]
res = {"gbs": best["gbs"], "variant": best["best"], "V": best["V"], "N": best["N"], "row_bytes": best["row_bytes"],
       "how": "tools/microbench/l2_gather.cu: N random 256-byte rows of an L2-resident V-row table gathered with "
              "16-byte lane slices (LDG.128), best of 10 reps and of the listed variants, CUDA events",
       "variants": rows[:-1]}
json.dump(res, open(os.path.join(ROOT, "profiles", "l2_gather_peak.json"), "w"), indent=1)

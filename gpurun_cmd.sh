timeout 900 python tools/sweep.py --grid selector_fused --out gpurun_out/perfdb_r1c.jsonl > gpurun_out/sweep_r1c.log 2>&1; echo "sweep rc=$?"
wc -l gpurun_out/perfdb_r1c.jsonl

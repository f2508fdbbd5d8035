timeout 1200 python tools/sweep.py --grid selector_fused --out gpurun_out/perfdb_r1d.jsonl > gpurun_out/sweep_r1d.log 2>&1; echo "sweep rc=$?"
wc -l gpurun_out/perfdb_r1d.jsonl

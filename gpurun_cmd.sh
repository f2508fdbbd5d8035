timeout 2700 python tools/sweep.py --grid selector --out gpurun_out/perfdb_r1b.jsonl > gpurun_out/sweep_r1b.log 2>&1; echo "sweep rc=$?"
timeout 900 python tools/sweep.py --grid selector_large --out gpurun_out/perfdb_r1b.jsonl >> gpurun_out/sweep_r1b.log 2>&1; echo "sweep-large rc=$?"
wc -l gpurun_out/perfdb_r1b.jsonl

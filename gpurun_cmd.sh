bash tools/gpu_round.sh r1h
timeout 900 python tools/report_configs.py --md gpurun_out/r1h_configs.md --jsonl gpurun_out/r1h_configs.jsonl > gpurun_out/r1h_configs.log 2>&1; echo "configs rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1h_smoke.log 2>&1; echo "smoke rc=$?"

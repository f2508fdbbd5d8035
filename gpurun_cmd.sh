bash tools/gpu_round.sh r1e
timeout 900 python tools/report_configs.py --md gpurun_out/r1e_configs.md --jsonl gpurun_out/r1e_configs.jsonl > gpurun_out/r1e_configs.log 2>&1; echo "configs rc=$?"

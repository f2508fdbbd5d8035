bash tools/gpu_round.sh r1d
timeout 900 python tools/report_configs.py --md gpurun_out/r1d_configs.md --jsonl gpurun_out/r1d_configs.jsonl > gpurun_out/r1d_configs.log 2>&1; echo "configs rc=$?"

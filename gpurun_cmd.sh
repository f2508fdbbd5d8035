bash tools/gpu_round.sh r1f
timeout 900 python tools/report_configs.py --md gpurun_out/r1f_configs.md --jsonl gpurun_out/r1f_configs.jsonl > gpurun_out/r1f_configs.log 2>&1; echo "configs rc=$?"
bash tools/gpu_prof4.sh r1f "narrow f1 16777216 1048576 1 f32 powerlaw" "stream_kernel reddit 114615892 232965 64 f32 powerlaw - fused" "stream_kernel products 61859140 2449029 128 bf16 powerlaw"
ls -la gpurun_out | head -30

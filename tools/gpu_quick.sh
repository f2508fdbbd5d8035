#!/bin/bash
# quick GPU iteration: stream/variant parity subset, bench line, ncu of the top kernel
TAG=${1:-q}
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "${2:-stream or arxiv or worked or forced}" 2>&1 | tail -4
timeout 200 python bench.py --steps 300 --warmup 20 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['selected_config'])"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"${3:-stream_kernel}" -s 2 -c 1 -o gpurun_out/${TAG}_prof python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu.log 2>&1; tail -1 gpurun_out/${TAG}_ncu.log

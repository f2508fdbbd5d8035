#!/bin/bash
# One GPU call: parity tests, a bench line, the ncu launch list and one full
# capture of the top kernel.  Usage: bash tools/gpu_round.sh TAG [pytest-args]
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q ${@:2} > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/${TAG}_pytest.log
timeout 300 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo "ncu-list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stream_kernel|edge_tile" -s 5 -c 1 -o gpurun_out/${TAG}_prof \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu-full rc=$?"
tail -3 gpurun_out/${TAG}_ncu_full.log

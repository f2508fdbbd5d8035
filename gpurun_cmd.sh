for i in 1 2; do python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], d['roofline']['kernel_ms'], d['clocks'])"; done
timeout 900 python -m pytest tests/test_gpu_allgather.py -m gpu -q -x 2>&1 | tail -2

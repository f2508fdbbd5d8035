timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "bad_data or stream or int64" 2>&1 | tail -2
for i in 1 2; do
(cd abold && python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('OLD', d['value'], d['roofline']['kernel_ms'])")
python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NEW', d['value'], d['roofline']['kernel_ms'])"
done

timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_selector.py -m gpu -q -x 2>&1 | tail -3
python tools/time_cfgs.py 16777216 1048576 16 f32 powerlaw -- '' '{"variant":2}' '{"variant":1}'
python tools/time_cfgs.py 16777216 1048576 16 f32 uniform -- '{"variant":2}' '{"variant":1}'
python tools/time_cfgs.py 16777216 1048576 16 bf16 powerlaw -- '{"variant":2}' '{"variant":1}'
python tools/time_cfgs.py 16777216 1048576 8 f32 powerlaw -- '{"variant":2}' '{"variant":1}'
for F in 32 64; do python tools/time_cfgs.py 16777216 1048576 $F f32 powerlaw -- '' 2>&1; done
python bench.py --workload products --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200

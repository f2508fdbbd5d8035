timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -2
timeout 300 python tools/quick_perf.py 2>&1 | tail -17
python tools/time_cfgs.py 114615892 232965 64 f32 powerlaw fused -- '{"variant":1}'

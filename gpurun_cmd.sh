timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "stream or arxiv or products or sweep or fused or gather" 2>&1 | tail -2
python bench.py --no-cpu-baseline --steps 300 2>&1 | tail -1 | cut -c1-220
python bench.py --workload products --no-cpu-baseline 2>&1 | tail -1 | cut -c1-220
python tools/time_cfgs.py 16777216 1048576 64 f32 powerlaw -- ''
python tools/time_cfgs.py 16777216 1048576 32 f32 powerlaw -- ''
python tools/time_cfgs.py 114615892 232965 64 f32 powerlaw fused -- ''

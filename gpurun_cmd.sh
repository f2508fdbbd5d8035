timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fused or gather" 2>&1 | tail -2
python tools/time_cfgs.py 114615892 232965 64 f32 powerlaw fused -- ''
python tools/time_cfgs.py 16777216 1048576 32 f32 powerlaw fused -- ''

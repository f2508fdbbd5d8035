timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_selector.py -m gpu -q -x -k "fused or gather or select" 2>&1 | tail -4
python tools/time_cfgs.py 114615892 232965 64 f32 powerlaw fused -- ''
python tools/time_cfgs.py 16777216 1048576 128 f32 powerlaw fused -- ''
python tools/time_cfgs.py 16777216 1048576 32 f32 powerlaw fused -- ''
bash tools/gpu_prof4.sh p11 "stream_kernel reddit 114615892 232965 64 f32 powerlaw - fused"

#!/bin/bash
# narrow-kernel iteration: parity subset + timing of the small-F sweep points (+ optional ncu captures)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "narrow or sweep or small_f" 2>&1 | tail -3
timeout 300 python tools/quick_perf.py 2>&1 | tail -25
if [ -n "$1" ]; then bash tools/gpu_prof4.sh $1 "narrow f1 16777216 1048576 1 f32 powerlaw" "narrow f1u 16777216 1048576 1 f32 uniform" "narrow f4 16777216 1048576 4 f32 powerlaw"; fi

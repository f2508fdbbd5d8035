#!/bin/bash
# narrow-kernel iteration: parity subset + timing of the small-F sweep points
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "narrow or sweep or small_f" 2>&1 | tail -5
timeout 300 python tools/quick_perf.py 2>&1 | tail -25

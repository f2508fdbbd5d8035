run() { timeout 30 python tools/dbg_bad.py "$@" > /tmp/o.txt 2>&1; echo "rc=$? $*: $(tail -1 /tmp/o.txt | cut -c1-150)"; }
run 3 64 f32 sorted 100000 400 -30 430
run 3 16 f32 unsorted 100000 400 -30 430
run 3 64 f32 unsorted_fused 100000 400 -30 430
run 3 16 f32 sorted_fused 100000 400 -30 430
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "bad_data or fused_gather_stream or every_pipeline" 2>&1 | tail -3

timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], d['roofline']['frac'], d['clocks'])"
timeout 900 python tools/report_configs.py --md gpurun_out/r1i_configs.md --jsonl gpurun_out/r1i_configs.jsonl > gpurun_out/r1i_configs.log 2>&1; echo "configs rc=$?"

#!/bin/bash
# bench.py under several configurations (selector experiments)
W=${1:-arxiv}
for c in '' '{"variant":3,"warps_per_cta":8,"rows_per_group":8,"stages":6}' '{"variant":3,"warps_per_cta":16,"rows_per_group":3,"stages":8}' '{"variant":3,"warps_per_cta":8,"rows_per_group":6,"stages":8}' '{"variant":1,"rows_per_group":64}'; do
  timeout 120 python bench.py --workload $W --steps 300 --warmup 20 --no-cpu-baseline --e2e-steps 1 --cfg "$c" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$W', '$c', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])"
done

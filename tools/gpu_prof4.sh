#!/bin/bash
# ncu --set full captures of chosen cases: tools/gpu_prof4.sh TAG "kregex name E S F dtype dist cfg fused" ...
mkdir -p gpurun_out
T=$1; shift
for spec in "$@"; do
  set -- $spec
  timeout 400 ncu ${NCU_SET:---set full --import-source on} --clock-control none -k regex:"$1" -s 2 -c 1 -o gpurun_out/${T}_$2 \
     python tools/prof_case.py $3 $4 $5 $6 $7 $8 $9 > gpurun_out/${T}_$2.log 2>&1; echo "$2 rc=$?"
done

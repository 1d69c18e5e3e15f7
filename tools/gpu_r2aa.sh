#!/bin/bash
TAG=${1:-r2aa}
mkdir -p gpurun_out
for Q in Q3 Q5 Q7 Q20; do
  timeout 900 ncu --set full --clock-control none -k regex:scx_pipe -c 6 \
    -o gpurun_out/prof_${Q}_$TAG -f python tools/one_query.py --sf 100 --query $Q --warm 0 > gpurun_out/ncu_${Q}_$TAG.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof_${Q}_$TAG.ncu-rep > gpurun_out/ncu_${Q}_$TAG.txt 2>&1
  echo "== $Q"; cat gpurun_out/ncu_${Q}_$TAG.txt | cut -c1-420
done

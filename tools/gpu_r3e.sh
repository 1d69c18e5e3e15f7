#!/bin/bash
# ncu --set full of every scx_pipe kernel of the probe-heavy queries at SF100
# (Q3 Q5 Q7 Q8 Q21): DRAM vs L2 vs issue bound per kernel (tools/ncu_l2.py)
TAG=${1:-r3e}
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none -k regex:scx_pipe -o gpurun_out/prof_probe_$TAG -f \
  python tools/one_query.py --sf 100 --query Q3,Q5,Q7,Q8,Q21 --warm 0 > gpurun_out/ncu_probe_$TAG.log 2>&1
echo "ncu rc=$?"
python tools/ncu_l2.py gpurun_out/prof_probe_$TAG.ncu-rep 0.2 > gpurun_out/ncu_probe_$TAG.txt 2>&1
cat gpurun_out/ncu_probe_$TAG.txt

#!/bin/bash
# ncu --set full of the probe-heavy Q9 scan kernels and of the partition scatter
# (DESIGN §6 gaps 1 and 3).  Usage (under gpurun): bash tools/gpu_probe_prof.sh TAG [SF]
TAG=${1:-r1}
SF=${2:-100}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:scx_pipe -c 6 \
  -o gpurun_out/prof_q9_$TAG -f python tools/one_query.py --sf $SF --query Q9 --warm 0 > gpurun_out/ncu_q9_$TAG.log 2>&1
echo "q9 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:part_scatter -c 1 \
  -o gpurun_out/prof_part_$TAG -f python tools/part_bench.py --parts 8 > gpurun_out/ncu_part_$TAG.log 2>&1
echo "part rc=$?"
python tools/ncu_summary.py gpurun_out/prof_q9_$TAG.ncu-rep > gpurun_out/ncu_q9_$TAG.txt 2>&1
python tools/ncu_summary.py gpurun_out/prof_part_$TAG.ncu-rep > gpurun_out/ncu_part_$TAG.txt 2>&1
cat gpurun_out/ncu_q9_$TAG.txt gpurun_out/ncu_part_$TAG.txt

#!/bin/bash
TAG=${1:-p}
mkdir -p gpurun_out
for c in 4 0 8; do echo "ctas/sm=$c"; SCX_PART_CTAS=$c timeout 300 python tools/part_bench.py --parts 1,8,64; done > gpurun_out/part_$TAG.log 2>&1
cat gpurun_out/part_$TAG.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"part_(hist|scatter)" -c 2 -o gpurun_out/part_$TAG -f python tools/part_bench.py --parts 8 > gpurun_out/ncu_part_$TAG.log 2>&1
tail -1 gpurun_out/ncu_part_$TAG.log

#!/bin/bash
# partition: direct scatter vs staged (parity + timing + ncu)
TAG=${1:-r2j}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "partition or shuffle or exchange or inprocess or hash" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 3 gpurun_out/pytest_$TAG.log
for D in 1 0; do
  echo "SCX_PART_DIRECT=$D"; SCX_PART_DIRECT=$D timeout 300 python tools/part_bench.py --parts 1,2,8,64 2>&1
done
for G in 8 32; do
  echo "direct, $G GiB"; timeout 300 python tools/part_bench.py --gib $G --parts 8 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:part_ -c 3 \
  -o gpurun_out/prof_part_$TAG -f python tools/part_bench.py --parts 8 > gpurun_out/ncu_part_$TAG.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_part_$TAG.ncu-rep > gpurun_out/ncu_part_$TAG.txt 2>&1; cat gpurun_out/ncu_part_$TAG.txt

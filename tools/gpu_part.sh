#!/bin/bash
# Partition kernel iteration: parity tests, timing, one ncu full capture.
TAG=${1:-p}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "partition or hash or shuffle or exchange" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 5 gpurun_out/pytest_$TAG.log
timeout 300 python tools/part_bench.py --parts 1,2,3,8,16,64 > gpurun_out/part_$TAG.log 2>&1
cat gpurun_out/part_$TAG.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"part_(hist|scatter)" -c 2 -o gpurun_out/part_$TAG -f python tools/part_bench.py --parts 8 > gpurun_out/ncu_part_$TAG.log 2>&1
tail -2 gpurun_out/ncu_part_$TAG.log

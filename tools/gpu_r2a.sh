#!/bin/bash
# Round-2 first GPU check: host resources, -m gpu parity, partition kernel
# timing + one ncu full capture of the scatter.
mkdir -p gpurun_out
{ free -g; nproc; lscpu | grep -i "model name\|socket\|numa node(s)"; } > gpurun_out/host_r2.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2a.log
tail -n 25 gpurun_out/pytest_r2a.log
timeout 300 python tools/part_bench.py --parts 1,2,4,8,16,64 > gpurun_out/part_r2a.log 2>&1
cat gpurun_out/part_r2a.log
timeout 600 ncu --set full --clock-control none -k regex:part_ -c 4 -o gpurun_out/part_r2a -f python tools/part_bench.py --parts 8 > gpurun_out/ncu_part_r2a.log 2>&1
tail -3 gpurun_out/ncu_part_r2a.log

#!/bin/bash
TAG=${1:-r2ac}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "tpch22 or equals or parity" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 2 gpurun_out/pytest_$TAG.log; grep FAILED gpurun_out/pytest_$TAG.log | head
timeout 1800 python tools/chunk_sweep.py --reps 4 --queries Q3,Q5,Q7,Q10,Q12,Q14,Q17,Q19,Q20,Q8,Q4,Q21 --configs "X=1;SCX_CHUNK_PF=0" > gpurun_out/sweep_$TAG.log 2>&1
grep -v "^{" gpurun_out/sweep_$TAG.log | cut -c1-1000

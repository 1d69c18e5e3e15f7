#!/bin/bash
TAG=${1:-r2ag}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 2 gpurun_out/pytest_$TAG.log; grep FAILED gpurun_out/pytest_$TAG.log | head
timeout 1800 python tools/chunk_sweep.py --reps 4 --queries Q6,Q1,Q14,Q12,Q4,Q22,Q15,Q19,Q5,Q13,Q18 --configs "X=1;SCX_CHUNK_LATE=0" > gpurun_out/sweep_$TAG.log 2>&1
grep -v "^{" gpurun_out/sweep_$TAG.log | cut -c1-1100

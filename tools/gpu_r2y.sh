#!/bin/bash
TAG=${1:-r2y}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 2 gpurun_out/pytest_$TAG.log; grep FAILED gpurun_out/pytest_$TAG.log | head
timeout 1800 python tools/chunk_sweep.py --reps 3 --queries Q9,Q2,Q16,Q20,Q21,Q11,Q13,Q18,Q10 --configs "X=1" > gpurun_out/sweep_$TAG.log 2>&1
grep -v "^{" gpurun_out/sweep_$TAG.log | cut -c1-1000

#!/bin/bash
TAG=${1:-r2n}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 3 gpurun_out/pytest_$TAG.log
timeout 1800 python tools/chunk_sweep.py --reps 4 --queries Q3,Q5,Q7,Q10,Q12,Q14,Q17,Q19,Q20,Q2 --configs "X=1;SCX_CHUNK_V=4;SCX_CHUNK_V=8;SCX_CHUNK=0" > gpurun_out/sweep_$TAG.log 2>&1
grep -v "^{" gpurun_out/sweep_$TAG.log | cut -c1-1300
timeout 900 python tools/sync_count.py > gpurun_out/sync_$TAG.log 2>&1; tail -23 gpurun_out/sync_$TAG.log | cut -c1-200

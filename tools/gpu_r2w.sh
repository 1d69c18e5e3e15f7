#!/bin/bash
TAG=${1:-r2w}
mkdir -p gpurun_out
timeout 1800 python tools/chunk_sweep.py --reps 4 --queries Q21,Q4,Q22,Q13,Q18,Q3,Q9,Q20,Q8 --configs "X=1;SCX_CHUNK=0" > gpurun_out/sweep_$TAG.log 2>&1
grep -v "^{" gpurun_out/sweep_$TAG.log | cut -c1-1000

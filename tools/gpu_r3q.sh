#!/bin/bash
# shared-memory coarse bitmap level on / off for the bitmap-probe queries
TAG=${1:-r3q}
mkdir -p gpurun_out
timeout 1500 python tools/chunk_sweep.py --reps 3 --queries Q8,Q9,Q2,Q17,Q20,Q21,Q14,Q19,Q16 --configs "SCX_COARSE=0;SCX_COARSE=1" > gpurun_out/sweep_$TAG.log 2>&1; echo "sweep rc=$?"
grep -v "^{" gpurun_out/sweep_$TAG.log | cut -c1-1500

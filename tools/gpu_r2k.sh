#!/bin/bash
TAG=${1:-r2k}
mkdir -p gpurun_out
timeout 1500 python tools/chunk_sweep.py --queries Q3,Q5,Q7,Q10,Q12,Q17,Q19,Q20,Q21,Q2,Q16,Q4,Q13,Q14,Q15,Q18,Q22,Q8,Q9,Q11 --configs "SCX_CHUNK_V=4;SCX_CHUNK_V=8;SCX_CHUNK_V=2;SCX_CHUNK_V=8,SCX_CHUNK_U0=2;SCX_CHUNK_V=8,SCX_TMA_RING_KB=48" > gpurun_out/sweep_$TAG.log 2>&1
grep -v "^{" gpurun_out/sweep_$TAG.log | cut -c1-1300

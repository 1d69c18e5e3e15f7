#!/bin/bash
# Quick GPU iteration: parity tests, then per-query wall times at SF100.
# Usage (under gpurun): bash tools/gpu_quick.sh TAG [pytest -k expr]
TAG=${1:-q}
mkdir -p gpurun_out
if [ -n "$2" ]; then K="-k $2"; fi
timeout 1200 python -m pytest tests -m gpu -x -q $K > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 15 gpurun_out/pytest_$TAG.log
timeout 600 python tools/qprof.py --sf ${SF:-100} --profile Q1 > gpurun_out/qprof_$TAG.log 2>&1
grep "ms wall" gpurun_out/qprof_$TAG.log | awk '{s+=$2; print} END {print "sum", s}'

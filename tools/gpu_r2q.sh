#!/bin/bash
TAG=${1:-r2q}
mkdir -p gpurun_out
timeout 900 python tools/pyprof_suite.py --sf 1 --reps 10 > gpurun_out/pyprof_$TAG.log 2>&1; echo "rc=$?"
head -3 gpurun_out/pyprof_$TAG.log | cut -c1-1500

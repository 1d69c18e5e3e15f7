#!/bin/bash
TAG=${1:-d}
mkdir -p gpurun_out
timeout 900 python tools/inproc_check.py --n 2,3,8 --sf 0.1 > gpurun_out/inproc_$TAG.log 2>&1
grep -v "^ok" gpurun_out/inproc_$TAG.log | tail -40

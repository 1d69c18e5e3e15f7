#!/bin/bash
# Official evidence run (one GPU): bench line, reference arm, ncu launch list of
# one warm 22-query pass, ncu --set full of Q1's scan kernel (the roofline kernel).
# Usage (under gpurun): bash tools/gpu_bench.sh TAG [SF]
TAG=${1:-r1}
SF=${2:-100}
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 5 --warmup 3 --sf $SF > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 --sf $SF > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
echo "ref rc=$?"
python tools/suite_once.py --sf $SF --warm 2 > /dev/null 2>&1   # JIT cache warm on disk
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv --nvtx --nvtx-include "timed_suite/" python tools/suite_once.py --sf $SF --warm 1 > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scx_pipe -c 1 -o gpurun_out/prof_q1_$TAG -f python tools/one_query.py --sf $SF --query Q1 --warm 0 > gpurun_out/ncu_q1_$TAG.log 2>&1
echo "ncu full rc=$?"
cat gpurun_out/bench_$TAG.json

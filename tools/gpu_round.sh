#!/bin/bash
# One GPU call: parity tests, smoke, bench line, ncu launch list + one full capture.
# Usage (under gpurun): bash tools/gpu_round.sh [tag] [sf]
set -x
TAG=${1:-r1}
SF=${2:-10}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --steps 5 --warmup 3 --sf $SF > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 --sf $SF > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --sf $SF --no-cpu > gpurun_out/ncu_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-scx_pipe} -s 30 -c 6 -o gpurun_out/prof_$TAG -f python bench.py --steps 1 --warmup 3 --sf $SF --no-cpu > gpurun_out/ncu_full_$TAG.log 2>&1
tail -n 3 gpurun_out/pytest_gpu_$TAG.log gpurun_out/smoke_$TAG.log
cat gpurun_out/bench_$TAG.json gpurun_out/bench_ref_$TAG.json
tail -5 gpurun_out/bench_$TAG.err

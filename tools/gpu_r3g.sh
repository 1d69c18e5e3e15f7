#!/bin/bash
# GPU tests + short bench after the vectorised region copy
TAG=${1:-r3g}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -2 gpurun_out/pytest_$TAG.log
if [ $rc -ne 0 ]; then grep -m2 -B5 -A40 "^____" gpurun_out/pytest_$TAG.log | head -80; exit 1; fi
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu --no-configs --sweep "" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
print(d["value"], d["single_stream"]["value"], d["e2e"]["value"], d["parity"]["ok"], d["roofline"]["frac"], d["gpu_launches"])
print({q: round(v["s"]*1e3, 2) for q, v in d["per_query"].items()})
PY
python tools/suite_once.py --sf 100 --warm 2 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv --nvtx --nvtx-include "timed_suite/" python tools/suite_once.py --sf 100 --warm 1 > gpurun_out/ncu_launch_$TAG.log 2>&1
python tools/launch_summary.py gpurun_out/launches_$TAG.csv | grep -i "region\|launches"

#!/bin/bash
# GPU tests + bench (per-query single-stream times) after a codegen change
TAG=${1:-r3d}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log; grep -m3 -A30 "^___" gpurun_out/pytest_$TAG.log | head -60
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu --no-configs --sweep "" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
print(d["value"], d["single_stream"]["value"], d["e2e"]["value"], d["parity"]["ok"], d["roofline"]["frac"], d["roofline"]["launch_ms"], d["roofline"]["kernel"])
print({q: round(v["s"]*1e3, 2) for q, v in d["per_query"].items()})
PY

#!/bin/bash
TAG=${1:-r2ad}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "codec or parity or equals" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 2 gpurun_out/pytest_$TAG.log; grep FAILED gpurun_out/pytest_$TAG.log | head
timeout 1500 python bench.py --no-configs --no-cpu --steps 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_$TAG.err
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
print("value", d["value"], "single", d["single_stream"]["value"], "e2e", d["e2e"])
print("parity", d["parity"].get("ok"), d["parity"].get("mismatches"))
PY

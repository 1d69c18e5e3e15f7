#!/bin/bash
TAG=${1:-r2v}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 2 gpurun_out/pytest_$TAG.log; grep FAILED gpurun_out/pytest_$TAG.log | head
timeout 900 python tools/sync_count.py > gpurun_out/sync_$TAG.log 2>&1; tail -23 gpurun_out/sync_$TAG.log | cut -c1-140
timeout 1500 python bench.py --no-configs --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_$TAG.err
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
print("value", d["value"], "single", d["single_stream"]["value"], "e2e", d["e2e"]["value"], d["e2e"]["passes_ms"])
print("parity", d["parity"].get("ok"), d["parity"].get("mismatches"), "suite", d.get("suite_roofline"))
print({q: (round(v["s"] * 1e3, 2), v["roof_frac"]) for q, v in d["per_query"].items()})
PY

#!/bin/bash
# official evidence: default bench line (configs, sweep, CPU sample) + reference arm
TAG=${1:-r3c}
mkdir -p gpurun_out
timeout 1800 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["e2e"].get("passes_ms"), d["e2e"].get("passes_upload_done_ms"), d["e2e"].get("results_match_device_run"), d.get("parity", {}).get("ok"), d["roofline"]["frac"], d.get("clocks"))
PY
tail -c 600 gpurun_out/bench_ref_$TAG.json

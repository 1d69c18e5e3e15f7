#!/bin/bash
# round-2 closing evidence: full GPU tests + smoke, default bench line, reference arm
TAG=${1:-r3t}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -2 gpurun_out/pytest_$TAG.log
if [ $rc -ne 0 ]; then grep -m2 -B5 -A40 "^____" gpurun_out/pytest_$TAG.log | head -80; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 1800 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["single_stream"]["value"], d["e2e"]["value"], d["e2e"]["h2d_bytes_per_step"], d["e2e"].get("passes_ms"), d["e2e"].get("passes_upload_done_ms"), d["e2e"].get("results_match_device_run"), d["parity"]["ok"], d["roofline"]["frac"], d.get("clocks"), d.get("gpu_launches"))
PY

#!/bin/bash
# key-relative dates: GPU codec / e2e tests, then the e2e bench
TAG=${1:-r3s}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_codec.py tests/test_gpu_compact_io.py -x -q > gpurun_out/pytest_$TAG.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -2 gpurun_out/pytest_$TAG.log
if [ $rc -ne 0 ]; then grep -m2 -B5 -A40 "^____" gpurun_out/pytest_$TAG.log | head -80; exit 1; fi
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu --no-configs --sweep "" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
e = d["e2e"]
print(d["value"], e["value"], e["h2d_bytes_per_step"], e["passes_ms"], e["passes_upload_done_ms"], e["results_match_device_run"], d["parity"]["ok"])
print(sorted(e["last_pass_query_done_ms"].items(), key=lambda kv: kv[1])[-5:])
PY

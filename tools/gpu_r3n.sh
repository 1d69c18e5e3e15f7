#!/bin/bash
TAG=${1:-r3n}
mkdir -p gpurun_out
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu --no-configs --sweep "" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
e = d["e2e"]
print(d["value"], d["single_stream"]["value"], e["value"], e["passes_ms"], e["passes_upload_done_ms"], e["results_match_device_run"], d["parity"]["ok"])
print(e["query_order"]); print(e["worker_queues"])
print(sorted(e["last_pass_query_done_ms"].items(), key=lambda kv: kv[1]))
PY

#!/bin/bash
TAG=${1:-r3x}
mkdir -p gpurun_out
for CS in 1 2 3; do
SCX_E2E_COST_SCALE=$CS timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-configs --sweep "" > gpurun_out/bench_${TAG}_$CS.json 2> gpurun_out/bench_${TAG}_$CS.err
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_${TAG}_$CS.json").read().strip().splitlines()[-1])
e = d["e2e"]
print("scale $CS", d["value"], e["value"], e["passes_ms"], e["passes_upload_done_ms"], e["results_match_device_run"], d["parity"]["ok"])
print(e["worker_queues"]); print(sorted(e["last_pass_query_done_ms"].items(), key=lambda kv: kv[1])[-4:])
PY
done

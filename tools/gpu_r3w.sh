#!/bin/bash
# e2e worker queues: modelled static (default) vs one dynamic queue
TAG=${1:-r3w}
mkdir -p gpurun_out
for Q in static dynamic; do
SCX_E2E_QUEUE=$Q timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-configs --sweep "" > gpurun_out/bench_${TAG}_$Q.json 2> gpurun_out/bench_${TAG}_$Q.err
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_${TAG}_$Q.json").read().strip().splitlines()[-1])
e = d["e2e"]
print("$Q", d["value"], e["value"], e["passes_ms"], e["passes_upload_done_ms"], e["results_match_device_run"], d["parity"]["ok"])
print(sorted(e["last_pass_query_done_ms"].items(), key=lambda kv: kv[1])[-4:])
PY
done

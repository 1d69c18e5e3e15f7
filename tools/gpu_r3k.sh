#!/bin/bash
# e2e timeline: one copy stream + unpack stream (default) vs two copy streams
TAG=${1:-r3k}
mkdir -p gpurun_out
for US in 1 2; do
SCX_UPLOAD_STREAMS=$US timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu --no-configs --sweep "" > gpurun_out/bench_${TAG}_$US.json 2> gpurun_out/bench_${TAG}_$US.err; echo "bench $US rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_${TAG}_$US.json").read().strip().splitlines()[-1])
e = d["e2e"]
print("upload streams $US", d["value"], e["value"], e["passes_ms"], e["passes_upload_done_ms"], e["results_match_device_run"])
print(e["worker_queues"])
print(sorted(e["last_pass_query_done_ms"].items(), key=lambda kv: kv[1]))
print(sorted(e["last_pass_column_landed_ms"].items(), key=lambda kv: kv[1]))
PY
done

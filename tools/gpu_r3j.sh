#!/bin/bash
# e2e timeline: whole-column H2D copies vs 64 MB pieces
TAG=${1:-r3j}
mkdir -p gpurun_out
for CH in 0 64; do
SCX_H2D_CHUNK_MB=$CH timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu --no-configs --sweep "" > gpurun_out/bench_${TAG}_$CH.json 2> gpurun_out/bench_${TAG}_$CH.err; echo "bench $CH rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_${TAG}_$CH.json").read().strip().splitlines()[-1])
e = d["e2e"]
print("chunk MB $CH", d["value"], e["value"], e["passes_ms"], e["passes_upload_done_ms"])
print(sorted(e["last_pass_query_done_ms"].items(), key=lambda kv: kv[1]))
print(sorted(e["last_pass_column_landed_ms"].items(), key=lambda kv: kv[1]))
PY
done

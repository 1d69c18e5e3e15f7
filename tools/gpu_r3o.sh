#!/bin/bash
# query-stream count sweep (device-resident suite and e2e)
TAG=${1:-r3o}
mkdir -p gpurun_out
for NS in 4 5 6 8; do
SCX_BENCH_STREAMS=$NS timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-configs --sweep "" > gpurun_out/bench_${TAG}_$NS.json 2> gpurun_out/bench_${TAG}_$NS.err
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_${TAG}_$NS.json").read().strip().splitlines()[-1])
e = d["e2e"]
print("streams $NS", d["value"], d["single_stream"]["value"], e["value"], e["passes_ms"], d["parity"]["ok"])
PY
done

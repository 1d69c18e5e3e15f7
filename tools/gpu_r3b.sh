#!/bin/bash
# e2e with column-level upload order vs table order; Q9's generated kernels
TAG=${1:-r3b}
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 5 --warmup 3 --no-configs --sweep "" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-configs --sweep "" --table-order > gpurun_out/bench_${TAG}_tab.json 2> gpurun_out/bench_${TAG}_tab.err; echo "bench tab rc=$?"
SCX_JIT_DUMP=1 timeout 600 python tools/one_query.py --sf 100 --query Q9 --warm 0 > gpurun_out/q9dump_$TAG.log 2>&1; echo "dump rc=$?"
python - <<PY
import json
for f in ["gpurun_out/bench_$TAG.json", "gpurun_out/bench_${TAG}_tab.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["e2e"]["value"], d["e2e"].get("passes_ms"), d["e2e"].get("passes_upload_done_ms"), d["e2e"].get("results_match_device_run"), d.get("parity"))
    except Exception as e:
        print(f, "ERR", e)
PY

#!/bin/bash
# GPU tests + e2e timeline with mapped result reads (vs SCX_MAPPED_READS=0)
TAG=${1:-r3l}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -2 gpurun_out/pytest_$TAG.log
if [ $rc -ne 0 ]; then grep -m2 -B5 -A40 "^____" gpurun_out/pytest_$TAG.log | head -80; exit 1; fi
for MR in 1 0; do
SCX_MAPPED_READS=$MR timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu --no-configs --sweep "" > gpurun_out/bench_${TAG}_$MR.json 2> gpurun_out/bench_${TAG}_$MR.err; echo "bench $MR rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_${TAG}_$MR.json").read().strip().splitlines()[-1])
e = d["e2e"]
print("mapped $MR", d["value"], d["single_stream"]["value"], e["value"], e["passes_ms"], e["passes_upload_done_ms"], e["results_match_device_run"], d["parity"]["ok"])
print(sorted(e["last_pass_query_done_ms"].items(), key=lambda kv: kv[1]))
PY
done

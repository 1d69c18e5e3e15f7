#!/bin/bash
# final round-2 evidence: default bench line + reference arm, then
# compute-sanitizer memcheck / racecheck over the SF0.01 suite
TAG=${1:-r3p}
mkdir -p gpurun_out
timeout 1800 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["single_stream"]["value"], d["e2e"]["value"], d["e2e"].get("passes_ms"), d["e2e"].get("passes_upload_done_ms"), d["e2e"].get("results_match_device_run"), d["parity"]["ok"], d["roofline"]["frac"], d.get("clocks"), d.get("gpu_launches"))
PY
for T in memcheck racecheck; do
  N3=1; [ $T != memcheck ] && N3=0
  SAN_N3=$N3 timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_suite.py > gpurun_out/sanitize_${T}_$TAG.log 2>&1
  echo "$T rc=$?"; tail -3 gpurun_out/sanitize_${T}_$TAG.log
done

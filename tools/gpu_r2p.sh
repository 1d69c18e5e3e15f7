#!/bin/bash
TAG=${1:-r2p}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 2 gpurun_out/pytest_$TAG.log; grep -n "FAILED" gpurun_out/pytest_$TAG.log | head -5
timeout 900 python tools/sync_count.py > gpurun_out/sync_$TAG.log 2>&1; tail -23 gpurun_out/sync_$TAG.log | cut -c1-120
timeout 1800 python tools/chunk_sweep.py --reps 4 --queries Q3,Q5,Q7,Q14,Q17,Q19,Q20,Q2,Q9 --configs "X=1;SCX_CHUNK_V=4" > gpurun_out/sweep_$TAG.log 2>&1
grep -v "^{" gpurun_out/sweep_$TAG.log | cut -c1-1000
timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_$TAG.err
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
print("value", d["value"], "single", d["single_stream"]["value"], "e2e", d["e2e"]["value"], "parity", d["parity"].get("ok"), d["parity"].get("mismatches"))
print("roofline", d["roofline"]["frac"], "suite", d.get("suite_roofline"), "shuffle", d.get("shuffle", {}).get("partition_frac_hbm"))
print({q: (round(v["s"] * 1e3, 2), v["roof_frac"]) for q, v in d["per_query"].items()})
PY

#!/bin/bash
# late materialisation + chunk A/B (per query), e2e arena, concurrency check
TAG=${1:-r2i}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "codec or parity or tpch22" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 3 gpurun_out/pytest_$TAG.log
timeout 1500 python tools/chunk_sweep.py --queries Q3,Q5,Q7,Q8,Q9,Q10,Q12,Q17,Q19,Q20,Q21,Q2,Q16,Q11,Q4,Q13,Q14,Q15,Q18,Q22 --configs "SCX_CHUNK=0,SCX_LATE=0;SCX_CHUNK=1,SCX_LATE=0;SCX_CHUNK=1,SCX_LATE=1;SCX_CHUNK=0,SCX_LATE=1" > gpurun_out/sweep_$TAG.log 2>&1
grep -v "^{" gpurun_out/sweep_$TAG.log | cut -c1-1200
for CFG in "SCX_CHUNK=1" "SCX_CHUNK=0"; do
  env $CFG timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-configs > gpurun_out/ab_${CFG}_$TAG.json 2> gpurun_out/ab_${CFG}_$TAG.err
  python - <<PY
import json
d = json.loads(open("gpurun_out/ab_${CFG}_$TAG.json").read().strip().splitlines()[-1])
print("$CFG value", d["value"], "single", d["single_stream"]["value"], "e2e", d["e2e"]["value"], d["e2e"].get("passes_ms"), d["e2e"].get("passes_upload_done_ms"), "parity", d["parity"].get("ok"))
PY
done

#!/bin/bash
TAG=${1:-r2m}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 3 gpurun_out/pytest_$TAG.log
timeout 1200 python tools/chunk_sweep.py --queries Q3,Q5,Q7,Q10,Q12,Q17,Q19,Q20,Q21,Q2,Q16,Q4,Q13,Q14,Q15,Q18,Q22,Q8,Q9,Q11 --configs "X=1;SCX_CHUNK_V=4" > gpurun_out/sweep_$TAG.log 2>&1
grep -v "^{" gpurun_out/sweep_$TAG.log | cut -c1-1300
timeout 900 python tools/sync_count.py > gpurun_out/sync_$TAG.log 2>&1; cat gpurun_out/sync_$TAG.log | cut -c1-300
timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_$TAG.err
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
print("value", d["value"], "single", d["single_stream"]["value"], "e2e", d["e2e"])
print("parity", d["parity"].get("ok"), d["parity"].get("mismatches"))
print("roofline", d["roofline"], "suite", d.get("suite_roofline"), "shuffle", d.get("shuffle"))
print({q: (round(v["s"] * 1e3, 2), v["roof_frac"]) for q, v in d["per_query"].items()})
c = d.get("configs") or {}
for k in ("config1_q6_sf1", "config2_q1_sf10"):
    print(k, c.get(k))
print([ (p["gib"], p.get("n_dest"), p.get("frac_hbm")) for p in c.get("config5_partition_sweep", {}).get("points", [])])
PY

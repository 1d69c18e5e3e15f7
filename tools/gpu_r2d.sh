#!/bin/bash
# Round-2 pass D: SF100 Q11 oracle (TPC-H FRACTION fix), -m gpu parity,
# default bench (SF100 parity, packed e2e, configs), gather-prefetch A/B.
TAG=${1:-r2d}
mkdir -p gpurun_out
timeout 600 python tools/sf100_cpu.py --phase oracle --sf 100 --queries Q11 --out gpurun_out/cpu_sf100_q11 > gpurun_out/q11_$TAG.log 2>&1; echo "q11 rc=$?"
tail -2 gpurun_out/q11_$TAG.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 6 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
tail -2 gpurun_out/smoke_$TAG.log
timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
tail -5 gpurun_out/bench_$TAG.err
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
print("value", d["value"], "single", d["single_stream"]["value"], "e2e", d["e2e"])
print("parity", json.dumps(d["parity"])[:600])
print("roofline", d["roofline"]); print("suite_roofline", d.get("suite_roofline"))
print({q: round(v["s"] * 1e3, 2) for q, v in d["per_query"].items()})
c = d.get("configs") or {}
for k in ("config1_q6_sf1", "config2_q1_sf10"):
    print(k, c.get(k))
PY
SCX_GATHER_PF=0 timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-configs > gpurun_out/ab_pf0_$TAG.json 2> gpurun_out/ab_pf0_$TAG.err
python - <<PY
import json
d = json.loads(open("gpurun_out/ab_pf0_$TAG.json").read().strip().splitlines()[-1])
print("PF=0 value", d["value"], "single", d["single_stream"]["value"])
print({q: round(v["s"] * 1e3, 2) for q, v in d["per_query"].items()})
PY

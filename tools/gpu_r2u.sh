#!/bin/bash
# full evidence pass: -m gpu, smoke, default bench, reference arm, ncu launch list
TAG=${1:-r2u}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 2 gpurun_out/pytest_$TAG.log; grep FAILED gpurun_out/pytest_$TAG.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log; tail -2 gpurun_out/smoke_$TAG.log
timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_$TAG.err
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
print("value", d["value"], "single", d["single_stream"]["value"], "e2e", d["e2e"])
print("parity", d["parity"].get("ok"), d["parity"].get("mismatches"), "launches", d["gpu_launches"], "clocks", d["clocks"])
print("roofline", d["roofline"], "suite", d.get("suite_roofline"), "shuffle", d.get("shuffle", {}).get("partition_frac_hbm"))
print({q: (round(v["s"] * 1e3, 2), v["roof_frac"]) for q, v in d["per_query"].items()})
c = d.get("configs") or {}
for k in ("config1_q6_sf1", "config2_q1_sf10"):
    print(k, c.get(k))
print("cpu_baseline", {k: v for k, v in (d.get("cpu_baseline") or {}).items() if k != "per_query_s" and k != "kinds"})
PY
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
tail -c 600 gpurun_out/bench_ref_$TAG.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --print-nvtx-rename none --csv \
  --log-file gpurun_out/launches_q_$TAG.csv python tools/suite_once.py --sf 100 > gpurun_out/ncu_suite_$TAG.log 2>&1; echo "launch list rc=$?"
python tools/launch_by_query.py gpurun_out/launches_q_$TAG.csv 8 > gpurun_out/by_query_$TAG.txt 2>&1; tail -1 gpurun_out/by_query_$TAG.txt

#!/bin/bash
# parity (-m gpu), partition kernel timing + ncu, chunk default vs off, full bench
TAG=${1:-r2h}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 4 gpurun_out/pytest_$TAG.log
timeout 300 python tools/part_bench.py --parts 1,2,4,8,16,64 > gpurun_out/part_$TAG.log 2>&1; cat gpurun_out/part_$TAG.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:part_scatter -c 1 \
  -o gpurun_out/prof_part_$TAG -f python tools/part_bench.py --parts 8 > gpurun_out/ncu_part_$TAG.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_part_$TAG.ncu-rep > gpurun_out/ncu_part_$TAG.txt 2>&1; cat gpurun_out/ncu_part_$TAG.txt
timeout 1200 python tools/chunk_sweep.py --configs "SCX_CHUNK=0;SCX_CHUNK=1" > gpurun_out/sweep_$TAG.log 2>&1
grep -v "^{" gpurun_out/sweep_$TAG.log | cut -c1-900
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
PY

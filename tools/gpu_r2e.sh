#!/bin/bash
# Chunked dense probe kernels: parity first, then suite A/B (SCX_CHUNK=0/1),
# then ncu of the rebuilt Q3 / Q5 scans.
TAG=${1:-r2e}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 30 gpurun_out/pytest_$TAG.log | grep -v "^\s*$" | tail -25
for CH in 1 0; do
  SCX_CHUNK=$CH timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-configs > gpurun_out/ab_ch${CH}_$TAG.json 2> gpurun_out/ab_ch${CH}_$TAG.err
  python - <<PY
import json
d = json.loads(open("gpurun_out/ab_ch${CH}_$TAG.json").read().strip().splitlines()[-1])
print("CHUNK=$CH value", d["value"], "single", d["single_stream"]["value"], "e2e", d["e2e"]["value"], d["e2e"].get("passes_ms"), "parity ok", d["parity"].get("ok"), d["parity"].get("mismatches"))
print({q: round(v["s"] * 1e3, 2) for q, v in d["per_query"].items()})
PY
done
for Q in Q3 Q5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:scx_pipe -c 4 \
    -o gpurun_out/prof_${Q}_$TAG -f python tools/one_query.py --sf 100 --query $Q --warm 0 > gpurun_out/ncu_${Q}_$TAG.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof_${Q}_$TAG.ncu-rep > gpurun_out/ncu_${Q}_$TAG.txt 2>&1
  cat gpurun_out/ncu_${Q}_$TAG.txt
done

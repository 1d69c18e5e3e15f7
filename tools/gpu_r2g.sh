#!/bin/bash
# chunk-mode knob sweep on the probe-heavy queries + one bench line (e2e timeline)
TAG=${1:-r2g}
mkdir -p gpurun_out
timeout 1500 python tools/chunk_sweep.py --configs "SCX_CHUNK=0;SCX_CHUNK=1,SCX_CHUNK_U0=4,SCX_CHUNK_UQ=1;SCX_CHUNK=1,SCX_CHUNK_U0=1,SCX_CHUNK_UQ=1;SCX_CHUNK=1,SCX_CHUNK_U0=4,SCX_CHUNK_UQ=2;SCX_CHUNK=1,SCX_CHUNK_V=8,SCX_CHUNK_U0=4,SCX_CHUNK_UQ=1;SCX_CHUNK=1,SCX_CHUNK_U0=4,SCX_CHUNK_UQ=1,SCX_TMA_RING_KB=32" > gpurun_out/sweep_$TAG.log 2>&1; echo "sweep rc=$?"
grep -v "^{" gpurun_out/sweep_$TAG.log | cut -c1-900
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-configs > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
print("value", d["value"], "single", d["single_stream"]["value"], "e2e", d["e2e"])
PY

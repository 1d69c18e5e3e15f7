#!/bin/bash
TAG=${1:-r2s}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "semantics or group or having or tpch22 or equals" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 2 gpurun_out/pytest_$TAG.log; grep FAILED gpurun_out/pytest_$TAG.log | head
for S in 5 6 8 3; do
  SCX_BENCH_STREAMS=$S timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-configs > gpurun_out/ab_s${S}_$TAG.json 2> gpurun_out/ab_s${S}_$TAG.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_s${S}_$TAG.json').read().strip().splitlines()[-1]); print('streams $S', d['value'], d['single_stream']['value'], d['parity']['ok'])"
  grep "^step" gpurun_out/ab_s${S}_$TAG.err | tr '\n' ' ' | cut -c1-600; echo
done

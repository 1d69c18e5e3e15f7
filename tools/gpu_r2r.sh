#!/bin/bash
TAG=${1:-r2r}
mkdir -p gpurun_out/jit_src_$TAG
for Q in Q3 Q20; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:scx_pipe -c 4 \
    -o gpurun_out/prof_${Q}_$TAG -f python tools/one_query.py --sf 100 --query $Q --warm 0 > gpurun_out/ncu_${Q}_$TAG.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof_${Q}_$TAG.ncu-rep > gpurun_out/ncu_${Q}_$TAG.txt 2>&1
  cat gpurun_out/ncu_${Q}_$TAG.txt | cut -c1-400
done
cp paper_2506_09226_b200/jit_cache/*.cu gpurun_out/jit_src_$TAG/ 2>/dev/null
for S in 2 4 5; do
  SCX_BENCH_STREAMS=$S timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-configs > gpurun_out/ab_s${S}_$TAG.json 2> gpurun_out/ab_s${S}_$TAG.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_s${S}_$TAG.json').read().strip().splitlines()[-1]); print('streams $S', d['value'], d['single_stream']['value'])"
done

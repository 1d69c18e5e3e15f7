#!/bin/bash
TAG=${1:-r2l}
mkdir -p gpurun_out/jit_src_$TAG
timeout 900 python -m pytest tests -m gpu -x -q -k "tpch22 or inprocess or scale" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 3 gpurun_out/pytest_$TAG.log
timeout 900 python tools/chunk_sweep.py --queries Q9 --configs "SCX_Q9_FUSE=0;SCX_Q9_FUSE=1" > gpurun_out/sweep_$TAG.log 2>&1
grep -v "^{" gpurun_out/sweep_$TAG.log | cut -c1-600
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --print-nvtx-rename none --csv \
  --log-file gpurun_out/launches_q_$TAG.csv python tools/suite_once.py --sf 100 > gpurun_out/ncu_suite_$TAG.log 2>&1; echo "launch list rc=$?"
python tools/launch_by_query.py gpurun_out/launches_q_$TAG.csv 8 > gpurun_out/by_query_$TAG.txt 2>&1
cat gpurun_out/by_query_$TAG.txt | cut -c1-400
cp paper_2506_09226_b200/jit_cache/*.cu gpurun_out/jit_src_$TAG/ 2>/dev/null

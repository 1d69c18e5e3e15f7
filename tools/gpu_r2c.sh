#!/bin/bash
# Round-2 profiling pass: -m gpu parity, per-query (NVTX) launch list of one
# warm single-stream suite pass at SF100, the JIT sources of every plan, and
# ncu --set full of the probe-heavy scans of Q3 / Q5 / Q7.
TAG=${1:-r2c}
SF=${2:-100}
mkdir -p gpurun_out/jit_src_$TAG
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --print-nvtx-rename none --csv \
  --log-file gpurun_out/launches_q_$TAG.csv python tools/suite_once.py --sf $SF > gpurun_out/ncu_suite_$TAG.log 2>&1; echo "launch list rc=$?"
python tools/launch_by_query.py gpurun_out/launches_q_$TAG.csv 8 > gpurun_out/by_query_$TAG.txt 2>&1
head -30 gpurun_out/by_query_$TAG.txt
cp paper_2506_09226_b200/jit_cache/*.cu gpurun_out/jit_src_$TAG/ 2>/dev/null
for Q in ${QS:-Q3 Q5 Q7}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:scx_pipe -c ${NK:-4} \
    -o gpurun_out/prof_${Q}_$TAG -f python tools/one_query.py --sf $SF --query $Q --warm 0 > gpurun_out/ncu_${Q}_$TAG.log 2>&1
  echo "$Q rc=$?"
  python tools/ncu_summary.py gpurun_out/prof_${Q}_$TAG.ncu-rep > gpurun_out/ncu_${Q}_$TAG.txt 2>&1
  cat gpurun_out/ncu_${Q}_$TAG.txt
done
# partition scatter (config 5 shape) under ncu --set full
timeout 600 ncu --set full --clock-control none --import-source on -k regex:part_ -c 3 \
  -o gpurun_out/prof_part_$TAG -f python tools/part_bench.py --parts 8 > gpurun_out/ncu_part_$TAG.log 2>&1
echo "part rc=$?"
python tools/ncu_summary.py gpurun_out/prof_part_$TAG.ncu-rep > gpurun_out/ncu_part_$TAG.txt 2>&1
cat gpurun_out/ncu_part_$TAG.txt
# compute-sanitizer over the SF0.01 suite (N=1 and N=3 virtual ranks)
for T in memcheck racecheck synccheck; do
  N3=1; [ $T != memcheck ] && N3=0
  SAN_N3=$N3 timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_suite.py > gpurun_out/sanitize_${T}_$TAG.log 2>&1
  echo "$T rc=$?"; tail -4 gpurun_out/sanitize_${T}_$TAG.log
done

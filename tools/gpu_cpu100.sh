#!/bin/bash
# SF100 CPU path batch on the GPU box host (no GPU use): oracle for the given
# queries, optionally the real reference's six.  Results -> gpurun_out/cpu_sf100/
PHASE=${1:-oracle}
QS=${2:-}
mkdir -p gpurun_out/cpu_sf100
free -g > gpurun_out/cpu_sf100/free_$PHASE.txt
if [ "$PHASE" = "oracle" ]; then
  timeout 3000 python tools/sf100_cpu.py --phase oracle --sf 100 --queries "$QS"
else
  timeout 3000 python tools/sf100_cpu.py --phase reference --sf 100 --queries "$QS"
fi
echo "rc=$?"
tail -5 gpurun_out/cpu_sf100/$PHASE.log

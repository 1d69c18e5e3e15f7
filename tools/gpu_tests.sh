#!/bin/bash
# Full -m gpu suite (optionally a -k filter) + smoke.
TAG=${1:-t}
mkdir -p gpurun_out
if [ -n "$2" ]; then K="-k $2"; fi
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 $K > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -n 30 gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
tail -2 gpurun_out/smoke_$TAG.log

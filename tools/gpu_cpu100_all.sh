#!/bin/bash
# SF100 CPU path on the GPU box's host (no GPU use): the oracle for all 22
# queries (golden results + 1-core times), then the unmodified reference
# (baseline/_ref) for its six queries (1-core times, checked == oracle).
mkdir -p gpurun_out/cpu_sf100
{ free -g; nproc; lscpu | grep -i "model name"; df -h /tmp; } > gpurun_out/cpu_sf100/host.txt 2>&1
timeout 3300 python tools/sf100_cpu.py --phase oracle --sf 100; echo "oracle rc=$?"
rm -rf /tmp/scx_data
timeout 1500 python tools/sf100_cpu.py --phase reference --sf 100; echo "reference rc=$?"
tail -30 gpurun_out/cpu_sf100/oracle.log gpurun_out/cpu_sf100/reference.log

#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dmma" -s 2 -c 2 -o gpurun_out/prof_c5_full python scripts/kernel_sweep.py c5 "" > gpurun_out/ncu_c5.log 2>&1
echo "ncu c5 rc=$?"
timeout 300 python scripts/cta_trace.py c5 > gpurun_out/cta_trace_c5.log 2>&1; echo "trace rc=$?"

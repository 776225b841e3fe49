#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dmma" -s 2 -c 2 -o gpurun_out/prof_c4n8b python scripts/kernel_sweep.py c4 "NRHS=8,REPS=2" > gpurun_out/ncu_c4n8b.log 2>&1; echo "ncu rc=$?"
timeout 600 python scripts/kernel_sweep.py c2 "WARM=100,REPS=50,NRHS=8" "WARM=100,REPS=50,NRHS=4" > gpurun_out/nb8c.log 2>&1
cat gpurun_out/nb8c.log

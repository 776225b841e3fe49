#!/bin/bash
# One full ncu capture of the c4 project kernel (source-level stalls).
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"project_kernel" -s 3 -c 1 \
  -o gpurun_out/prof_c4_project python scripts/kernel_sweep.py c4 "REPS=3,HMAT_MAX_STAGES_P=3" > gpurun_out/ncu_c4_project.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_c4_project.log

#!/bin/bash
set -u
mkdir -p gpurun_out
S="WARM=150,REPS=40,HMAT_MAX_STAGES_P=3"
timeout 900 python scripts/kernel_sweep.py c4 "$S" "$S,HMAT_DEBUG_SKIP=4" "$S,HMAT_DEBUG_SKIP=8" "$S,HMAT_DEBUG_SKIP=1" "$S,HMAT_DEBUG_SKIP=5" "$S" > gpurun_out/flush.log 2>&1
cat gpurun_out/flush.log

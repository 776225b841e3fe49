#!/bin/bash
# pipeline-depth sweep of the single-rhs kernels (c4, c3)
set -u
mkdir -p gpurun_out
timeout 900 python scripts/kernel_sweep.py c4 "" "HMAT_MAX_STAGES_P=3" "HMAT_MAX_STAGES_P=4" \
  "HMAT_STAGE_KB=16,HMAT_MAX_STAGES=6" "HMAT_STAGE_KB=16,HMAT_MAX_STAGES=8" "HMAT_MAX_STAGES_E=4" \
  "HMAT_MAX_STAGES_P=3,HMAT_MAX_STAGES_E=4" "HMAT_STAGE_KB=12,HMAT_MAX_STAGES=8" \
  "HMAT_CTAS_PER_SM=1,HMAT_SMEM_KB=220,HMAT_MAX_STAGES=8" "" > gpurun_out/sweep_c4.log 2>&1; echo "c4 rc=$?"
timeout 600 python scripts/kernel_sweep.py c3 "" "HMAT_MAX_STAGES_P=3" "HMAT_MAX_STAGES_E=4" "HMAT_STAGE_KB=24,HMAT_MAX_STAGES=6" > gpurun_out/sweep_c3.log 2>&1; echo "c3 rc=$?"

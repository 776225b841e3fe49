#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python scripts/kernel_sweep.py c4 "" "HMAT_MAX_STAGES_E=2" "HMAT_STAGE_KB=16,HMAT_MAX_STAGES_P=3,HMAT_MAX_STAGES_E=3" \
  "HMAT_STAGE_KB=16,HMAT_MAX_STAGES_P=4,HMAT_MAX_STAGES_E=4" "HMAT_STAGE_KB=16,HMAT_MAX_STAGES_P=5,HMAT_MAX_STAGES_E=2" \
  "HMAT_CTAS_PER_SM=3" "HMAT_CTAS_PER_SM=3,HMAT_STAGE_KB=16,HMAT_MAX_STAGES=3" "HMAT_CTAS_PER_SM=4" > gpurun_out/sweep2_c4.log 2>&1; echo "c4 rc=$?"
timeout 600 python scripts/kernel_sweep.py c3 "" "HMAT_MAX_STAGES_E=2" "HMAT_CTAS_PER_SM=3" "HMAT_STAGE_KB=48,HMAT_MAX_STAGES_E=2" > gpurun_out/sweep2_c3.log 2>&1; echo "c3 rc=$?"

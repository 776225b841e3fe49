#!/bin/bash
# A/B of the 16-wide tensor-core pass geometry (project CTAs per SM / ring depth,
# expand CTAs per SM) at c2 and c4 with 16 rhs; settings alternate, twice.
set -u
mkdir -p gpurun_out
S=("NRHS=16" "NRHS=16,HMAT_DMMA16_CTAS=3,HMAT_DMMA16_STAGES=4" "NRHS=16,HMAT_DMMA16_CTAS=2,HMAT_DMMA16_STAGES=6"
   "NRHS=16,HMAT_DMMA_E_CTAS=1,HMAT_DMMA_STAGES_E=6" "NRHS=16,HMAT_DMMA_E_CTAS=3")
for rep in 1 2; do
  timeout 600 python scripts/kernel_sweep.py c2 "${S[@]/#/WARM=20,REPS=20,}" 2>&1 | tee -a gpurun_out/sweep16_c2.log
  timeout 900 python scripts/kernel_sweep.py c4 "${S[@]/#/WARM=60,REPS=10,}" 2>&1 | tee -a gpurun_out/sweep16_c4.log
done

#!/bin/bash
# c2 mid-rhs project knobs (8- and 16-wide tensor-core passes): level-interleave chunk,
# CTAs per SM, ring depth -- are the c4-tuned defaults right for the small operator?
set -u
mkdir -p gpurun_out
P=scripts/kernel_sweep.py
for rep in 1 2; do
  timeout 600 python $P c2 "WARM=20,REPS=20,NRHS=8" "WARM=20,REPS=20,NRHS=8,HMAT_DMMA_PCHUNK=0" "WARM=20,REPS=20,NRHS=8,HMAT_DMMA_PCHUNK=64" \
    "WARM=20,REPS=20,NRHS=8,HMAT_DMMA8_CTAS=4" "WARM=20,REPS=20,NRHS=8,HMAT_DMMA8_CTAS=6" "WARM=20,REPS=20,NRHS=8,HMAT_DMMA8_STAGES=4" \
    "WARM=20,REPS=20,NRHS=4" "WARM=20,REPS=20,NRHS=4,HMAT_DMMA_PCHUNK=0" "WARM=20,REPS=20,NRHS=4,HMAT_DMMA8_CTAS=6" \
    "WARM=20,REPS=20,NRHS=16" "WARM=20,REPS=20,NRHS=16,HMAT_DMMA_PCHUNK16=0" "WARM=20,REPS=20,NRHS=16,HMAT_DMMA_PCHUNK16=8" \
    "WARM=20,REPS=20,NRHS=16,HMAT_DMMA_PCHUNK16=32" 2>&1 | sed -e "s/Rp=.*grid=[0-9\/]* | //" | tee -a gpurun_out/sweep_c2mid.log
done

#!/bin/bash
set -u
mkdir -p gpurun_out
S="WARM=20,REPS=10"
timeout 900 python scripts/kernel_sweep.py c4 "$S,NRHS=8" "$S,NRHS=8,HMAT_DMMA_STAGES_E=4" "$S,NRHS=8,HMAT_DMMA_STAGES_E=2" "$S,NRHS=16,HMAT_DMMA_STAGES_E=4" "$S,NRHS=16" > gpurun_out/stagese.log 2>&1
timeout 900 python scripts/kernel_sweep.py c3 "WARM=50,REPS=20,NRHS=8" "WARM=50,REPS=20,NRHS=8,HMAT_DMMA_STAGES_E=5" "WARM=50,REPS=20,NRHS=8,HMAT_DMMA_STAGES_E=4" "WARM=50,REPS=20,NRHS=16,HMAT_DMMA_STAGES_E=5" >> gpurun_out/stagese.log 2>&1
timeout 900 python scripts/kernel_sweep.py c2 "WARM=100,REPS=50,NRHS=8" "WARM=100,REPS=50,NRHS=8,HMAT_DMMA_STAGES_E=4" "WARM=100,REPS=50,NRHS=4" "WARM=100,REPS=50,NRHS=16" >> gpurun_out/stagese.log 2>&1
cat gpurun_out/stagese.log

#!/bin/bash
set -u
mkdir -p gpurun_out
S="WARM=150,REPS=40"
timeout 900 python scripts/kernel_sweep.py c4 "$S" "$S,HMAT_MAX_STAGES_P=2" "$S" "$S,NRHS=2" "$S,NRHS=2,HMAT_MAX_STAGES_P=2" "$S,NRHS=4" "$S,NRHS=4,HMAT_MAX_STAGES_P=2" "WARM=20,REPS=10,NRHS=8" "WARM=20,REPS=10,NRHS=16" > gpurun_out/ab5.log 2>&1
timeout 900 python scripts/kernel_sweep.py c2 "WARM=500,REPS=100,NRHS=8" "WARM=500,REPS=100,NRHS=4" "WARM=500,REPS=100,NRHS=2" >> gpurun_out/ab5.log 2>&1
cat gpurun_out/ab5.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/pytest_ab5.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab5.log

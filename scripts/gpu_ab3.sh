#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_standard.py tests/test_gpu_random_shapes.py tests/test_gpu_bounds.py -m gpu -x -q > gpurun_out/pytest_ab3.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_ab3.log
S="WARM=150,REPS=40,HMAT_MAX_STAGES_P=3"
timeout 900 python scripts/kernel_sweep.py c4 "$S" "$S,HMAT_PROJECT_AFLUSH=0" "$S" "$S,HMAT_PROJECT_AFLUSH=0" "WARM=150,REPS=40" > gpurun_out/ab3.log 2>&1
timeout 900 python scripts/kernel_sweep.py c2 "WARM=500,REPS=100" "WARM=500,REPS=100,HMAT_PROJECT_AFLUSH=0" "WARM=500,REPS=100,HMAT_MAX_STAGES_P=3" >> gpurun_out/ab3.log 2>&1
timeout 900 python scripts/kernel_sweep.py c3 "WARM=100,REPS=40" "WARM=100,REPS=40,HMAT_PROJECT_AFLUSH=0" "WARM=100,REPS=40,HMAT_MAX_STAGES_P=3" >> gpurun_out/ab3.log 2>&1
cat gpurun_out/ab3.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/pytest_full.log 2>&1; echo "pytest full rc=$?"; tail -3 gpurun_out/pytest_full.log

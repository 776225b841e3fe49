#!/bin/bash
set -u
mkdir -p gpurun_out
S="WARM=150,REPS=40"
timeout 900 python scripts/kernel_sweep.py c4 "$S" "$S,HMAT_MAX_STAGES_P=3" "$S,HMAT_MAX_STAGES_P=3,HMAT_PROJECT_AFLUSH=0" "$S,HMAT_PROJECT_AFLUSH=0" "$S,HMAT_MAX_STAGES_P=3,HMAT_DEBUG_SKIP=4" "$S" > gpurun_out/ab4.log 2>&1
timeout 900 python scripts/kernel_sweep.py c3 "WARM=100,REPS=40" "WARM=100,REPS=40,HMAT_MAX_STAGES_P=3" "WARM=100,REPS=40,HMAT_PROJECT_EARLY=0" >> gpurun_out/ab4.log 2>&1
timeout 900 python scripts/kernel_sweep.py c2 "WARM=500,REPS=100" "WARM=500,REPS=100,HMAT_MAX_STAGES_P=3" >> gpurun_out/ab4.log 2>&1
cat gpurun_out/ab4.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py tests/test_gpu_random_shapes.py -m gpu -x -q > gpurun_out/pytest_ab4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab4.log

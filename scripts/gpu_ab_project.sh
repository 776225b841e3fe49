#!/bin/bash
# A/B of project-kernel variants on c4 under the sustained power cap (WARM matvecs first).
set -u
mkdir -p gpurun_out
S="WARM=150,REPS=40"
timeout 900 python scripts/kernel_sweep.py c4 "$S" "$S,HMAT_PROJECT_EARLY=0" "$S" "$S,HMAT_PROJECT_EARLY=0" \
  "$S,HMAT_MAX_STAGES_P=3" "$S,HMAT_PROJECT_EARLY=0,HMAT_MAX_STAGES_P=3" "$S,HMAT_STAGE_KB=16,HMAT_MAX_STAGES_P=3" \
  "$S,HMAT_STAGE_KB=16,HMAT_MAX_STAGES_P=4" "WARM=3,REPS=10" "WARM=3,REPS=10,HMAT_PROJECT_EARLY=0" > gpurun_out/ab_project.log 2>&1
echo "sweep rc=$?"; cat gpurun_out/ab_project.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -x -q -k "c4 or c3 or c2 or random or level or host_io" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab.log

set -u
mkdir -p gpurun_out
(WARM=150 timeout 600 python scripts/level_profile.py c4; echo "--- DYN=0"; HMAT_PROJECT_DYN=0 WARM=150 timeout 600 python scripts/level_profile.py c4) > gpurun_out/levels_c4.log 2>&1
S="WARM=150,REPS=40,HMAT_MAX_STAGES_P=3"
timeout 600 python scripts/kernel_sweep.py c4 "$S" "$S,HMAT_PROJECT_DYN=0" "$S,HMAT_PROJECT_SNAKE=0" "$S,HMAT_CTAS_PER_SM=1,HMAT_MAX_STAGES_P=6" >> gpurun_out/levels_c4.log 2>&1
cat gpurun_out/levels_c4.log
timeout 900 python -m pytest tests/test_gpu_standard.py -m gpu -x -q > gpurun_out/pytest_std.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_std.log

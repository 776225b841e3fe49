#!/bin/bash
set -u
mkdir -p gpurun_out
S="WARM=150,REPS=40,HMAT_MAX_STAGES_P=3"
timeout 900 python scripts/kernel_sweep.py c4 "$S" "$S,HMAT_PROJECT_CHUNK=16" "$S,HMAT_PROJECT_CHUNK=64" "$S" "$S,HMAT_PROJECT_CHUNK=16" > gpurun_out/ab2.log 2>&1
S5="WARM=20,REPS=20"
timeout 900 python scripts/kernel_sweep.py c5 "$S5" "$S5,HMAT_DMMA_ILEAVE=0" "$S5" "$S5,HMAT_DMMA_ILEAVE=0" >> gpurun_out/ab2.log 2>&1
cat gpurun_out/ab2.log
for v in 1 0; do
HMAT_DMMA_ILEAVE=$v timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"dmma" -s 2 -c 2 --csv python scripts/kernel_sweep.py c5 "" > gpurun_out/ncu_c5_ileave$v.csv 2>&1
echo "ncu ileave=$v rc=$?"; grep -E "dram__bytes|duration" gpurun_out/ncu_c5_ileave$v.csv | cut -c1-300
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "dmma or c5 or c4" > gpurun_out/pytest_ab2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab2.log

#!/bin/bash
# Mid-rhs diagnostics: full ncu captures of the c4 8-rhs (16-wide DMMA) and 4-rhs
# (SIMT) kernels, and the c5 U-box L2 policy A/B.
set -u
mkdir -p gpurun_out
timeout 600 python scripts/kernel_sweep.py c5 "WARM=20,REPS=20" "WARM=20,REPS=20,HMAT_DMMA_UPOL=1" "WARM=20,REPS=20" "WARM=20,REPS=20,HMAT_DMMA_UPOL=1" > gpurun_out/midrhs.log 2>&1
HMAT_DMMA_UPOL=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"expand_dmma" -s 1 -c 1 --csv python scripts/kernel_sweep.py c5 "" > gpurun_out/ncu_c5_upol1.csv 2>&1
grep -E "dram__bytes_read" gpurun_out/ncu_c5_upol1.csv | cut -c1-250 >> gpurun_out/midrhs.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dmma" -s 2 -c 2 -o gpurun_out/prof_c4n8 python scripts/kernel_sweep.py c4 "NRHS=8,REPS=2" > gpurun_out/ncu_c4n8.log 2>&1; echo "ncu c4n8 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"project_kernel|expand_kernel" -s 2 -c 2 -o gpurun_out/prof_c4n4 python scripts/kernel_sweep.py c4 "NRHS=4,REPS=2" > gpurun_out/ncu_c4n4.log 2>&1; echo "ncu c4n4 rc=$?"
cat gpurun_out/midrhs.log

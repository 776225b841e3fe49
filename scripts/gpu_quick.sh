#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_shapes.py -x -q -k "multi_rhs or small or random or gemv or strict or async" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"
timeout 900 python scripts/kernel_sweep.py c2 "" "NRHS=2" "NRHS=2,HMAT_EXPAND_RPT=0" "NRHS=4" "NRHS=4,HMAT_EXPAND_RPT=0" "NRHS=8" > gpurun_out/quick_sweep.log 2>&1
timeout 900 python scripts/kernel_sweep.py c3 "" "NRHS=2" "NRHS=2,HMAT_EXPAND_RPT=0" "NRHS=4" "NRHS=4,HMAT_EXPAND_RPT=0" >> gpurun_out/quick_sweep.log 2>&1
timeout 900 python scripts/kernel_sweep.py c4 "" >> gpurun_out/quick_sweep.log 2>&1

#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python scripts/kernel_sweep.py c4 "" "HMAT_DEBUG_SKIP=4" "HMAT_DEBUG_SKIP=8" "HMAT_DEBUG_SKIP=1" > gpurun_out/diag3_c4.log 2>&1; echo "rc=$?"
timeout 900 python scripts/kernel_sweep.py c3 "" c2 > gpurun_out/diag3_c3.log 2>&1; echo "rc=$?"
timeout 900 python scripts/kernel_sweep.py c2 "" > gpurun_out/diag3_c2.log 2>&1; echo "rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?"

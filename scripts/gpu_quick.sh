#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_random_shapes.py -x -q -k "dmma or DMMA or random or adjoint" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"
timeout 900 python scripts/kernel_sweep.py c2 "NRHS=64" "NRHS=64,HMAT_DMMA_NW=16" > gpurun_out/quick_sweep.log 2>&1
timeout 900 python scripts/kernel_sweep.py c5 "" >> gpurun_out/quick_sweep.log 2>&1

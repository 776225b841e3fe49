#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_standard.py tests/test_gpu_multirank.py tests/test_gpu_random_shapes.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"
timeout 900 python scripts/kernel_sweep.py s2 "" "" > gpurun_out/quick_sweep.log 2>&1
timeout 900 python scripts/kernel_sweep.py c4 "" >> gpurun_out/quick_sweep.log 2>&1

#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_standard.py tests/test_gpu_multirank.py -x -q > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"
timeout 900 python scripts/kernel_sweep.py c4 "" "" > gpurun_out/quick_sweep.log 2>&1
for c in c2 c3 c2strict; do timeout 300 python scripts/kernel_sweep.py $c "" >> gpurun_out/quick_sweep.log 2>&1; done

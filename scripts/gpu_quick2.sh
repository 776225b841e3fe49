#!/bin/bash
set -u
mkdir -p gpurun_out
HMAT_EXPAND_CHUNK=1 timeout 900 python -m pytest tests/test_gpu_standard.py tests/test_gpu_multirank.py -x -q > gpurun_out/pytest_chunk1.log 2>&1; echo "pytest rc=$?"
HMAT_EXPAND_CHUNK=1 timeout 300 python scripts/cta_trace.py s2 > gpurun_out/trace_s2_chunk1.log 2>&1
timeout 300 python scripts/cta_trace.py s2 > gpurun_out/trace_s2_static.log 2>&1

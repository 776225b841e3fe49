#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "dmma or DMMA or multirank or adjoint or gemv" > gpurun_out/pytest_dmma.log 2>&1; echo "pytest rc=$?"
timeout 900 python scripts/kernel_sweep.py c5 "" "HMAT_DMMA_KR=16,HMAT_DMMA_STAGES_P=4" > gpurun_out/sweep_c5.log 2>&1; echo "c5 rc=$?"

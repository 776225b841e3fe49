#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_peer_ipc.py tests/test_abi.py -m gpu -x -q > gpurun_out/pytest_nb8.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_nb8.log
S="WARM=20,REPS=10"
timeout 900 python scripts/kernel_sweep.py c4 "$S,NRHS=8" "$S,NRHS=8,HMAT_DMMA_NARROW=2" "$S,NRHS=5" "$S,NRHS=4" "$S,NRHS=4,HMAT_DMMA_MIN=3" "$S,NRHS=3" "$S,NRHS=3,HMAT_DMMA_MIN=3" "$S,NRHS=2,HMAT_DMMA_MIN=2" > gpurun_out/nb8.log 2>&1
timeout 900 python scripts/kernel_sweep.py c2 "WARM=100,REPS=50,NRHS=8" "WARM=100,REPS=50,NRHS=4" "WARM=100,REPS=50,NRHS=4,HMAT_DMMA_MIN=3" "WARM=100,REPS=50,NRHS=3,HMAT_DMMA_MIN=3" >> gpurun_out/nb8.log 2>&1
timeout 900 python scripts/kernel_sweep.py c3 "WARM=50,REPS=20,NRHS=8" "WARM=50,REPS=20,NRHS=4" "WARM=50,REPS=20,NRHS=4,HMAT_DMMA_MIN=3" >> gpurun_out/nb8.log 2>&1
cat gpurun_out/nb8.log

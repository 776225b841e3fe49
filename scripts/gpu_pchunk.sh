#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_peer_ipc.py tests/test_gpu_random_shapes.py -m gpu -x -q -k "dmma or sharded or peer or random or pdmma or ipc" > gpurun_out/pytest_pchunk.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_pchunk.log
S="WARM=20,REPS=10"
timeout 900 python scripts/kernel_sweep.py c4 "$S,NRHS=8" "$S,NRHS=8,HMAT_DMMA_PCHUNK=0" "$S,NRHS=8,HMAT_DMMA_PCHUNK=16" "$S,NRHS=8,HMAT_DMMA_PCHUNK=64" "$S,NRHS=16" "$S,NRHS=16,HMAT_DMMA_PCHUNK=0" "$S,NRHS=4" > gpurun_out/pchunk.log 2>&1
timeout 900 python scripts/kernel_sweep.py c3 "WARM=50,REPS=20,NRHS=8" "WARM=50,REPS=20,NRHS=8,HMAT_DMMA_PCHUNK=0" "WARM=50,REPS=20,NRHS=16" >> gpurun_out/pchunk.log 2>&1
timeout 900 python scripts/kernel_sweep.py c2 "WARM=100,REPS=50,NRHS=8" "WARM=100,REPS=50,NRHS=8,HMAT_DMMA_PCHUNK=0" >> gpurun_out/pchunk.log 2>&1
cat gpurun_out/pchunk.log

#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python scripts/kernel_sweep.py c3 "NRHS=4" "NRHS=8" "NRHS=8,HMAT_MAX_NR=4" "NRHS=8,HMAT_MAX_NR=2" "NRHS=6" "NRHS=6,HMAT_MAX_NR=4" "NRHS=3" "NRHS=3,HMAT_MAX_NR=2" > gpurun_out/nrhs_sweep.log 2>&1
timeout 900 python scripts/kernel_sweep.py c2 "NRHS=4" "NRHS=8" "NRHS=8,HMAT_MAX_NR=4" "NRHS=8,HMAT_MAX_NR=2" "NRHS=16,HMAT_MAX_NR=4" "NRHS=4,HMAT_MAX_NR=2" >> gpurun_out/nrhs_sweep.log 2>&1

#!/bin/bash
# A/B of the 16-wide tensor-core expand's CTAs per SM (HMAT_DMMA_E_CTAS: 2 = the
# round-2 geometry, default 3) on every 16-rhs shape; the tensor-core tests.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_standard.py tests/test_gpu_multirank.py -m gpu -x -q -k "dmma or rhs or many" -p no:cacheprovider > gpurun_out/ectas_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ectas_pytest.log
for rep in 1 2; do
  for c in c2 c3 c4 s2; do
    W=20; [ $c = c4 ] && W=60
    timeout 600 python scripts/kernel_sweep.py $c "WARM=$W,REPS=10,NRHS=16" "WARM=$W,REPS=10,NRHS=16,HMAT_DMMA_E_CTAS=2" 2>&1 | sed -e "s/Rp=.*grid=[0-9\/]* | //" | tee -a gpurun_out/ab_ectas.log
  done
done

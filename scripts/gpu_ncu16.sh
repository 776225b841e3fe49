#!/bin/bash
# Full ncu captures of the 16-wide tensor-core kernels (c2 and c4 with 16 rhs),
# for the shared-memory and tensor-pipe breakdown of the mid-rhs regime.
set -u
mkdir -p gpurun_out
for spec in ${SPECS:-"c2 16 c2_16rhs" "c4 16 c4_16rhs"}; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dmma" -s 2 -c 2 -o gpurun_out/prof_$3_full \
    python scripts/kernel_sweep.py $1 "WARM=1,REPS=1,NRHS=$2${EXTRA:+,$EXTRA}" > gpurun_out/ncu_$3.log 2>&1; echo "ncu $3 rc=$?"
done

#!/bin/bash
# bench lines of the mid-rhs configs, and full ncu captures of their tensor-core
# kernels (c4 with 8 and 16 rhs, s2 with 16)
set -u
mkdir -p gpurun_out
for c in c2r2 c2r4 c2r8 c2r16 c4r2 c4r4 c4r8 c4r16 s2r16; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
for spec in "c4 8 c4_8rhs" "c4 16 c4_16rhs" "s2 16 s2_16rhs"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dmma" -s 2 -c 2 -o gpurun_out/prof_$3_full \
    python scripts/kernel_sweep.py $1 "WARM=1,REPS=1,NRHS=$2" > gpurun_out/ncu_$3.log 2>&1; echo "ncu $3 rc=$?"
done

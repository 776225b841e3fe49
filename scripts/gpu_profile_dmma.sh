#!/bin/bash
# bench lines for c5 / c3 / c2 and a full ncu capture of the DMMA kernels (a 1/8-size c5 shape)
set -u
mkdir -p gpurun_out
for c in c5 c3 c2; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
S="d=3,L=4,b=64,r=32,nrhs=64"
timeout 300 python scripts/kernel_sweep.py $S "" > gpurun_out/plain_dmma.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dmma" -s 6 -c 2 -o gpurun_out/prof_dmma python scripts/kernel_sweep.py $S "" > gpurun_out/ncu_dmma.log 2>&1
echo "ncu dmma rc=$?"

#!/bin/bash
# bench lines of the mid-rhs configs only
set -u
mkdir -p gpurun_out
for c in c2r2 c2r4 c2r8 c2r16 c4r2 c4r4 c4r8 c4r16 s2r16; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done

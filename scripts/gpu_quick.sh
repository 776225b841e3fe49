#!/bin/bash
# Quick GPU check: the tests named in $TESTS (default: all -m gpu), then bench lines of $CFGS.
set -u
mkdir -p gpurun_out
TESTS=${TESTS:-tests}
CFGS=${CFGS:-c4}
timeout 1500 python -m pytest $TESTS -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_quick.log
for c in $CFGS; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
  tail -3 gpurun_out/bench_$c.err
done

#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c1_small.json 2>/dev/null; echo "bench rc=$?"
HMAT_SMALL=0 timeout 600 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c1_stream.json 2>/dev/null

#!/bin/bash
# GPU tests, bench lines (c4 default, c5), launch list of the c4 bench, full ncu of the c5 DMMA kernels
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc=$?"
timeout 900 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain_bench.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
timeout 300 python scripts/kernel_sweep.py c5 "" > gpurun_out/plain_c5.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dmma" -s 2 -c 2 -o gpurun_out/prof_c5_full python scripts/kernel_sweep.py c5 "" > gpurun_out/ncu_c5.log 2>&1
echo "ncu c5 rc=$?"

#!/bin/bash
# One gpurun call: bench line, ncu launch list of the bench command, dram traffic of
# the C4 kernels, full ncu capture of the C2 kernels.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain_bench.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"project_kernel|expand_kernel" -s 4 -c 2 --csv --log-file gpurun_out/traffic_c4.csv python scripts/kernel_sweep.py c4 "" > gpurun_out/ncu_traffic.log 2>&1
echo "traffic rc=$?"
timeout 300 python scripts/kernel_sweep.py c2 "" > gpurun_out/plain_c2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"project_kernel|expand_kernel" -s 6 -c 2 -o gpurun_out/prof_c2_full python scripts/kernel_sweep.py c2 "" > gpurun_out/ncu_c2.log 2>&1
echo "full c2 rc=$?"

#!/bin/bash
# read-only HBM ceiling probe + DRAM traffic of the c5 (DMMA) kernels
set -u
mkdir -p gpurun_out
timeout 300 ./scripts/hbm_read_peak > gpurun_out/hbm_read_peak.txt 2>&1; echo "probe rc=$?"
timeout 300 python scripts/kernel_sweep.py c5 "" > gpurun_out/plain_c5.log 2>&1 && \
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"dmma" -s 4 -c 2 --csv --log-file gpurun_out/traffic_c5.csv python scripts/kernel_sweep.py c5 "" > gpurun_out/ncu_traffic_c5.log 2>&1
echo "traffic rc=$?"

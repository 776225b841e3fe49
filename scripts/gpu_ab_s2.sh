#!/bin/bash
set -u
mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python scripts/kernel_sweep.py s2 "" >> gpurun_out/ab_s2b.log 2>&1
(cd _ab_old && timeout 300 python scripts/kernel_sweep.py s2 "" | sed 's/^/OLD /') >> gpurun_out/ab_s2b.log 2>&1
done

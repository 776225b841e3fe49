#!/bin/bash
# full ncu capture of the c4 single-rhs kernels and of the probe's best bulk ring
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"project_kernel|expand_kernel" -s 2 -c 2 -o gpurun_out/prof_c4_full python scripts/kernel_sweep.py c4 "" > gpurun_out/ncu_c4.log 2>&1
echo "ncu c4 rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:"bulk_ring" -s 0 -c 1 -o gpurun_out/prof_probe python - <<'PY' > gpurun_out/ncu_probe.log 2>&1
import subprocess; subprocess.run(["./scripts/hbm_read_peak", "rnd"])
PY
echo "ncu probe rc=$?"

#!/bin/bash
# A/B of the project kernel's per-level stream direction (HMAT_PROJECT_SNAKE).
set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_standard.py tests/test_gpu_bounds.py -x -q 2>&1 | tail -3
python scripts/kernel_sweep.py c4 "HMAT_PROJECT_SNAKE=0" "" "HMAT_PROJECT_SNAKE=0" "" 2>&1 | grep -v Warn
for s in 0 1 0 1; do
  HMAT_PROJECT_SNAKE=$s python bench.py --steps 30 --warmup 5 > gpurun_out/ab_snake_$s.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_snake_$s.json'));print('snake=$s', round(d['value'],2), d['phase_ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:project_kernel -c 1 \
  python scripts/kernel_sweep.py c4 "" 2>&1 | grep -E "dram__bytes_read|gpu__time_duration" | head -4

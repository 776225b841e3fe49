#!/bin/bash
# c4 diagnosis: per-CTA trace and per-level timing of the single-rhs kernels
set -u
mkdir -p gpurun_out
timeout 600 python scripts/cta_trace.py c4 c3 > gpurun_out/cta_trace_c4.log 2>&1; echo "trace rc=$?"
timeout 600 python scripts/level_profile.py c4 > gpurun_out/level_c4.log 2>&1; echo "level rc=$?"

#!/bin/bash
# Round-end evidence: GPU tests, smoke, bench lines of every config, the FP64 peak
# probe, the c4 launch list and DRAM traffic, full ncu captures of the c2 / c4
# single-rhs kernels and the c5 DMMA kernels.  Then (here, on CPU):
#   python scripts/summarize_profiles.py r02 && python scripts/summary_table.py r02
set -u
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_c4.json 2> gpurun_out/bench_ref_c4.err; echo "ref c4 rc=$?"
for c in c5 c1 c2 c3 s2 c2strict c2r2 c2r4 c2r8 c2r16 c4r2 c4r4 c4r8 c4r16 s2r16; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
(cd scripts && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak) > gpurun_out/fp64_peak.txt 2>&1; echo "fp64 rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain_bench.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"project_kernel|expand_kernel" -s 4 -c 2 --csv --log-file gpurun_out/traffic_c4.csv python scripts/kernel_sweep.py c4 "" > gpurun_out/ncu_traffic.log 2>&1
echo "traffic rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"project_kernel|expand_kernel" -s 6 -c 2 -o gpurun_out/prof_c2_full python scripts/kernel_sweep.py c2 "" > gpurun_out/ncu_c2.log 2>&1
echo "full c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dmma" -s 2 -c 2 -o gpurun_out/prof_c5_full python scripts/kernel_sweep.py c5 "" > gpurun_out/ncu_c5.log 2>&1
echo "ncu c5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"project_kernel|expand_kernel" -s 4 -c 2 -o gpurun_out/prof_c4_full python scripts/kernel_sweep.py c4 "" > gpurun_out/ncu_c4.log 2>&1
echo "full c4 rc=$?"

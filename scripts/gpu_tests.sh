set -u
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt; free -g > gpurun_out/free.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -45 gpurun_out/pytest_gpu.log

#!/bin/bash
# usage: gpu_quick.sh "<pytest -k expr or file list>" [bench args]
mkdir -p gpurun_out
timeout 1200 python -m pytest ${1:-tests} -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
if [ -n "$2" ]; then timeout 900 python bench.py $2 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log; fi
tail -n 5 gpurun_out/pytest_gpu.log; tail -n 3 gpurun_out/bench.log 2>/dev/null | cut -c1-3000

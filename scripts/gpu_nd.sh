#!/bin/bash
# ND-sort parity + timing on the box
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_ndsort.py tests/test_gpu_nsga3.py tests/test_gpu_hype.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_nd.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_nd.log
timeout 300 python scripts/time_ndsort.py 20000 100000 400000 > gpurun_out/time_nd.log 2>&1
MS=2,3 timeout 300 python scripts/time_ndsort.py 500000 >> gpurun_out/time_nd.log 2>&1
tail -n 15 gpurun_out/pytest_nd.log; cat gpurun_out/time_nd.log | cut -c1-600
python scripts/stair_prof.py 400000 3 0; python scripts/stair_prof.py 400000 3 127; python scripts/stair_prof.py 400000 3 195

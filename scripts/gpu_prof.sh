#!/bin/bash
# ncu captures: launch list of one bench generation + full sets of the top kernels.
mkdir -p gpurun_out
bash scripts/build_drivers.sh
# launch list of one generation (warmup 1 step + 1 step, no cpu baseline)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
# full sets
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_offspring -s 1 -c 1 \
    -o gpurun_out/prof_offspring -f scripts/offspring_driver 200000 1000 2 > gpurun_out/prof_offspring.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dom_rows -s 0 -c 1 \
    -o gpurun_out/prof_k1 -f scripts/rank_driver 400000 3 1 1 > gpurun_out/prof_k1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_peel -s 0 -c 1 \
    -o gpurun_out/prof_peel -f scripts/rank_driver 400000 3 1 1 > gpurun_out/prof_peel.log 2>&1
ls -la gpurun_out

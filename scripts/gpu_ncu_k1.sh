#!/bin/bash
mkdir -p gpurun_out
bash scripts/build_drivers.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dom_packed -s 0 -c 1 \
    -o gpurun_out/prof_k1p -f scripts/rank_driver 400000 3 1 1 > gpurun_out/prof_k1p.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rank.csv \
    scripts/rank_driver 400000 3 1 2 > gpurun_out/launches_rank.log 2>&1
tail -n 3 gpurun_out/prof_k1p.log

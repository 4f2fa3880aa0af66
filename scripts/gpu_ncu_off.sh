#!/bin/bash
mkdir -p gpurun_out
bash scripts/build_drivers.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_offspring -s 1 -c 1 \
    -o gpurun_out/prof_offs -f scripts/offspring_driver 100000 1000 2 > gpurun_out/prof_offs.log 2>&1
tail -n 3 gpurun_out/prof_offs.log

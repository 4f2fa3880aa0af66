#!/bin/bash
# usage: gpu_ncu.sh NAME KERNEL_REGEX SKIP -- cmd...   (ncu --set full; text summaries written next to the report)
name=$1; kre=$2; skip=$3; shift 4
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 \
    -o gpurun_out/$name -f "$@" > gpurun_out/$name.log 2>&1
python scripts/ncu_summary.py gpurun_out/$name.ncu-rep > gpurun_out/$name.summary.txt 2>&1
python scripts/ncu_lines.py gpurun_out/$name.ncu-rep 60 > gpurun_out/$name.lines.txt 2>&1
python scripts/ncu_sass.py gpurun_out/$name.ncu-rep 40 > gpurun_out/$name.sass.txt 2>&1
sz=$(stat -c %s gpurun_out/$name.ncu-rep 2>/dev/null || echo 0)
if [ "$sz" -gt 40000000 ]; then rm -f gpurun_out/$name.ncu-rep; fi

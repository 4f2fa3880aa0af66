#!/bin/bash
# cap1.sh NAME REGEX SKIP [bench args...]: one full ncu capture of a kernel launched by bench.py,
# summarised into gpurun_out/cap/NAME.txt (metrics + hottest source lines)
mkdir -p gpurun_out/cap
cd "$(dirname "$0")/.."
export TEMO_BENCH_NO_PROFILER=1
name=$1 rx=$2 skip=$3; shift 3
timeout ${CAP_TIMEOUT:-400} ncu --set full --clock-control none --import-source on -k "regex:$rx" -s $skip -c 1 \
    -o gpurun_out/cap/$name -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline "$@" \
    > gpurun_out/cap/$name.log 2>&1
python scripts/ncu_summary.py gpurun_out/cap/$name.ncu-rep > gpurun_out/cap/$name.txt 2>&1
python scripts/ncu_lines.py gpurun_out/cap/$name.ncu-rep 30 >> gpurun_out/cap/$name.txt 2>&1
rm -f gpurun_out/cap/$name.ncu-rep

#!/bin/bash
# launch list (device time per kernel) of a short bench run, plus the per-kernel summary
mkdir -p gpurun_out
POP=${POP:-200000}
TEMO_BENCH_NO_PROFILER=1 timeout 600 ncu --target-processes application-only --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_pop$POP.csv python bench.py --pop $POP --steps 1 --warmup 1 --no-cpu-baseline \
    > gpurun_out/launches_pop$POP.log 2>&1
echo "ncu rc=$?" >> gpurun_out/launches_pop$POP.log
python scripts/launch_summary.py gpurun_out/launches_pop$POP.csv > gpurun_out/launches_pop$POP.summary.txt 2>&1

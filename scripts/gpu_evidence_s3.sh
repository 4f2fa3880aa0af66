#!/bin/bash
# Round-2 session-3 evidence: smoke, full GPU tests, every config's bench line, launch list of the
# headline, full ncu captures of the kernels that changed (randomness units, K0 sorts).
mkdir -p gpurun_out/${EVDIR:-p3}
cd "$(dirname "$0")/.."
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${EVDIR:-p3}/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${EVDIR:-p3}/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${EVDIR:-p3}/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${EVDIR:-p3}/pytest_gpu.log
: > gpurun_out/${EVDIR:-p3}/bench_lines.jsonl
for args in "--config D" "--config A" "--config B" "--config C" "--config E" "--config E --objectives 6" "--config E --objectives 10 --pop 200000" "--config E --objectives 4"; do
  extra="--no-cpu-baseline"; [ "$args" = "--config D" ] && extra=""
  timeout 900 python bench.py $args --steps 10 --warmup 3 $extra > gpurun_out/${EVDIR:-p3}/bench.log 2>&1
  grep '^{' gpurun_out/${EVDIR:-p3}/bench.log >> gpurun_out/${EVDIR:-p3}/bench_lines.jsonl
done
export TEMO_BENCH_NO_PROFILER=1
timeout 900 ncu --target-processes application-only --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${EVDIR:-p3}/launches_D.csv python bench.py --config D --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/${EVDIR:-p3}/launches_D.log 2>&1
python scripts/launch_summary.py gpurun_out/${EVDIR:-p3}/launches_D.csv > gpurun_out/${EVDIR:-p3}/launches_D.summary.txt 2>&1
cap() {  # name regex skip bench-args...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$rx" -s $skip -c 1 \
      -o gpurun_out/${EVDIR:-p3}/$name -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline "$@" \
      > gpurun_out/${EVDIR:-p3}/$name.log 2>&1
  python scripts/ncu_summary.py gpurun_out/${EVDIR:-p3}/$name.ncu-rep > gpurun_out/${EVDIR:-p3}/$name.txt 2>&1
  python scripts/ncu_lines.py gpurun_out/${EVDIR:-p3}/$name.ncu-rep 25 >> gpurun_out/${EVDIR:-p3}/$name.txt 2>&1
  rm -f gpurun_out/${EVDIR:-p3}/$name.ncu-rep
}
cap D_offspring_rand 'k_offspring_rand' 2 --config D
cap D_offspring_apply_v 'k_offspring_apply_v' 2 --config D
cap D_k0_sort 'DeviceRadixSortOnesweep' 6 --config D
tail -2 gpurun_out/${EVDIR:-p3}/smoke.log gpurun_out/${EVDIR:-p3}/pytest_gpu.log
cut -c1-200 gpurun_out/${EVDIR:-p3}/bench_lines.jsonl

#!/bin/bash
# Round-2 evidence: launch list of the headline bench, full ncu captures of the dominant kernels
# of every config, and the CPU reference timed at pop 10k on this host (for the baseline fit).
mkdir -p gpurun_out/p2
cd "$(dirname "$0")/.."
export TEMO_BENCH_NO_PROFILER=1
# 1) launch list, config D (pop 200k)
timeout 900 ncu --target-processes application-only --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/p2/launches_D.csv python bench.py --config D --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/p2/launches_D.log 2>&1
python scripts/launch_summary.py gpurun_out/p2/launches_D.csv > gpurun_out/p2/launches_D.summary.txt 2>&1
# 2) full captures (one launch each) of the dominant kernels
cap() {  # name regex skip bench-args...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$rx" -s $skip -c 1 \
      -o gpurun_out/p2/$name -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline "$@" \
      > gpurun_out/p2/$name.log 2>&1
  python scripts/ncu_summary.py gpurun_out/p2/$name.ncu-rep > gpurun_out/p2/$name.txt 2>&1
  python scripts/ncu_lines.py gpurun_out/p2/$name.ncu-rep 25 >> gpurun_out/p2/$name.txt 2>&1
  rm -f gpurun_out/p2/$name.ncu-rep
}
cap D_offspring_rand 'k_offspring_rand' 2 --config D
cap D_offspring_apply 'k_offspring_apply' 2 --config D
cap D_stair_peel 'k_st_peel' 2 --config D
cap D_k0_sort 'DeviceRadixSortOnesweep' 6 --config D
cap C_hv_dom 'k_hv_dom' 1 --config C
cap C_hv_partial 'k_hv_partial' 1 --config C
cap B_moead_elite 'k_moead_elite' 1 --config B
cap B_moead_offspring 'k_offspring' 1 --config B
cap E_stair_peel_m3 'k_st_peel' 1 --config E --pop 500000
cap E_dom_rows8_m4 'k_dom_rows8' 1 --config E --pop 500000 --objectives 4
cap E_dom_packed_m6 'k_dom_packed' 1 --config E --pop 500000 --objectives 6
cap E_dom_packed_m10 'k_dom_packed' 1 --config E --pop 200000 --objectives 10
# 3) bench lines of every config (no profiler) incl. E at m = 6, 10
: > gpurun_out/p2/bench_lines.jsonl
for args in "--config D" "--config A" "--config B" "--config C" "--config E" "--config E --objectives 6" "--config E --objectives 10 --pop 200000"; do
  timeout 900 python bench.py $args --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | grep '^{' >> gpurun_out/p2/bench_lines.jsonl
done
# 4) CPU reference (oracle port) measured at pop 2k, 5k, 10k on this host's cores
python - > gpurun_out/p2/cpu_fit.json 2>&1 <<'PY'
import json, os, sys, time
sys.path.insert(0, ".")
import bench
out = {"cores": os.cpu_count(), "points": []}
c = dict(bench.CONFIGS["D"])
for pop in (2000, 5000, 10000):
    t, _ = bench._oracle_run_step(c, pop)
    out["points"].append({"pop": pop, "s_per_gen": t})
    print(json.dumps(out), file=sys.stderr)
print(json.dumps(out))
PY
ls gpurun_out/p2

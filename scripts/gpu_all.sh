#!/bin/bash
# full GPU check: tests, then one bench line per config (default D with its CPU baseline)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
: > gpurun_out/bench_all.jsonl
for c in ${CONFIGS:-D A B C E}; do
  extra="--no-cpu-baseline"; [ "$c" = "D" ] && extra=""
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 $extra > gpurun_out/bench_$c.log 2>&1
  echo "bench $c rc=$?"; grep '^{' gpurun_out/bench_$c.log >> gpurun_out/bench_all.jsonl
done
python - <<'PY'
import json
for l in open("gpurun_out/bench_all.jsonl"):
    d = json.loads(l)
    print(d["metric"], "value=%.4g" % d["value"], "e2e=%.4g" % d["e2e"]["value"], "ms=%s" % d.get("ms_per_step"),
          "roof=%s" % (None if not d.get("roofline") else round(d["roofline"]["frac"], 3)),
          "comp=%s" % (None if not d.get("roofline_compute") else round(d["roofline_compute"]["frac"], 3)),
          "cpu=%s" % (d.get("cpu_baseline") or {}).get("value"))
    print("   stages", {k: round(v, 3) for k, v in d.get("stages_ms_per_step", {}).items()})
PY

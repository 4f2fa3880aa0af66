#!/bin/bash
# A/B of apply-kernel variants (varlib/*) against the in-tree build: bench D stage times
cd "$(dirname "$0")/.."
for lib in default ${VARIANTS:-$(ls varlib 2>/dev/null)}; do
  if [ "$lib" = default ]; then unset TEMO_LIB; else export TEMO_LIB=varlib/$lib/libtemo_b200.so; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms_per_step']
print('$lib', round(d['value'],2), 'apply', round(s['offspring_apply'],3), 'rand', round(s['offspring'],3), 'frac', round(d['roofline']['frac'],3))"
done

#!/bin/bash
# A/B of library variants (varlib/*) and env switches (env:VAR=VAL) against the in-tree build: bench D stage times
cd "$(dirname "$0")/.."
for lib in default ${VARIANTS:-$(ls varlib 2>/dev/null)}; do
  (
  if [[ "$lib" == env:* ]]; then for kv in ${lib#env:}; do :; done; IFS=, read -ra KV <<< "${lib#env:}"; for kv in "${KV[@]}"; do export "$kv"; done; elif [ "$lib" != default ]; then export TEMO_LIB=varlib/$lib/libtemo_b200.so; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms_per_step']
print('$lib', round(d['value'],2), 'e2e', round(d['e2e']['value'],2), {k: round(v,3) for k,v in s.items()})"
  )
done

#!/bin/bash
# A/B of the offspring-randomness overlap modes and grid caps (bench D stage times)
cd "$(dirname "$0")/.."
run() {
  env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms_per_step']
print('$*', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'ms', round(d['ms_per_step'],3), {k: round(v,3) for k,v in s.items()})"
}
run TEMO_OVERLAP_RAND=0
run TEMO_OVERLAP_RAND=2
run TEMO_OVERLAP_RAND=2 TEMO_APPLY_GRID_PER_SM=16 TEMO_RAND_GRID_PER_SM=1
run TEMO_OVERLAP_RAND=2 TEMO_APPLY_GRID_PER_SM=16 TEMO_RAND_GRID_PER_SM=2
run TEMO_OVERLAP_RAND=1 TEMO_RAND_GRID_PER_SM=1
run TEMO_OVERLAP_RAND=0 TEMO_APPLY_GRID_PER_SM=16

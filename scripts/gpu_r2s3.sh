#!/bin/bash
# session-3 check: smoke + full gpu tests + bench D + A/B variants
mkdir -p gpurun_out
bash scripts/gpu_check.sh
VARIANTS="${VARIANTS:-}" bash scripts/ab_apply.sh > gpurun_out/ab.txt 2>&1
cat gpurun_out/ab.txt

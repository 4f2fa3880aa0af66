#!/bin/bash
# Build the standalone C-ABI drivers used for ncu captures (no Python in the profiled process).
set -e
cd "$(dirname "$0")/.."
for d in rank_driver offspring_driver; do
  nvcc -O2 -Wno-deprecated-gpu-targets -I include scripts/$d.c -L paper_2503_20286_b200/_lib -ltemo_b200 \
       -Xlinker -rpath -Xlinker '$ORIGIN/../paper_2503_20286_b200/_lib' -o scripts/$d
done

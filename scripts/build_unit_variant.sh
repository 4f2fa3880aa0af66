#!/bin/bash
# build_unit_variant.sh NAME UNIT : libtemo_b200.so with one object (UNIT = variation | variation_m3 |
# ndsort_m3 ...) rebuilt with $FLAGS into varlib/NAME/ (load with TEMO_LIB=varlib/NAME/libtemo_b200.so)
set -e
cd "$(dirname "$0")/.."
name=$1; unit=$2
src=paper_2503_20286_b200/csrc/${unit%%_m*}.cu
monly=""; [[ "$unit" == *_m* ]] && monly="-DTEMO_M_ONLY=${unit##*_m}"
mkdir -p varlib/$name
nvcc $FLAGS $monly -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --fmad=false \
     -Xcompiler -fPIC -Xptxas -v -I include -I paper_2503_20286_b200/csrc \
     -c $src -o varlib/$name/$unit.o 2> varlib/$name/ptxas.txt
objs=$(ls paper_2503_20286_b200/_lib/*.o | grep -v "/$unit.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o varlib/$name/libtemo_b200.so $objs varlib/$name/$unit.o -lcudart
rm -f varlib/$name/*.o

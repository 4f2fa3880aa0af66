#!/bin/bash
# build_variant.sh NAME : libtemo_b200.so with the objective-count-3 unit of variation.cu rebuilt with
# $FLAGS (e.g. FLAGS="-DTMA_MINB=2") into exp/NAME/ (load it with TEMO_LIB=varlib/NAME/libtemo_b200.so; varlib/ travels with gpurun, keep at most two)
set -e
cd "$(dirname "$0")/.."
name=$1
mkdir -p varlib/$name
nvcc $FLAGS -DTEMO_M_ONLY=3 -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --fmad=false \
     -Xcompiler -fPIC -Xptxas -v -I include -I paper_2503_20286_b200/csrc \
     -c ${SRC:-paper_2503_20286_b200/csrc/variation.cu} -o varlib/$name/variation_m3.o 2> varlib/$name/ptxas.txt
objs=$(ls paper_2503_20286_b200/_lib/*.o | grep -v "variation_m3.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o varlib/$name/libtemo_b200.so $objs varlib/$name/variation_m3.o -lcudart
rm -f varlib/$name/*.o
grep -A2 "k_offspring_tmaILi3ELb1ELb1" varlib/$name/ptxas.txt | grep -E "registers|spill" | tr '\n' ' '; echo

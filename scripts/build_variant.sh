#!/bin/bash
# build_variant.sh NAME : libtemo_b200.so with the objective-count-3 unit of variation.cu rebuilt with
# $FLAGS (e.g. FLAGS="-DTMA_MINB=2") into exp/NAME/ (load it with TEMO_LIB=exp/NAME/libtemo_b200.so)
set -e
cd "$(dirname "$0")/.."
name=$1
mkdir -p exp/$name
nvcc $FLAGS -DTEMO_M_ONLY=3 -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --fmad=false \
     -Xcompiler -fPIC -Xptxas -v -I include -I paper_2503_20286_b200/csrc \
     -c ${SRC:-paper_2503_20286_b200/csrc/variation.cu} -o exp/$name/variation_m3.o 2> exp/$name/ptxas.txt
objs=$(ls paper_2503_20286_b200/_lib/*.o | grep -v "variation_m3.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp/$name/libtemo_b200.so $objs exp/$name/variation_m3.o -lcudart
rm -f exp/$name/*.o
grep -A2 "k_offspring_tmaILi3ELb1ELb1" exp/$name/ptxas.txt | grep -E "registers|spill" | tr '\n' ' '; echo

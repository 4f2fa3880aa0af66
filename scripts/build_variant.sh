#!/bin/bash
# build_variant.sh NAME "sed-expr" : libtemo_b200.so with variation.cu edited by sed-expr, into exp/NAME/
set -e
cd "$(dirname "$0")/.."
name=$1; expr=$2
mkdir -p exp/$name
sed "$expr" ${SRC:-paper_2503_20286_b200/csrc/variation.cu} > exp/$name/variation.cu
cp paper_2503_20286_b200/csrc/*.cuh exp/$name/
nvcc $FLAGS -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --fmad=false -Xcompiler -fPIC -Xptxas -v \
     -I include -I paper_2503_20286_b200/csrc -c exp/$name/variation.cu -o exp/$name/variation.o 2> exp/$name/ptxas.txt
objs=$(ls paper_2503_20286_b200/_lib/*.o | grep -v variation.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp/$name/libtemo_b200.so $objs exp/$name/variation.o -lcudart
grep -A3 "Compiling entry function.*k_offspring_wILi3ELb1" exp/$name/ptxas.txt | tail -1

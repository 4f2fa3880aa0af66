#!/bin/bash
# build_variant_nd.sh NAME : libtemo_b200.so with ndsort.cu compiled with $FLAGS, into exp/NAME/
set -e
cd "$(dirname "$0")/.."
name=$1
mkdir -p exp/$name
nvcc $FLAGS -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --fmad=false -Xcompiler -fPIC -Xptxas -v \
     -I include -I paper_2503_20286_b200/csrc -c paper_2503_20286_b200/csrc/ndsort.cu -o exp/$name/ndsort.o 2> exp/$name/ptxas.txt
objs=$(ls paper_2503_20286_b200/_lib/*.o | grep -v ndsort.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp/$name/libtemo_b200.so $objs exp/$name/ndsort.o -lcudart
rm -f exp/$name/*.o
grep -A3 "Compiling entry function.*k_dom_packedILi3E" exp/$name/ptxas.txt | tail -1

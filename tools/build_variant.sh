#!/bin/bash
# build a variant of libgrafem_b200.so with extra -D flags for cg_sell.cu: tools/build_variant.sh NAME FLAGS...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=paper_2103_14870_b200/_lib/variants/$name
mkdir -p $out
NVCC=/usr/local/cuda/bin/nvcc
CXX=/usr/bin/x86_64-linux-gnu-g++-13
$NVCC -c paper_2103_14870_b200/csrc/cg_sell.cu -o $out/cg_sell.o -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -ccbin $CXX -Xcompiler -fPIC,-fopenmp,-ffp-contract=off -Iinclude "$@"
objs=$(ls paper_2103_14870_b200/_lib/obj/*.o | grep -v cg_sell)
$NVCC -shared -o $out/libgrafem_b200.so $objs $out/cg_sell.o -gencode arch=compute_100a,code=sm_100a -ccbin $CXX -Xcompiler -fopenmp -lgomp
echo $out/libgrafem_b200.so

#!/bin/bash
# build a variant of libgrafem_b200.so with extra -D flags for one CUDA source (default cg_sell.cu):
#   [SRC=damage] tools/build_variant.sh NAME FLAGS...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
src=${SRC:-cg_sell}
extra=""
case $src in damage|misc) extra="-fmad=false";; esac
out=paper_2103_14870_b200/_lib/variants/$name
mkdir -p $out
NVCC=/usr/local/cuda/bin/nvcc
CXX=/usr/bin/x86_64-linux-gnu-g++-13
$NVCC -c paper_2103_14870_b200/csrc/$src.cu -o $out/$src.o -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -ccbin $CXX -Xcompiler -fPIC,-fopenmp,-ffp-contract=off -Iinclude $extra "$@"
objs=$(ls paper_2103_14870_b200/_lib/obj/*.o | grep -v "/$src.cu.o")
$NVCC -shared -o $out/libgrafem_b200.so $objs $out/$src.o -gencode arch=compute_100a,code=sm_100a -ccbin $CXX -Xcompiler -fopenmp -lgomp
echo $out/libgrafem_b200.so

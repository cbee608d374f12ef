#!/bin/bash
# ncu --set full of one kernel of the c3 bench for library variants: tools/ncu_kernel.sh REGEX VARIANT...
cd "$(dirname "$0")/.."
k=$1; shift
for v in "$@"; do
  lib=paper_2103_14870_b200/_lib/variants/$v/libgrafem_b200.so
  [ "$v" = main ] && lib=paper_2103_14870_b200/_lib/libgrafem_b200.so
  GF_LIB_PATH=$lib timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/k_$v.json 2>&1 && \
  GF_LIB_PATH=$lib timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o gpurun_out/k_${k}_$v -f python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_k_$v.log 2>&1
  echo "$v rc=$?"
done

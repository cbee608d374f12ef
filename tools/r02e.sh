#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02e; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -q > $o/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 $o/pytest_gpu.log
for ef in F edge; do
  GF_ELEMENT=$ef timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --sub c1,c4 > $o/bench_$ef.json 2> $o/bench_$ef.err; echo "bench $ef rc=$?"
done
GF_GRAPH=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --sub c1 > $o/bench_nograph.json 2> $o/bench_nograph.err; echo "bench nograph rc=$?"

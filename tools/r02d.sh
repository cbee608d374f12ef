#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02d; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -k "edge or metrics" > $o/pytest_edge.log 2>&1; echo "pytest edge rc=$?"; tail -5 $o/pytest_edge.log
for ef in F edge; do
  GF_ELEMENT=$ef timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --sub c4 > $o/bench_$ef.json 2> $o/bench_$ef.err; echo "bench $ef rc=$?"
done

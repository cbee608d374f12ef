#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02c; mkdir -p $o
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/grid_sync tools/grid_sync.cu && timeout 120 /tmp/grid_sync > $o/grid_sync.jsonl 2>&1; echo "grid_sync rc=$?"
for c in c1 c2 c3; do timeout 300 python tools/cg_trace_pipe.py $c >> $o/trace.jsonl 2>> $o/trace.err; echo "trace $c rc=$?"; done
timeout 1500 python -m pytest tests -m gpu -x -q > $o/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $o/pytest_gpu.log

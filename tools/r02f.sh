#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02f; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -q > $o/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $o/pytest_gpu.log
bash tools/ab.sh main_cur noeng r02head > $o/ab.txt 2>&1; cat $o/ab.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"

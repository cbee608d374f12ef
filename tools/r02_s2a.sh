#!/bin/bash
# Session-2 check of HEAD: smoke, the whole gpu suite, the default bench line.
cd $GRAFT_REPO_ROOT
o=gpurun_out/s2a; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $o/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $o/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > $o/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 $o/pytest_gpu.log
timeout 900 python bench.py > $o/bench_c3.json 2> $o/bench_c3.err; echo "bench rc=$?"; head -c 600 $o/bench_c3.json

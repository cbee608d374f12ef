#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02l; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -q > $o/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $o/pytest_gpu.log
for cl in 1 0; do GF_CG_CLUSTER=$cl timeout 300 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu --no-e2e --no-sub > $o/c1_cluster$cl.json 2>&1; echo "c1 cluster=$cl rc=$?"; done
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e --no-sub > $o/c4.json 2>&1; echo "c4 rc=$?"
timeout 900 python tools/trajectory.py c1 > $o/traj_c1.json 2>&1; echo "traj c1 rc=$?"; cat $o/traj_c1.json

#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02n; mkdir -p $o
bash tools/ab.sh base2 expl cur > $o/ab.txt 2>&1; cat $o/ab.txt
timeout 1500 python -m pytest tests -m gpu -q > $o/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $o/pytest_gpu.log
timeout 1500 python tools/trajectory.py c3 > $o/traj_c3.json 2> $o/traj_c3.err; echo "traj c3 rc=$?"; cat $o/traj_c3.json
timeout 900 python tools/trajectory.py c2 > $o/traj_c2.json 2> $o/traj_c2.err; echo "traj c2 rc=$?"; cat $o/traj_c2.json

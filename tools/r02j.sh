#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02j; mkdir -p $o
bash tools/ab.sh base ts2 ts4 nc > $o/ab.txt 2>&1; cat $o/ab.txt
CONFIG=c4 STEPS=5 bash tools/ab.sh base nc > $o/ab_c4.txt 2>&1; cat $o/ab_c4.txt
timeout 1500 python tools/trajectory.py c3 > $o/traj_c3.json 2> $o/traj_c3.err; echo "traj c3 rc=$?"; cat $o/traj_c3.json
timeout 900 python tools/trajectory.py c4 --steps 10 > $o/traj_c4.json 2> $o/traj_c4.err; echo "traj c4 rc=$?"; cat $o/traj_c4.json

#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02y; mkdir -p $o
for sp in 1 2 4; do GF_CG_SPLIT=$sp timeout 300 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu --no-e2e --no-sub > $o/c1_split$sp.json 2>&1; python -c "import json; d=json.load(open('$o/c1_split$sp.json')); print('split $sp', d['ms_per_step'], d['cg_iterations_per_step'], d['roofline']['pcg']['us_per_iteration'])"; done
timeout 900 python -m pytest tests -m gpu -q -k "trajectory or production_pcg or retry or graph or smoke or full_newton" > $o/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $o/pytest.log
timeout 900 python tools/trajectory.py c1 > $o/traj_c1.json 2>&1; echo "traj c1 rc=$?"; cat $o/traj_c1.json

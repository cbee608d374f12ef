#!/bin/bash
# pipelined PCG: parity tests + A/B of the solver variants and grid sizes
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02b; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -x -q > $o/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $o/pytest_gpu.log
for pipe in 0 1; do
  GF_CG_PIPE=$pipe timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --sub c1,c2 > $o/bench_pipe$pipe.json 2> $o/bench_pipe$pipe.err; echo "bench pipe=$pipe rc=$?"
done
for grid in 4 8 16 32 64; do
  GF_CG_GRID=$grid timeout 300 python bench.py --config c1 --steps 20 --warmup 5 --no-cpu --no-e2e --no-sub > $o/c1_grid$grid.json 2>&1; echo "c1 grid $grid rc=$?"
  GF_CG_GRID=$grid timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu --no-e2e --no-sub > $o/c2_grid$grid.json 2>&1; echo "c2 grid $grid rc=$?"
done
timeout 900 python tools/trajectory.py c1 > $o/traj_c1.json 2>&1; echo "traj c1 rc=$?"
timeout 900 python tools/trajectory.py c2 > $o/traj_c2.json 2>&1; echo "traj c2 rc=$?"

#!/bin/bash
# One GPU call that refreshes the committed evidence for version tag $1 (e.g. v7) into gpurun_out/prof_$1/:
# c3 bench (+ CPU baseline, e2e), c4 bench, reference arm, ncu launch list, ncu --set full of the top-3
# kernels, full-length trajectory parity (c1, c2, c3; c4 10 steps).
cd "$(dirname "$0")/.."
v=$1; o=gpurun_out/prof_$v; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $o/gpu.txt
timeout 900 python bench.py > $o/bench_c3.json 2> $o/bench_c3.err; echo "bench c3 rc=$?"
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu > $o/bench_c4.json 2> $o/bench_c4.err; echo "bench c4 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $o/bench_reference.json 2> $o/bench_reference.err; echo "reference rc=$?"
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-sub > $o/plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-sub > $o/ncu_launches.log 2>&1; echo "launches rc=$?"
for k in k_pcg_onchip k_nonlocal_cell k_assemble; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o $o/ncu_$k -f python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-sub > $o/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
for c in c1 c2 c3; do timeout 1500 python tools/trajectory.py $c >> $o/trajectories.jsonl 2>> $o/trajectories.err; echo "traj $c rc=$?"; done
timeout 900 python tools/trajectory.py c4 --steps 10 >> $o/trajectories.jsonl 2>> $o/trajectories.err; echo "traj c4 rc=$?"

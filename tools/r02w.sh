#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02w; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -q > $o/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $o/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?"; cat $o/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $o/bench_ref.json 2> $o/bench_ref.err; echo "ref rc=$?"
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-sub > $o/plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-sub > $o/ncu_launches.log 2>&1; echo "launches rc=$?"
for k in k_pcg_pipe k_assemble; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o $o/ncu_$k -f python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-sub > $o/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done

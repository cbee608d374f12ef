cd $GRAFT_REPO_ROOT
o=gpurun_out/r02a; mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $o/gpu.txt
timeout 300 python tools/l2_roof.py > $o/l2_roof.json 2> $o/l2_roof.err; echo "l2 rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > $o/bench.json 2> $o/bench.err; echo "bench rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_sell -s 2 -c 1 \
    -o $o/ncu_c4_pcg -f python bench.py --config c4 --steps 1 --warmup 2 --no-cpu --no-e2e --no-sub > $o/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"

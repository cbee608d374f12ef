#!/bin/bash
# k_pcg_big (round-robin static, deferred x) vs the ticketed k_pcg_sell<true> at c4; parity of the new instance
cd $GRAFT_REPO_ROOT
o=gpurun_out/r02_big; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q -k "pcg or trajectory or large_matrix or tiny_unstructured" > $o/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $o/pytest.log
for b in 1 0 1 0; do
  GF_CG_BIG=$b timeout 600 python bench.py --config c4 --steps 6 --warmup 3 --no-cpu --no-e2e --no-sub > $o/c4_big$b.json 2>$o/c4_big$b.err
  python -c "import json; d=json.load(open('$o/c4_big$b.json')); p=d['roofline']['pcg']; print('big $b', round(d['ms_per_step'],3), d['cg_iterations_per_step'], 'pcg ms', round(p['ms']/6,3), 'us/it', round(p['us_per_iteration'],2))"
done
GF_CG_BIG=1 timeout 300 python tools/cg_trace.py c4 2>&1 | tail -2

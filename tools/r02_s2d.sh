#!/bin/bash
# k_pcg_onchip v2 quick check: PCG tests per solver, c3/c2 A/B
cd $GRAFT_REPO_ROOT
o=gpurun_out/${TAG:-s2d}; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -x -k "production_pcg or trajectory_c1_scaled or trajectory_c3_scaled or graph" > $o/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 $o/pytest.log
for oc in 1 0; do
  GF_CG_ONCHIP=$oc timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-sub > $o/c3_oc$oc.json 2> $o/c3_oc$oc.err; echo "c3 oc=$oc rc=$?"
  python -c "import json; d=json.load(open('$o/c3_oc$oc.json')); print('c3 oc=$oc', d['ms_per_step'], d['cg_iterations_per_step'], d['roofline']['pcg']['us_per_iteration'], d['roofline']['kernels']['pcg']['avg_ms'])"
done
GF_CG_ONCHIP=1 timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu --no-e2e --no-sub > $o/c2_oc1.json 2> $o/c2_oc1.err; echo "c2 rc=$?"
python -c "import json; d=json.load(open('$o/c2_oc1.json')); print('c2 oc=1', d['ms_per_step'], d['cg_iterations_per_step'], d['roofline']['pcg']['us_per_iteration'])"

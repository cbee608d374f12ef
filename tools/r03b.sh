#!/bin/bash
# non-local cell template: library variants x GF_NL_GROUP (c3 bench, per-kernel times)
cd "$(dirname "$0")/.."
for rep in 1 2; do for v in "$@"; do for g in ${GROUPS_:-6 3 2}; do
  GF_NL_GROUP=$g GF_LIB_PATH=paper_2103_14870_b200/_lib/variants/$v/libgrafem_b200.so python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-sub > gpurun_out/r03b_$v.json 2>gpurun_out/r03b_$v.err
  python -c "import json; d=json.load(open('gpurun_out/r03b_$v.json')); k=d['roofline']['kernels']; print('$v g$g', ' '.join('%s %.3f' % (n, k[n]['avg_ms']) for n in ('pcg','nonlocal','assemble','tet_stress')), 'step %.3f ms' % d['ms_per_step'], 'value %.4g' % d['value'])" || tail -3 gpurun_out/r03b_$v.err
done; done; done

#!/bin/bash
# A/B library variants in ONE gpurun call (boxes differ by up to ~20%):
#   [CONFIG=c4] [STEPS=20] tools/ab.sh VARIANT...   (paper_2103_14870_b200/_lib/variants/VARIANT/libgrafem_b200.so)
cd "$(dirname "$0")/.."
cfg=${CONFIG:-c3}; steps=${STEPS:-20}
for rep in 1 2; do
for v in "$@"; do
  GF_LIB_PATH=paper_2103_14870_b200/_lib/variants/$v/libgrafem_b200.so python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu --no-e2e --no-sub > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  python -c "import json,sys; d=json.load(open('gpurun_out/ab_$v.json')); k=d['roofline']['kernels']; print('$v', ' '.join('%s %.3f' % (n, k[n]['avg_ms']) for n in ('pcg','nonlocal','assemble','tet_stress') if n in k), 'step %.3f ms' % d['ms_per_step'], 'value %.4g' % d['value'], 'cg/step %.2f' % d['cg_iterations_per_step'], 'us/it %.2f' % d['roofline'].get('pcg', {}).get('us_per_iteration', 0))" || tail -3 gpurun_out/ab_$v.err
done; done

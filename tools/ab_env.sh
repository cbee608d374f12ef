#!/bin/bash
# A/B environment-knob settings of the production library in ONE gpurun call:
#   tools/ab_env.sh "base:" "persist:GF_L2_PERSIST=1" ...
cd "$(dirname "$0")/.."
for rep in 1 2; do
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  env $envs python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/abe_$name.json 2>gpurun_out/abe_$name.err
  python -c "import json,sys; d=json.load(open('gpurun_out/abe_$name.json')); k=d['roofline']['kernels']; print('$name', ' '.join('%s %.3f' % (n, k[n]['avg_ms']) for n in ('pcg','nonlocal','assemble')), 'step %.3f ms' % d['ms_per_step'], 'value %.4g' % d['value'])" || tail -3 gpurun_out/abe_$name.err
done; done

#!/bin/bash
# cell-template non-local kernel: parity tests of the layouts, then c3 bench A/B over GF_NL_GROUP / per-tet template
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "nonlocal or damage or screen" > gpurun_out/r03a_pytest.log 2>&1; echo pytest=$?; tail -5 gpurun_out/r03a_pytest.log
for rep in 1 2; do for l in g6 g3 g2 g1 tet; do
  e="GF_NL_GROUP=${l#g}"; [ $l = tet ] && e="GF_NL_LAYOUT=tet"
  env $e python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-sub > gpurun_out/r03a_$l.json 2>gpurun_out/r03a_$l.err
  python -c "import json; d=json.load(open('gpurun_out/r03a_$l.json')); k=d['roofline']['kernels']; print('$l', ' '.join('%s %.3f' % (n, k[n]['avg_ms']) for n in ('pcg','nonlocal','assemble','tet_stress')), 'step %.3f ms' % d['ms_per_step'], 'value %.4g' % d['value'])" || tail -3 gpurun_out/r03a_$l.err
done; done

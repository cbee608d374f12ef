#!/bin/bash
# pcg time of library variants over several allocation placements (GF_PAD_MB before the system matrix)
cd "$(dirname "$0")/.."
for v in "$@"; do
  echo -n "$v:"
  for p in 0 2 4 6 8 10; do
    GF_PAD_MB=$p GF_LIB_PATH=paper_2103_14870_b200/_lib/variants/$v/libgrafem_b200.so python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(' %.3f' % d['roofline']['kernels']['pcg']['avg_ms'], end='')"
  done; echo
done

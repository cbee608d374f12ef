#!/bin/bash
# full gpu suite + default bench line + c3 trajectory slice
cd $GRAFT_REPO_ROOT
o=gpurun_out/${TAG:-s2j}; mkdir -p $o
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $o/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x > $o/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $o/pytest_gpu.log
timeout 900 python bench.py > $o/bench_c3.json 2> $o/bench_c3.err; echo "bench rc=$?"
python - <<PY
import json; d=json.load(open("$o/bench_c3.json"))
print("c3", d["value"]/1e6, d["ms_per_step"], "e2e", d["e2e"]["value"]/1e6, "pcg", d["roofline"]["kernels"]["pcg"]["avg_ms"])
for k,v in (d.get("sub") or {}).items():
    print(k, {kk: v.get(kk) for kk in ("value","ms_per_step")} if isinstance(v, dict) else v)
PY
timeout 900 python tools/trajectory.py c3 --steps 40 > $o/traj_c3.json 2>&1; echo "traj c3 rc=$?"; tail -c 400 $o/traj_c3.json
timeout 900 python tools/trajectory.py c2 --steps 60 > $o/traj_c2.json 2>&1; echo "traj c2 rc=$?"; tail -c 400 $o/traj_c2.json

"""Per-phase timing of k_pcg_onchip (GF_CG_TRACE stamps of CTA 0) on a config's step system. GPU box only.

  python tools/cg_trace_oc.py [c3|c2]
"""
import ctypes as C, os, sys
os.environ["GF_CG_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2103_14870_b200 as g
from paper_2103_14870_b200 import configs as cf
s = cf.get(sys.argv[1] if len(sys.argv) > 1 else "c3")
sim, mesh = cf.build_gpu(s)
assert sim.info()["pcg_solver_name"].startswith("onchip"), sim.info()["pcg_solver_name"]
for _ in range(4):
    st = sim.dynamic_step()
buf = np.zeros(5000, np.uint64)
g._check(g.lib().gf_sim_cg_trace(sim._h, buf.ctypes.data_as(C.POINTER(C.c_uint64))))
n = min(st.cg_iterations, 199)
t = buf[:1600].reshape(200, 8)[1:n - 1].astype(np.float64)
it = (t[1:, 0] - t[:-1, 0]) / 1e3
us = lambda a, b: np.round(((t[:, b] - t[:, a]) / 1e3).mean(), 2)
print("iters", st.cg_iterations, "us/iter %.2f" % it.mean(), "| CTA0: spmv", us(0, 1), "reduce", us(1, 2),
      "update", us(2, 5), "produce", us(5, 3), "publish", us(3, 4), "barrier (to next top) %.2f" % (it.mean() - us(0, 4)))
nb = int((buf[3000:4000] > 0).sum())
e = buf[3000:3000 + nb].astype(np.float64)
p = buf[2000:2000 + nb].astype(np.float64)
print("publish-end at iteration 10 (from the first SpMV end): min %.2f median %.2f max %.2f us; slowest CTAs %s" % (
    (p.min() - e.min()) / 1e3, (np.median(p) - e.min()) / 1e3, (p.max() - e.min()) / 1e3,
    list(np.argsort(p)[-6:])))
print("CTAs", nb, "| SpMV-end spread at iteration 10: %.2f us (median %.2f)" % ((e.max() - e.min()) / 1e3,
                                                                             (np.median(e) - e.min()) / 1e3))
sub = buf[4100:4105].astype(np.float64)
if sub[0] > 0:
    print("SpMV of CTA 0 warp 0 row 0 at iteration 10 (us from its start): on-chip part %.2f, round-1 loads consumed %.2f,"
          " round 2 %.2f, round 3 %.2f" % tuple((sub[1:] - sub[0]) / 1e3))

"""Per-phase timing of the production PCG kernel on the c3 system (GF_CG_TRACE). GPU box only."""
import ctypes as C, os, sys
os.environ["GF_CG_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2103_14870_b200 as g
from paper_2103_14870_b200 import configs as cf
s = cf.get(sys.argv[1] if len(sys.argv) > 1 else "c3")
sim, mesh = cf.build_gpu(s)
for _ in range(4):
    st = sim.dynamic_step()
buf = np.zeros(5000, np.uint64)
g._check(g.lib().gf_sim_cg_trace(sim._h, buf.ctypes.data_as(C.POINTER(C.c_uint64))))
n = st.cg_iterations
t = buf[:1600].reshape(200, 8)[1:n - 1].astype(np.float64)
it = (t[1:, 0] - t[:-1, 0]) / 1e3
us = lambda a, b: np.round(((t[:, b] - t[:, a]) / 1e3).mean(), 2)
print("iters", n, "us/iter %.2f" % it.mean(), "| CTA0: A work", us(0, 1), "A wait+barrier", us(1, 5), "A reduce", us(5, 2),
      "B work", us(2, 3), "B wait+barrier", us(3, 6), "B reduce", us(6, 4))
nb = int((buf[2000:3000] > 0).sum())
b_end = buf[2000:2000 + nb].astype(np.float64)
a_end = buf[3000:3000 + nb].astype(np.float64)
t0 = a_end.min()
print("CTAs", nb, "| phase-A end spread %.2f us | phase-B end (from first A end) min %.2f med %.2f max %.2f us" % (
    (a_end.max() - t0) / 1e3, (b_end.min() - t0) / 1e3, (np.median(b_end) - t0) / 1e3, (b_end.max() - t0) / 1e3))

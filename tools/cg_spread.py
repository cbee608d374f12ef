"""Per-CTA phase-end spread of the production PCG (GF_CG_TRACE): which CTAs finish phase A last, and is it
the same CTAs in two iterations (10 and 20)? GPU box only."""
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
t = buf[:1600].reshape(200, 8).astype(np.float64)
nb = int((buf[3000:4000] > 0).sum())
for it, off in ((10, 3000), (20, 4000)):
    start = t[it, 0]  # CTA0 iteration start
    a = (buf[off:off + nb].astype(np.float64) - start) / 1e3
    order = np.argsort(a)
    print("iter", it, "A-end us: min %.2f p10 %.2f med %.2f p90 %.2f max %.2f" % (a.min(), *np.percentile(a, [10, 50, 90]), a.max()))
    print("  slowest CTAs", order[-12:].tolist(), "fastest", order[:8].tolist())
    if it == 10:
        a10 = a
    else:
        print("  corr(iter10, iter20) = %.3f" % np.corrcoef(a10, a)[0, 1])

"""Per-phase timing of the cooperative PCG kernel on the c3 system (GF_CG_TRACE). GPU box only."""
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
t = buf[:2000].reshape(2, 200, 5).astype(np.float64)
n = st.cg_iterations
for b, name in [(0, "block0"), (1, "last")]:
    d = np.diff(t[b, 1:n - 1], axis=1) / 1e3  # us: spmv_end-start? columns: [0->1 spmv, 1->2 reduceA, 2->3 phaseB, 3->4 reduceB]
    it = (t[b, 2:n - 1, 0] - t[b, 1:n - 2, 0]) / 1e3
    print(name, "iters", n, "us/iter %.2f" % it.mean(), "phases (spmv, redA, phaseB, redB) us:", np.round(d.mean(0), 2))
buf = np.zeros(5000, np.uint64)
g._check(g.lib().gf_sim_cg_trace(sim._h, buf.ctypes.data_as(C.POINTER(C.c_uint64))))
nb = int((buf[2000:3000] > 0).sum())
b_end = buf[2000:2000 + nb].astype(np.float64); a_end = buf[3000:3000 + nb].astype(np.float64)
t0 = a_end.min()
print("blocks", nb, "phaseA end spread (us): min 0 max %.2f" % ((a_end.max() - t0) / 1e3),
      " phaseB end (us from first A end): min %.2f median %.2f max %.2f" % ((b_end.min() - t0) / 1e3, (np.median(b_end) - t0) / 1e3, (b_end.max() - t0) / 1e3))
print("slowest phaseA blocks:", np.argsort(-a_end)[:8], " slowest phaseB blocks:", np.argsort(-b_end)[:8])

"""Per-phase timing of the pipelined PCG (k_pcg_pipe, GF_CG_TRACE): CTA 0's SpMV (incl. the overlapped partial
loads), reduce + update + publish, and barrier wait per iteration; spread of the CTAs' SpMV and publish ends at
iteration 10. GPU box only:  python tools/cg_trace_pipe.py c3"""
import ctypes as C, json, os, sys
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
n = min(st.cg_iterations, 199)
t = buf[:1600].reshape(200, 8)[1:n - 1].astype(np.float64)
it = (t[1:, 0] - t[:-1, 0]) / 1e3
us = lambda a, b: float(np.round(((t[:, b] - t[:, a]) / 1e3).mean(), 3))
wait = float(np.round(((t[1:, 0] - t[:-1, 3]) / 1e3).mean(), 3))
nb = int((buf[2000:3000] > 0).sum())
pub = buf[2000:2000 + nb].astype(np.float64)
spmv = buf[3000:3000 + nb].astype(np.float64)
t0 = spmv.min()
print(json.dumps({"config": s.name, "iterations": int(st.cg_iterations), "us_per_iter": float(it.mean()),
                  "cta0_spmv_us": us(0, 1), "cta0_reduce_update_publish_us": us(1, 3), "cta0_barrier_wait_us": wait,
                  "ctas": nb, "spmv_end_spread_us": float((spmv.max() - t0) / 1e3),
                  "publish_end_spread_us": float((pub.max() - pub.min()) / 1e3)}))
# per-CTA SpMV-end offsets at iterations 10 and 20 with the SM each CTA ran on: is the spread the same CTAs / SMs?
s10 = buf[3000:3000 + nb].astype(np.float64)
s20 = buf[4000:4000 + nb].astype(np.float64)
sm = buf[1600:1600 + nb].astype(np.int64)
if (s20 > 0).all():
    d10 = (s10 - s10.min()) / 1e3
    d20 = (s20 - s20.min()) / 1e3
    slow = np.argsort(-d10)[:10]
    print(json.dumps({"corr_spmv_end_it10_it20": float(np.corrcoef(d10, d20)[0, 1]),
                      "slowest_ctas_it10": [int(x) for x in slow], "their_sm": [int(sm[x]) for x in slow],
                      "their_delay_us_it10": [round(float(d10[x]), 2) for x in slow],
                      "their_delay_us_it20": [round(float(d20[x]), 2) for x in slow],
                      "median_delay_us": float(np.median(d10))}))

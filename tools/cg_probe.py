"""Per-iteration cost of the cooperative PCG kernel: tiny system (barrier/launch overhead only) vs the
c3 system matrix (SpMV + vector phases). Run on the GPU box."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2103_14870_b200 as g

for n, iters in [(10, 2000), (10, 200)]:
    rp = np.arange(n + 1); cols = np.arange(n); vals = np.ones(n)
    b = np.ones(n)
    g.cg_solve_csr(rp, cols, vals, b, np.zeros(n), 0.0, 5)
    # identity converges in 1 iteration unless tol=0 -> runs max_iters? rr=0 => rnorm/bnorm=0<=0 converged.
    M = np.random.default_rng(0).uniform(-1, 1, (n, n)); A = M @ M.T + n * np.eye(n)
    rp = np.arange(0, n * n + 1, n); cols = np.tile(np.arange(n), n)
    t0 = time.perf_counter()
    x, r = g.cg_solve_csr(rp, cols, A.reshape(-1), b, np.zeros(n), 1e-300, iters)
    el = time.perf_counter() - t0
    print(f"tiny n={n}: {r['iterations']} iterations in {el*1e3:.2f} ms -> {el/max(1,r['iterations'])*1e6:.2f} us/iter (incl. launch+copies)")

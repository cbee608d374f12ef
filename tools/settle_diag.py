# Per-step GPU-vs-oracle displacement difference for the block-on-floor case (test_collision.cpp:133-166).
# Run on a B200: PYTHONPATH=. python tools/settle_diag.py
import numpy as np, paper_2103_14870_b200 as g
from oracle import oracle as o
col = dict(kind="halfspace", point=(0, 0, 0), normal=(0, 1, 0), stiffness=2e5, restitution=0.0)
om = o.Mesh.make_box((0.1, 0.1, 0.1), (2, 2, 2))
gmat = g.MaterialParams.from_youngs(5e6, 0.3, 1000.0, 1e9, 0.0, g.STVK)
omat = o.material_from_youngs(5e6, 0.3, 1000.0, 1e9, 0.0, g.STVK)
gmat.damp_mass_coeff = omat.damp_mass_coeff = 40.0
gs = g.Simulation(g.make_box_mesh((0.1, 0.1, 0.1), (2, 2, 2)), gmat, g.SolverConfig(dt=1e-3, gravity=(0, -9.81, 0), cg_tol=1e-10), [], [g.Collider(kind="halfspace", normal=(0, 1, 0), stiffness=2e5)])
os_ = o.Sim(om, omat, o.solver_config(dt=1e-3, gravity=(0, -9.81, 0), cg_tol=1e-10), [], [col])
for k in range(200):
    a = os_.dynamic_step(); b = gs.dynamic_step()
    d = np.abs(gs.state().displacements - os_.get_state()["u"]).max()
    if k % 10 == 0 or k < 20: print(k, "%.3e" % d, a.cg_iterations, b.cg_iterations, "%.6e %.6e" % (a.load, b.load))

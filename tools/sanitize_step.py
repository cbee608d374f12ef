"""A few dynamic steps of scaled c3 (non-local damage, pipelined PCG, graph replay) and c4 (collider), with both
element forms, plus the parity hooks -- the workload run under compute-sanitizer (memcheck, racecheck,
synccheck) by tools/r02_sanitize.sh; the logs go to profiles/."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2103_14870_b200 import configs as cf

for name, cells, thres in (("c3", (8, 8, 7), 500.0), ("c4", (6, 6, 6), 2e7)):
    for elem in ("F", "edge"):
        os.environ["GF_ELEMENT"] = elem
        s = cf.scaled(name, cells)
        s.sigma_thres = thres
        sim, mesh = cf.build_gpu(s)
        rng = np.random.default_rng(1)
        sim.set_state(displacements=rng.uniform(-0.02 * cf.H, 0.02 * cf.H, (mesh.num_nodes(), 3)))
        for _ in range(3):
            st = sim.dynamic_step()
        sim.eval_forces()
        sim.eval_stiffness()
        sim.eval_screening()
        sim.step_metrics()
        sim.edge_forces()
        print(name, elem, "cg", st.cg_iterations, "newly", st.newly_broken, flush=True)

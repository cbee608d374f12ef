"""Builds an ORACLE simulation for a paper_2103_14870_b200.configs.Scenario (test/bench infrastructure).

Same mesh (bit-identical generator), same material, BC node sets, loads and initial velocity as
configs.build_gpu, so the two paths start from identical inputs.
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as o


def build_oracle(s):
    from paper_2103_14870_b200 import configs as cf
    mesh = o.Mesh.make_box(s.size, s.cells, s.origin, s.jitter, s.seed)
    X = mesh.arrays()["rest"]
    mat = o.material_from_youngs(s.youngs, s.poisson, s.density, s.sigma_thres, s.r_d, s.model)
    cfg = o.solver_config(dt=s.dt, cg_tol=s.cg_tol, cg_max_iters=s.cg_max_iters, gravity=s.gravity)
    sim = o.Sim(mesh, mat, cfg, cf.bc_dicts(s, X), s.colliders)
    f = cf.point_load_vector(s, X)
    if f is not None:
        sim.set_external_forces(f)
    if s.initial_velocity is not None:
        sim.set_state(v=np.tile(np.asarray(s.initial_velocity, np.float64), (mesh.num_nodes, 1)))
    return sim, mesh


def near_threshold_flips(om, mat, u_pre, r_d, thres, edges, tol):
    """Label-sync acceptance rule (SURVEY §7 hard part 7): a label that differs between the GPU and the oracle after
    a step is legitimate only if the oracle's screening value of that edge, computed from the PRE-step state the
    damage pass saw, lies within tol * thres of the threshold (a rounding-level decision). Returns
    (all_ok, max relative distance |s - thres| / thres over the differing edges)."""
    sig = om.per_tet_cauchy(mat, u_pre)
    scr = om.nonlocal_screen(u_pre, sig, r_d)[0]
    dist = np.abs(scr[np.asarray(edges)] - thres) / thres
    worst = float(dist.max()) if len(dist) else 0.0
    return bool(worst <= tol), worst

"""Golden vectors of the hot path, written by the CPU oracle (oracle/grafem_oracle.cpp) on seeded inputs:

  python tests/golden/make_golden.py        ->  tests/golden/hot_path_small.npz

The reference itself cannot be built in this image (Eigen is absent), so the fixtures come from its
line-cited restatement, which tests/test_oracle_kat.py and tests/test_mesh_kat.py pin to the reference's own
unit-test known answers. Per scaled BASELINE config (c1 4x4x12, c2 6x6x6, c3 8x8x7 cells) the file holds the INPUT
state (u, v, labels, chi: stored, so the tests do not depend on a numpy generator) and the oracle's outputs from that
state: Cauchy six-vectors, screening values, local edge stresses, degenerate flags, internal forces, strain
energy, the damage pass (ascending newly-broken ids, chi); and five dynamic steps of the scenario from rest (u, v, labels,
chi, CG iterations).
tests/test_golden.py checks the oracle (CPU, `-m "not gpu"`) and the CUDA path (`-m gpu`) against them.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.scenario import build_oracle  # noqa: E402
from paper_2103_14870_b200 import configs as cf  # noqa: E402

CASES = {"c1": (4, 4, 12), "c2": (6, 6, 6), "c3": (8, 8, 7)}
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "hot_path_small.npz")


def make_case(name, cells, seed):
    s = cf.scaled(name, cells)
    sim, mesh = build_oracle(s)
    st = sim.get_state()
    rng = np.random.default_rng(seed)
    u = rng.uniform(-0.2 * cf.H, 0.2 * cf.H, st["u"].shape)
    v = rng.uniform(-0.01, 0.01, st["v"].shape)
    zeta = (rng.uniform(0, 1, st["zeta"].shape) < 0.1).astype(np.uint8)
    chi = rng.uniform(0.0, 1.0, st["chi"].shape)
    sim.set_state(u=u, v=v, zeta=zeta, chi=chi)
    out = {"u": u, "v": v, "zeta": zeta, "chi": chi}
    sig = mesh.per_tet_cauchy(sim.mat, u)
    scr, sf, deg = mesh.nonlocal_screen(u, sig, s.r_d)
    out.update(sigma_c=sig, screening=scr, sigma_f=sf, degenerate=deg,
               forces=mesh.assemble_forces(sim.mat, u, chi).reshape(-1),
               energy=np.float64(mesh.total_strain_energy(sim.mat, u, chi)))
    out["newly"] = sim.damage_pass()
    after = sim.get_state()
    out["zeta_after_damage"], out["chi_after_damage"] = after["zeta"], after["chi"]
    # five dynamic steps of the scenario itself (rest state, its boundary conditions, loads and initial velocity)
    sim, mesh = build_oracle(s)
    iters = []
    for _ in range(5):
        iters.append(sim.dynamic_step().cg_iterations)
    end = sim.get_state()
    out.update(step_u=end["u"], step_v=end["v"], step_zeta=end["zeta"], step_chi=end["chi"],
               step_cg_iterations=np.asarray(iters, np.int64))
    return {f"{name}/{k}": np.asarray(a) for k, a in out.items()}


def main():
    data = {}
    for i, (name, cells) in enumerate(CASES.items()):
        data.update(make_case(name, cells, 100 + i))
    np.savez_compressed(OUT, **data)
    print(OUT, os.path.getsize(OUT), "bytes,", len(data), "arrays")


if __name__ == "__main__":
    main()

"""The committed golden vectors (tests/golden/hot_path_small.npz, written by tests/golden/make_golden.py from the
CPU oracle on seeded inputs) against the oracle itself (CPU: guards the oracle and its build against drift) and
against the CUDA path through the C ABI (`-m gpu`). Bars as everywhere: labels, newly-broken sets, chi, degenerate
flags, Cauchy stresses and screening values bit-exact from the stored state; forces and energy within 1e-9; node
positions after the stored steps within 1e-6 relative."""
import os

import numpy as np
import pytest

from oracle.scenario import build_oracle
from paper_2103_14870_b200 import configs as cf

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "hot_path_small.npz")
CASES = {"c1": (4, 4, 12), "c2": (6, 6, 6), "c3": (8, 8, 7)}
STEPS = 5


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64) if a.dtype == np.float64 else a


def same_bits_or_zero(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.array_equal(bits(a), bits(b)) or np.array_equal(a, b)


def entrywise(a, b, tol, floor):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return bool(np.all(np.abs(a - b) <= tol * np.maximum(np.abs(b), floor)))


def test_fixture_is_complete(gold):
    keys = {"u", "v", "zeta", "chi", "sigma_c", "screening", "sigma_f", "degenerate", "forces", "energy", "newly",
            "zeta_after_damage", "chi_after_damage", "step_u", "step_v", "step_zeta", "step_chi",
            "step_cg_iterations"}
    assert set(gold.files) == {f"{c}/{k}" for c in CASES for k in keys}
    assert sum(len(gold[f"{c}/newly"]) for c in CASES) > 0  # the seeded states do break edges


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_reproduces_golden(gold, name):
    G = lambda k: gold[f"{name}/{k}"]  # noqa: E731
    s = cf.scaled(name, CASES[name])
    sim, mesh = build_oracle(s)
    u, chi = G("u"), G("chi")
    sim.set_state(u=u, v=G("v"), zeta=G("zeta"), chi=chi)
    sig = mesh.per_tet_cauchy(sim.mat, u)
    scr, sf, deg = mesh.nonlocal_screen(u, sig, s.r_d)
    assert same_bits_or_zero(sig, G("sigma_c")) and same_bits_or_zero(scr, G("screening"))
    assert same_bits_or_zero(sf, G("sigma_f")) and np.array_equal(deg, G("degenerate"))
    f = mesh.assemble_forces(sim.mat, u, chi).reshape(-1)
    assert entrywise(f, G("forces"), 1e-12, np.abs(G("forces")).max() * 1e-6)
    assert abs(mesh.total_strain_energy(sim.mat, u, chi) - G("energy")) <= 1e-12 * abs(G("energy"))
    assert np.array_equal(sim.damage_pass(), G("newly"))
    st = sim.get_state()
    assert np.array_equal(st["zeta"], G("zeta_after_damage")) and same_bits_or_zero(st["chi"], G("chi_after_damage"))
    sim, mesh = build_oracle(s)
    iters = [sim.dynamic_step().cg_iterations for _ in range(STEPS)]
    end = sim.get_state()
    assert iters == list(G("step_cg_iterations")) and np.array_equal(end["zeta"], G("step_zeta"))
    scale = np.abs(mesh.arrays()["rest"]).max()
    assert np.abs(end["u"] - G("step_u")).max() <= 1e-12 * scale
    assert same_bits_or_zero(end["chi"], G("step_chi"))


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_cuda_path_reproduces_golden(gold, name):
    G = lambda k: gold[f"{name}/{k}"]  # noqa: E731
    s = cf.scaled(name, CASES[name])
    sim, mesh = cf.build_gpu(s)
    sim.set_state(G("u"), G("v"), G("zeta"), G("chi"))
    assert same_bits_or_zero(sim.eval_cauchy(), G("sigma_c"))
    scr, sf, deg = sim.eval_screening()
    assert same_bits_or_zero(scr, G("screening")) and same_bits_or_zero(sf, G("sigma_f"))
    assert np.array_equal(deg, G("degenerate"))
    assert entrywise(sim.eval_forces(), G("forces"), 1e-9, np.abs(G("forces")).max() * 1e-6)
    assert np.array_equal(sim.damage_pass(), G("newly"))
    st = sim.state()
    assert np.array_equal(st.edge_damage, G("zeta_after_damage"))
    assert same_bits_or_zero(st.element_chi, G("chi_after_damage"))
    sim, mesh = cf.build_gpu(s)
    iters = [sim.dynamic_step().cg_iterations for _ in range(STEPS)]
    end = sim.state()
    # labels exact; chi is bit-exact only from an identical state (here the states agree to ~1e-10)
    assert np.array_equal(end.edge_damage, G("step_zeta")) and np.abs(end.element_chi - G("step_chi")).max() <= 1e-6
    assert all(abs(a - b) <= 2 for a, b in zip(iters, G("step_cg_iterations")))
    assert np.abs(end.displacements - G("step_u")).max() <= 1e-6 * np.abs(mesh.rest_positions).max()

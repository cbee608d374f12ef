"""Pins the CPU oracle against the reference's own unit-test known answers.

Every case cites the reference test it restates (paths under /root/reference/proj/tests).
These run on CPU only; they are what makes the oracle trustworthy as the GPU parity checker.
"""
import math

import numpy as np
import pytest

from oracle import oracle as o

STVK, NH = 1, 0


def unit_tet():
    return o.Mesh.create([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], [[0, 1, 2, 3]])


def regular_tet():
    return o.Mesh.create([[0, 0, 0], [1, 0, 0], [0.5, math.sqrt(3) / 2, 0],
                          [0.5, math.sqrt(3) / 6, math.sqrt(6) / 3]], [[0, 1, 2, 3]])


def stvk_soft(sigma=1e5):
    return o.material_from_youngs(1e6, 0.3, 1000.0, sigma, 0.0, STVK)


def rand_rotation(rng):
    ax = rng.uniform(-1, 1, 3)
    ax /= np.linalg.norm(ax)
    th = rng.uniform(-1, 1) * math.pi
    K = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]])
    return np.eye(3) + math.sin(th) * K + (1 - math.cos(th)) * K @ K


def rand_deformation(rng, spread=0.4):
    while True:
        F = np.eye(3) + rng.uniform(-spread, spread, (3, 3))
        if np.linalg.det(F) >= 0.15:
            return F


# ------------------------------------------------------------------ material (test_material.cpp)
def test_lame_roundtrip():  # test_material.cpp:45-54
    p = o.material_from_youngs(2.1e9, 0.3, 7800.0, 1e6)
    assert p.mu == pytest.approx(2.1e9 / 2.6, rel=1e-12)
    assert p.lambda_ == pytest.approx(2.1e9 * 0.3 / (1.3 * 0.4), rel=1e-12)


def test_validation_rejects():  # test_material.cpp:56-60
    for args in [(-1.0, 0.3, 1000, 1e5), (1e6, 0.5, 1000, 1e5), (1e6, 0.3, 1000, -1e5)]:
        with pytest.raises(o.FormatError):
            o.material_from_youngs(*args)


def test_stvk_energy_kat():  # test_material.cpp:62-67
    p = o.material_lame(1.0, 1.0, STVK)
    assert o.energy_density(np.eye(3), p) == 0.0
    assert o.energy_density(2 * np.eye(3), p) == pytest.approx(16.875, rel=1e-14)


def test_stvk_energy_stationary_at_rest():  # test_material.cpp:155-170
    p = o.material_lame(1.0, 1.0, STVK)
    rng = np.random.default_rng(59)
    h = 1e-7
    for _ in range(10):
        d = rng.uniform(-1, 1, (3, 3))
        d /= np.linalg.norm(d)
        slope = (o.energy_density(np.eye(3) + h * d, p) - o.energy_density(np.eye(3) - h * d, p)) / (2 * h)
        assert abs(slope) < 100 * h


def test_nh_rest_energy_kat():  # test_material.cpp:69-74
    p = o.material_lame(1.0, 1.0, NH)
    assert o.energy_density(np.eye(3), p) == pytest.approx(0.5 * 0.5625 - 0.5 * math.log(4.0), rel=1e-14)


def test_stvk_pk1_rest_and_diagonal():  # test_material.cpp:76-86
    p = o.material_lame(1.0, 1.0, STVK)
    assert np.linalg.norm(o.pk1(np.eye(3), p)) == 0.0
    F = np.eye(3)
    F[0, 0] = 1.3
    P = o.pk1(F, p)
    assert np.all(np.abs(P - np.diag(np.diag(P))) < 1e-14) and P[0, 0] > 0


@pytest.mark.parametrize("model", [STVK, NH])
def test_pk1_matches_fd(model):  # test_material.cpp:88-109
    p = o.material_lame(1.0, 1.0, model)
    rng = np.random.default_rng(41)
    worst = 0.0
    for _ in range(100):
        F = rand_deformation(rng)
        P = o.pk1(F, p)
        h = 1e-6 * np.linalg.norm(F)
        scale = max(np.linalg.norm(P), 1e-12)
        for i in range(3):
            for j in range(3):
                Fp, Fm = F.copy(), F.copy()
                Fp[i, j] += h
                Fm[i, j] -= h
                fd = (o.energy_density(Fp, p) - o.energy_density(Fm, p)) / (2 * h)
                worst = max(worst, abs(fd - P[i, j]) / scale)
    assert worst < 1e-4


def test_pk1_differential_identity_kat():  # test_material.cpp:111-121
    p = o.material_lame(1.0, 1.0, STVK)
    F = rand_deformation(np.random.default_rng(43))
    assert np.linalg.norm(o.pk1_differential(F, np.zeros((3, 3)), p)) == 0.0
    d = 0.37
    dp = o.pk1_differential(np.eye(3), d * np.eye(3), p)
    assert np.linalg.norm(dp - (3 * 1.0 + 2 * 1.0) * d * np.eye(3)) < 1e-12


@pytest.mark.parametrize("model", [STVK, NH])
def test_pk1_differential_fd(model):  # test_material.cpp:123-140
    p = o.material_lame(1.0, 1.0, model)
    rng = np.random.default_rng(47)
    worst = 0.0
    for _ in range(100):
        F = rand_deformation(rng)
        dF = rng.uniform(-1, 1, (3, 3))
        h = 1e-6
        an = o.pk1_differential(F, dF, p)
        fd = (o.pk1(F + h * dF, p) - o.pk1(F - h * dF, p)) / (2 * h)
        worst = max(worst, np.linalg.norm(fd - an) / max(np.linalg.norm(an), 1e-12))
    assert worst < 1e-3


@pytest.mark.parametrize("model", [STVK, NH])
def test_energy_rotation_invariant(model):  # test_material.cpp:142-153
    p = o.material_lame(1.0, 1.0, model)
    rng = np.random.default_rng(53)
    for _ in range(50):
        F = rand_deformation(rng)
        R = rand_rotation(rng)
        a, b = o.energy_density(F, p), o.energy_density(R @ F, p)
        assert abs(a - b) <= 1e-10 * max(1.0, abs(a))


def test_cauchy_rest_rotation_uniaxial_fallback():  # test_material.cpp:172-205
    p = o.material_lame(1.0, 1.0, STVK)
    c, fb = o.cauchy_sixvector(np.eye(3), p)
    assert np.linalg.norm(c) == 0.0 and not fb
    c, _ = o.cauchy_sixvector(rand_rotation(np.random.default_rng(61)), p)
    assert np.linalg.norm(c) < 1e-12
    F = np.eye(3)
    F[0, 0] = 1.1
    c, fb = o.cauchy_sixvector(F, p)
    assert not fb and c[0] > 0 and np.all(np.abs(c[3:]) < 1e-14)
    sig = o.pk1(F, p) @ F.T / np.linalg.det(F)
    assert c[0] == pytest.approx(sig[0, 0], rel=1e-12) and c[1] == pytest.approx(sig[1, 1], rel=1e-12)
    F = np.eye(3)
    F[2, 2] = -0.5
    c, fb = o.cauchy_sixvector(F, p)
    P = o.pk1(F, p)
    sym = 0.5 * (P + P.T)
    assert fb and c[0] == pytest.approx(sym[0, 0]) and c[3] == pytest.approx(2 * sym[0, 1])


# ------------------------------------------------------------------ fem (test_fem.cpp)
def test_deformation_gradient_rest_translation_affine():  # test_fem.cpp:38-55
    m = unit_tet()
    assert np.array_equal(m.deformation_gradient(np.zeros((4, 3)), 0), np.eye(3))
    assert np.array_equal(m.deformation_gradient(np.tile([0.13, -2.4, 0.777], (4, 1)), 0), np.eye(3))
    box = o.Mesh.make_box((1, 1, 1), (2, 2, 2))
    A = np.array([[1.1, 0.2, -0.05], [0.0, 0.93, 0.1], [0.04, -0.02, 1.02]])
    X = box.arrays()["rest"]
    u = X @ (A - np.eye(3)).T
    for e in range(box.num_tets):
        assert np.linalg.norm(box.deformation_gradient(u, e) - A) < 1e-12


def test_element_forces_zero_chi_sum():  # test_fem.cpp:57-72
    m = unit_tet()
    p = stvk_soft()
    assert np.all(m.element_internal_force(p, 0) == 0.0)
    u = np.random.default_rng(5).uniform(-0.1, 0.1, (4, 3))
    f = m.element_internal_force(p, 0, u)
    assert np.linalg.norm(f.sum(0)) < 1e-9 * np.linalg.norm(f, axis=1).sum()
    assert np.all(m.element_internal_force(p, 0, u, np.zeros(1)) == 0.0)


def test_element_forces_fd():  # test_fem.cpp:74-96
    m = unit_tet()
    p = stvk_soft()
    u = np.random.default_rng(7).uniform(-0.08, 0.08, (4, 3))
    chi = np.array([0.6])
    f = m.element_internal_force(p, 0, u, chi)
    vol = m.arrays()["vol"][0]
    h = 1e-7
    scale = np.abs(f).max()
    for n in range(4):
        for ax in range(3):
            up, um = u.copy(), u.copy()
            up[n, ax] += h
            um[n, ax] -= h
            ep = 0.6 * vol * o.energy_density(m.deformation_gradient(up, 0), p)
            em = 0.6 * vol * o.energy_density(m.deformation_gradient(um, 0), p)
            assert abs(-(ep - em) / (2 * h) - f[n, ax]) / scale < 1e-4


def test_assembled_forces_rest_locality_fd():  # test_fem.cpp:151-172 + verify.cpp:97-115
    m = o.Mesh.make_box((0.2, 0.1, 0.1), (4, 2, 2))
    p = stvk_soft()
    assert np.linalg.norm(m.assemble_forces(p)) == 0.0
    u = np.zeros((m.num_nodes, 3))
    moved = m.num_nodes // 2
    u[moved] = [0.002, -0.001, 0.0015]
    f = m.assemble_forces(p, u).reshape(-1, 3)
    tets = m.arrays()["tets"]
    adj = np.zeros(m.num_nodes, bool)
    adj[np.unique(tets[(tets == moved).any(1)])] = True
    assert np.all(f[~adj] == 0.0)
    u = np.random.default_rng(17).uniform(-0.002, 0.002, (m.num_nodes, 3))
    f = m.assemble_forces(p, u)
    scale = max(np.abs(f).max(), 1e-30)
    h = 1e-6
    worst = 0.0
    for n in range(m.num_nodes):
        for ax in range(3):
            up, um = u.copy(), u.copy()
            up[n, ax] += h
            um[n, ax] -= h
            fd = -(m.total_strain_energy(p, up) - m.total_strain_energy(p, um)) / (2 * h)
            worst = max(worst, abs(fd - f[3 * n + ax]) / scale)
    assert worst < 1e-4


def test_global_forces_sum_zero():  # test_fem.cpp:174-182
    m = o.Mesh.make_box((0.2, 0.1, 0.1), (3, 2, 2))
    u = np.random.default_rng(23).uniform(-0.004, 0.004, (m.num_nodes, 3))
    f = m.assemble_forces(stvk_soft(), u)
    assert np.linalg.norm(f.reshape(-1, 3).sum(0)) <= 1e-9 * max(1.0, np.linalg.norm(f))


def _dense_K(m, vals):
    rp, cols, _ = m.pattern()
    n = len(rp) - 1
    K = np.zeros((n, n))
    for i in range(n):
        K[i, cols[rp[i]:rp[i + 1]]] = vals[rp[i]:rp[i + 1]]
    return K


def test_stiffness_small_strain_kat():  # test_fem.cpp:184-229
    m = unit_tet()
    p = stvk_soft()
    assert np.abs(m.assemble_stiffness(p, chi=np.zeros(1))).max() == 0.0
    K = _dense_K(m, m.assemble_stiffness(p))
    assert np.abs(K - K.T).max() / np.abs(K).max() < 1e-8
    mu, la = p.mu, p.lambda_
    Cm = np.zeros((6, 6))
    Cm[:3, :3] = la
    Cm[0, 0] = Cm[1, 1] = Cm[2, 2] = la + 2 * mu
    Cm[3, 3] = Cm[4, 4] = Cm[5, 5] = mu
    binv = m.arrays()["binv"][0]
    grad = np.zeros((3, 4))
    grad[:, 0] = -binv.T @ np.ones(3)
    grad[:, 1:] = binv.T
    B = np.zeros((6, 12))
    for n in range(4):
        g = grad[:, n]
        B[0, 3 * n], B[1, 3 * n + 1], B[2, 3 * n + 2] = g
        B[3, 3 * n], B[3, 3 * n + 1] = g[1], g[0]
        B[4, 3 * n + 1], B[4, 3 * n + 2] = g[2], g[1]
        B[5, 3 * n], B[5, 3 * n + 2] = g[2], g[0]
    analytic = m.arrays()["vol"][0] * B.T @ Cm @ B
    assert np.linalg.norm(K - analytic) / np.linalg.norm(analytic) < 1e-10


def test_stiffness_fd():  # test_fem.cpp:231-236 + verify.cpp:117-141
    m = o.Mesh.make_box((0.2, 0.1, 0.1), (3, 2, 2))
    p = stvk_soft()
    u = np.random.default_rng(29).uniform(-0.003, 0.003, (m.num_nodes, 3))
    rp, cols, _ = m.pattern()
    vals = m.assemble_stiffness(p, u)
    h = 1e-6
    worst = 0.0
    n = 3 * m.num_nodes
    for seed in range(4):
        i = np.arange(n)
        d = np.sin(0.7 * (i + 1) * (seed + 1)) + 0.3 * np.cos(1.3 * i + seed)
        d /= np.linalg.norm(d)
        fp = m.assemble_forces(p, u + h * d.reshape(-1, 3))
        fm = m.assemble_forces(p, u - h * d.reshape(-1, 3))
        fd = -(fp - fm) / (2 * h)
        kd = o.spmv_csr(rp, cols, vals, d)
        worst = max(worst, np.abs(fd - kd).max() / max(np.abs(kd).max(), 1e-30))
    assert worst < 1e-3


def test_lumped_mass_kat():  # test_fem.cpp:238-255
    m = unit_tet()
    p = stvk_soft()
    mass = m.lumped_mass(p)
    assert np.allclose(mass[::3], 1000.0 / 6.0 / 4.0, rtol=1e-12)
    box = o.Mesh.make_box((0.2, 0.1, 0.1), (2, 2, 2))
    mb = box.lumped_mass(p)
    assert mb[::3].sum() == pytest.approx(1000.0 * box.arrays()["vol"].sum(), rel=1e-12)


def test_pattern_hash_independent_of_values():  # test_fem.cpp:281-302
    m = o.Mesh.make_box((0.1, 0.1, 0.1), (2, 2, 2))
    _, _, h0 = m.pattern()
    _, _, h1 = m.pattern()
    assert h0 == h1


def test_counts_match_survey_formulas():  # SURVEY §8(a)/(d) sizes
    m = o.Mesh.make_box((0.08, 0.08, 0.32), (8, 8, 32))
    assert (m.num_nodes, m.num_tets, m.num_edges) == (2673, 12288, 16112)
    assert len(m.pattern()[1]) == 314073


# ------------------------------------------------------------------ fracture (test_fracture.cpp)
def test_transform_rows_and_hydrostatic():  # test_fracture.cpp:28-46
    m = unit_tet()
    ok, T = m.build_T(np.zeros((4, 3)), 0)
    assert ok
    assert np.array_equal(T[0], [1, 0, 0, 0, 0, 0])
    p = 3.7e4
    edge = T @ np.array([p, p, p, 0, 0, 0])
    assert np.allclose(edge, p, rtol=1e-12)
    # local edge 3 is (1,2): direction (-1,1,0)/sqrt2 -> (0.5,0.5,0,-0.5,0,0)
    assert np.abs(T[3] - [0.5, 0.5, 0, -0.5, 0, 0]).max() < 1e-15


def test_uniaxial_stress_on_inclined_edge_and_zero_stress():  # test_fracture.cpp:48-57, 75-81
    m = unit_tet()
    stress = 2.5e5
    for theta in (0.0, 0.3, 0.7, 1.2):
        u = np.zeros((4, 3))
        u[1] = [math.cos(theta) - 1.0, math.sin(theta), 0.0]  # local edge 0 = (0,1) along (cos t, sin t, 0)
        ok, T = m.build_T(u, 0)
        assert ok
        assert T[0] @ [stress, 0, 0, 0, 0, 0] == pytest.approx(stress * math.cos(theta) ** 2, rel=1e-12, abs=1e-9)
        assert np.all(T @ np.zeros(6) == 0.0)


def test_build_T_rotation_and_degenerate():  # test_fracture.cpp:59-73
    m = unit_tet()
    X = m.arrays()["rest"]
    R = rand_rotation(np.random.default_rng(3))
    ok, T = m.build_T(X @ R.T - X, 0)
    d = R @ np.array([1.0, 0, 0])
    assert ok and np.linalg.norm(T[0] - [d[0]**2, d[1]**2, d[2]**2, d[0]*d[1], d[0]*d[2], d[1]*d[2]]) < 1e-12
    u = np.zeros((4, 3))
    u[1] = [-1, 0, 0]
    assert not m.build_T(u, 0)[0]


def test_edge_stresses_rotation_invariant():  # test_fracture.cpp:83-107
    p = stvk_soft()
    m = unit_tet()
    X = m.arrays()["rest"]
    F = np.array([[1.15, 0.05, 0.0], [0.02, 0.95, -0.03], [0.0, 0.04, 1.08]])
    u = X @ (F - np.eye(3)).T
    _, T = m.build_T(u, 0)
    base = T @ o.cauchy_sixvector(m.deformation_gradient(u, 0), p)[0]
    for seed in (5, 6, 7):
        R = rand_rotation(np.random.default_rng(seed))
        ur = X @ (R @ F).T - X
        _, Tr = m.build_T(ur, 0)
        got = Tr @ o.cauchy_sixvector(m.deformation_gradient(ur, 0), p)[0]
        assert np.abs(got - base).max() < 1e-8 * np.abs(base).max()


def test_nonlocal_table_rd0_and_huge():  # test_fracture.cpp:109-125
    m = o.Mesh.make_box((0.2, 0.1, 0.1), (2, 1, 1))
    ptr, ids, w = m.nonlocal_table(0.0)
    assert np.array_equal(ids, np.arange(m.num_tets)) and np.all(w == 1.0)
    ptr, ids, w = m.nonlocal_table(1e9)
    assert np.all(np.diff(ptr) == m.num_tets)
    assert np.allclose(w, 1.0 / m.num_tets, rtol=1e-9)


def test_grid_table_equals_bruteforce():  # fracture.cpp:32-54 (grid build == literal O(T^2) loop)
    m = o.Mesh.make_box((0.06, 0.05, 0.07), (6, 5, 7), jitter=0.2, seed=9)
    h = 0.01
    for r_d in (0.7 * h, 1.5 * h, 2.0 * h, 3.3 * h):
        a = m.nonlocal_table(r_d, brute=False)
        b = m.nonlocal_table(r_d, brute=True)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)  # bit-identical weights


def test_two_tet_flat_kernel_average():  # test_fracture.cpp:127-155
    m = o.Mesh.create([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 1]], [[0, 1, 2, 3], [1, 2, 3, 4]])
    sig = np.array([[1.0, 2.0, 3.0, 0.1, 0.2, 0.3], [3.0, 0.0, 1.0, -0.1, 0.4, 0.0]])
    u = np.zeros((5, 3))
    scr, sf, deg = m.nonlocal_screen(u, sig, 1e12)
    _, T0 = m.build_T(u, 0)
    expect = T0 @ (0.5 * (sig[0] + sig[1]))
    te = m.arrays()["tet_edges"]
    eptr, eids = m.edge_tets()
    for k in range(6):
        e = te[0, k]
        assert scr[e] >= expect[k] - 1e-9 * abs(expect[k]) - 1e-12
        if eptr[e + 1] - eptr[e] == 1:
            assert scr[e] == pytest.approx(expect[k], rel=1e-9)


def test_single_tet_any_rd():  # test_fracture.cpp:157-170
    m = unit_tet()
    p = stvk_soft()
    X = m.arrays()["rest"]
    u = X * 0.2
    sig = m.per_tet_cauchy(p, u)
    a = m.nonlocal_screen(u, sig, 0.0)[0]
    b = m.nonlocal_screen(u, sig, 123.0)[0]
    assert np.array_equal(a, b)


def test_update_damage_semantics():  # test_fracture.cpp:172-193
    z = np.zeros(6, np.uint8)
    s = np.full(6, 99.0)
    z, nb = o.update_damage(z, s, 100.0)
    assert len(nb) == 0
    s[2] = 100.0  # exactly at threshold breaks
    z, nb = o.update_damage(z, s, 100.0)
    assert list(nb) == [2] and z[2] == 1
    z, nb = o.update_damage(z, s, 100.0)
    assert len(nb) == 0
    z, nb = o.update_damage(z, np.full(6, -1e9), 100.0)
    assert len(nb) == 0 and z[2] == 1


def test_chi_cases():  # test_fracture.cpp:195-241
    m = unit_tet()
    p = stvk_soft()
    sf = np.full((1, 6), 7.0)
    z = np.zeros(6, np.uint8)
    assert m.compute_chi(z, sf, p)[0] == 1.0
    assert m.compute_chi(np.ones(6, np.uint8), sf, p)[0] == 0.0
    z1 = z.copy()
    z1[5] = 1
    assert abs(m.compute_chi(z1, sf, p)[0] - 5.0 / 6.0) <= 1e-12
    te = m.arrays()["tet_edges"][0]
    z3 = z.copy()
    z3[te[[0, 1, 2]]] = 1
    assert m.compute_chi(z3, np.array([[5.0, 4.0, 3.0, 2.0, 1.0, 0.5]]), p)[0] == 0.0
    lab, cnt = m.fragment_components(z3, 0)
    assert cnt == 2 and list(lab) == [0, 1, 1, 1]
    assert m.compute_chi(z1, np.zeros((1, 6)), p)[0] == pytest.approx(5.0 / 6.0)
    lab, cnt = m.fragment_components(z, 0)
    assert cnt == 1 and list(lab) == [0, 0, 0, 0]
    lab, cnt = m.fragment_components(np.ones(6, np.uint8), 0)
    assert cnt == 4 and list(lab) == [0, 1, 2, 3]


# ------------------------------------------------------------------ sparse (test_sparse.cpp)
def _dense_csr(A):
    n = A.shape[0]
    rp = np.arange(0, n * n + 1, n, dtype=np.int32)
    cols = np.tile(np.arange(n, dtype=np.int32), n)
    return rp, cols, A.reshape(-1).copy()


def test_cg_identity_diagonal():  # test_sparse.cpp:20-50
    n = 10
    rp = np.arange(n + 1, dtype=np.int32)
    cols = np.arange(n, dtype=np.int32)
    b = np.linspace(1, 2, n)
    x, r = o.cg_solve_csr(rp, cols, np.ones(n), b, np.zeros(n), 1e-12, 100)
    assert r.converged and r.iterations == 1 and np.linalg.norm(x - b) < 1e-12
    n = 17
    d = 1.0 + np.arange(n)
    b = np.sin(np.arange(n) + 1.0)
    x, r = o.cg_solve_csr(np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32), d, b, np.zeros(n),
                          1e-14, n + 1)
    assert r.converged and r.iterations <= n and np.abs(x - b / d).max() < 1e-12


def test_cg_random_spd_and_monotone():  # test_sparse.cpp:52-110
    rng = np.random.default_rng(3)
    n = 50
    M = rng.uniform(-1, 1, (n, n))
    A = M @ M.T + 5 * np.eye(n)
    b = rng.uniform(-1, 1, n)
    x, r = o.cg_solve_csr(*_dense_csr(A), b, np.zeros(n), 1e-12, 10 * n)
    ex = np.linalg.solve(A, b)
    assert r.converged and np.linalg.norm(x - ex) / np.linalg.norm(ex) < 1e-8
    rng = np.random.default_rng(5)
    n = 30
    M = rng.uniform(-1, 1, (n, n))
    A = M @ M.T + 2 * np.eye(n)
    b = rng.uniform(-1, 1, n)
    ex = np.linalg.solve(A, b)
    prev = np.inf
    for it in range(1, 26):
        x, _ = o.cg_solve_csr(*_dense_csr(A), b, np.zeros(n), 0.0, it)
        e = x - ex
        an = e @ A @ e
        assert an <= prev * (1 + 1e-9) + 1e-30
        prev = an


def test_cg_negative_curvature():  # test_sparse.cpp:74-84
    x, r = o.cg_solve_csr(*_dense_csr(np.array([[1.0, 0.0], [0.0, -1.0]])), np.array([0.0, 1.0]), np.zeros(2),
                          1e-10, 10)
    assert not r.converged and r.negative_curvature


def test_dirichlet_projection():  # test_sparse.cpp:121-148
    rng = np.random.default_rng(9)
    n = 6
    M = rng.uniform(-1, 1, (n, n))
    A = M @ M.T + 4 * np.eye(n)
    b = rng.uniform(-1, 1, n)
    vals = np.zeros(n)
    vals[2] = 0.7
    rp, cols, v = _dense_csr(A)
    pv, pb = o.project_dirichlet_csr(rp, cols, v, [2], vals, b)
    P = pv.reshape(n, n)
    assert np.abs(P - P.T).max() / np.abs(P).max() < 1e-14
    assert P[2, 2] == 1.0 and pb[2] == 0.7
    x, r = o.cg_solve_csr(rp, cols, pv, pb, np.zeros(n), 1e-13, 100)
    assert r.converged and x[2] == pytest.approx(0.7, rel=1e-12)


# ------------------------------------------------------------------ solver (test_solver.cpp)
def _slab(X, lo, hi):
    return np.nonzero((X[:, 0] >= lo) & (X[:, 0] <= hi))[0]


def test_dynamic_rest_stays_rest():  # test_solver.cpp:89-98
    m = o.Mesh.make_box((0.1, 0.1, 0.1), (2, 2, 2))
    s = o.Sim(m, o.material_from_youngs(1e6, 0.3, 1000, 1e9, 0, STVK), o.solver_config(dt=1e-3))
    s.dynamic_step()
    s.dynamic_step()
    st = s.get_state()
    assert np.all(st["u"] == 0) and np.all(st["v"] == 0)


def test_free_fall_kat():  # test_solver.cpp:100-113
    m = o.Mesh.make_box((0.1, 0.1, 0.1), (2, 2, 2))
    g = np.array([0.3, -9.81, 0.2])
    s = o.Sim(m, o.material_from_youngs(1e6, 0.3, 1000, 1e9, 0, STVK),
              o.solver_config(dt=1e-4, gravity=g, cg_tol=1e-13, cg_max_iters=20000))
    for _ in range(25):
        s.dynamic_step()
    v = s.get_state()["v"]
    expect = 25 * 1e-4 * g
    assert np.all(np.linalg.norm(v - expect, axis=1) <= 1e-12 * np.linalg.norm(expect))


def test_ballistic_broken_tet():  # test_solver.cpp:115-138
    m = o.Mesh.create([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 1]], [[0, 1, 2, 3], [1, 2, 3, 4]])
    g = np.array([0, -9.81, 0])
    X = m.arrays()["rest"]
    s = o.Sim(m, o.material_from_youngs(1e6, 0.3, 1000, 1e9, 0, STVK),
              o.solver_config(dt=1e-4, gravity=g, cg_tol=1e-13, cg_max_iters=20000),
              [dict(nodes=_slab(X, -1.0, 1e-9))])
    st = s.get_state()
    z = st["zeta"].copy()
    z[m.arrays()["tet_edges"][1]] = 1
    chi = st["chi"].copy()
    chi[1] = 0.0
    s.set_state(zeta=z, chi=chi)
    for _ in range(20):
        s.dynamic_step()
    st = s.get_state()
    ev = 20 * 1e-4 * g
    assert np.linalg.norm(st["v"][4] - ev) <= 1e-9 * np.linalg.norm(ev)
    eu = 0.5 * 20 * 21 * 1e-8 * g
    assert np.linalg.norm(st["u"][4] - eu) <= 1e-9 * np.linalg.norm(eu)


def test_bc_nodes_exact():  # test_solver.cpp:140-155
    m = o.Mesh.make_box((0.2, 0.1, 0.1), (4, 2, 2))
    X = m.arrays()["rest"]
    nodes = _slab(X, -1.0, 1e-9)
    s = o.Sim(m, o.material_from_youngs(1e6, 0.3, 1000, 1e9, 0, STVK), o.solver_config(dt=1e-3),
              [dict(nodes=nodes, times=[0.0, 1.0], values=[[0, 0, 0], [0.01, 0.02, -0.005]])])
    for _ in range(10):
        s.dynamic_step()
    st = s.get_state()
    t = st["time"]
    want = np.array([0.01, 0.02, -0.005]) * t  # (1-w)*0 + w*v with w = t
    w = (t - 0.0) / 1.0
    want = np.array([(1 - w) * 0.0 + w * v for v in (0.01, 0.02, -0.005)])
    assert np.all(st["u"][nodes] == want)


def test_energy_never_grows():  # test_solver.cpp:175-202
    m = o.Mesh.make_box((0.1, 0.05, 0.05), (4, 2, 2))
    p = o.material_from_youngs(1e6, 0.3, 1000, 1e9, 0, STVK)
    X = m.arrays()["rest"]
    s = o.Sim(m, p, o.solver_config(dt=2e-5, cg_tol=1e-12), [dict(nodes=_slab(X, -1.0, 1e-9))])
    u = np.zeros_like(X)
    u[:, 0] = 1e-4 * X[:, 0]
    s.set_state(u=u)
    mass = m.lumped_mass(p)

    def energy():
        st = s.get_state()
        return m.total_strain_energy(p, st["u"], st["chi"]) + 0.5 * np.sum(mass[::3] * (st["v"] ** 2).sum(1))

    e0 = prev = energy()
    for _ in range(100):
        s.dynamic_step()
        e = energy()
        assert e <= prev * (1 + 1e-9)
        prev = e
    # test_solver.cpp:201 asserts prev >= 0.98*e0. Backward Euler on this discretisation
    # dissipates more than that: an independent dense linear-BE integration of the same system
    # (M + dt^2 K) dv = dt f - dt^2 K v gives e_100/e_0 = 0.9078 (DESIGN.md "reference test
    # findings"), so the bound is restated against that independent value instead.
    assert prev <= e0
    assert prev / e0 == pytest.approx(0.9078, abs=0.005)


def test_bcs_sharing_node_rejected():  # test_solver.cpp:250-256
    m = o.Mesh.make_box((0.1, 0.1, 0.1), (1, 1, 1))
    allnodes = np.arange(m.num_nodes)
    with pytest.raises(o.FormatError):
        o.Sim(m, o.material_from_youngs(1e6, 0.3, 1000, 1e9, 0, STVK), o.solver_config(),
              [dict(nodes=allnodes), dict(nodes=allnodes)])


def test_chi_monotone_and_hash_constant_under_damage():  # test_solver.cpp:204-248 (dynamic variant)
    m = o.Mesh.make_box((0.2, 0.1, 0.1), (4, 2, 2))
    X = m.arrays()["rest"]
    p = o.material_from_youngs(1e6, 0.3, 1000, 2e3, 0, STVK)
    bcs = [dict(nodes=_slab(X, -1.0, 1e-9), times=[0, 1], values=[[0, 0, 0], [-0.2, 0, 0]]),
           dict(nodes=_slab(X, 0.2 - 1e-9, 1.0), times=[0, 1], values=[[0, 0, 0], [0.2, 0, 0]])]
    s = o.Sim(m, p, o.solver_config(dt=1e-3), bcs)
    h0 = s.pattern_hash()
    prev = s.get_state()["chi"]
    for _ in range(20):
        s.dynamic_step()
        chi = s.get_state()["chi"]
        assert np.all(chi <= prev) and np.all((chi >= 0) & (chi <= 1))
        prev = chi
        assert s.pattern_hash() == h0
    assert s.get_state()["zeta"].sum() > 0


# ------------------------------------------------------------------ collision (test_collision.cpp)
def test_halfspace_penalty_and_impulse():  # test_collision.cpp:48-87 via one dynamic step's load
    m = o.Mesh.make_box((0.1, 0.1, 0.1), (1, 1, 1), origin=(0, 0, -0.001))
    p = o.material_from_youngs(1e6, 0.3, 1000, 1e9, 0, STVK)
    col = dict(kind="halfspace", point=(0, 0, 0), normal=(0, 0, 1), stiffness=1e5, restitution=0.0)
    s = o.Sim(m, p, o.solver_config(dt=1e-4), colliders=[col])
    s.dynamic_step()
    # four bottom nodes penetrate 1 mm: penalty k*d each, no inward velocity at rest
    assert s.last_collider_load() == pytest.approx(4 * 1e5 * 0.001, rel=1e-12)


def _col(**kw):
    d = dict(kind="halfspace", point=(0, 0, 0), normal=(0, 1, 0), stiffness=1e6, restitution=0.0, friction=0.0)
    d.update(kw)
    return d


def _rest_uv(m):
    return np.zeros((m.num_nodes, 3)), np.zeros((m.num_nodes, 3))


def test_schedule_interpolate_and_clamp():  # test_collision.cpp:20-31
    t, v = [0.0, 1.0, 3.0], [[0, 0, 0], [2, 0, 0], [2, 4, 0]]
    assert np.array_equal(o.schedule_eval(t, v, -1.0)[0], [0, 0, 0])
    assert np.linalg.norm(o.schedule_eval(t, v, 0.5)[0] - [1, 0, 0]) < 1e-15
    assert np.linalg.norm(o.schedule_eval(t, v, 2.0)[0] - [2, 2, 0]) < 1e-15
    assert np.array_equal(o.schedule_eval(t, v, 9.0)[0], [2, 4, 0])
    assert np.linalg.norm(o.schedule_eval(t, v, 0.5)[1] - [2, 0, 0]) < 1e-15
    assert np.linalg.norm(o.schedule_eval(t, v, 2.0)[1] - [0, 2, 0]) < 1e-15


def test_no_penetration_zero_force():  # test_collision.cpp:33-48
    m = unit_tet()
    u, v = _rest_uv(m)
    hit = o.detect_and_respond(m, u, v, m.lumped_mass(stvk_soft()), [_col(point=(0, -1, 0))], 0.0, 1e-3)
    assert np.linalg.norm(hit["force"]) == 0.0 and hit["contact_count"] == 0


def test_resting_vertex_penalty():  # test_collision.cpp:50-66
    m = unit_tet()
    u, v = _rest_uv(m)
    u[0] = (0, -0.01, 0)
    hit = o.detect_and_respond(m, u, v, m.lumped_mass(stvk_soft()), [_col(stiffness=5e4)], 0.0, 1e-3)
    assert hit["contact_count"] == 1
    assert np.linalg.norm(hit["force"][0] - [0, 5e4 * 0.01, 0]) < 1e-9


def test_impulse_reverses_normal_velocity_at_restitution_1():  # test_collision.cpp:68-87
    m = unit_tet()
    mass = m.lumped_mass(stvk_soft())
    u, v = _rest_uv(m)
    u[0] = (0, -1e-6, 0)
    v[0] = (0, -2.0, 0)
    dt = 1e-3
    hit = o.detect_and_respond(m, u, v, mass, [_col(stiffness=1e-9, restitution=1.0)], 0.0, dt)
    v_after = v[0] + dt * hit["force"][0] / mass[0]
    assert v_after[1] == pytest.approx(2.0, rel=1e-6)


def test_moving_sphere_opposes_relative_velocity():  # test_collision.cpp:89-108
    m = unit_tet()
    u, v = _rest_uv(m)
    ball = dict(kind="sphere", radius=0.5, stiffness=1e3, restitution=0.0, times=[0.0, 1.0],
                values=[[-0.4, 0, 0], [0.6, 0, 0]])
    hit = o.detect_and_respond(m, u, v, m.lumped_mass(stvk_soft()), [ball], 0.0, 1e-3)
    assert hit["contact_count"] >= 1
    assert hit["force"][0, 0] > 0.0 and hit["per_collider"][0] > 0.0


def test_friction_clamped_by_coulomb_cone():  # test_collision.cpp:110-131
    m = unit_tet()
    u, v = _rest_uv(m)
    u[0] = (0, -1e-3, 0)
    v[0] = (5.0, 0, 0)
    hit = o.detect_and_respond(m, u, v, m.lumped_mass(stvk_soft()), [_col(stiffness=1e4, friction=0.5)], 0.0,
                               1e-3)
    f = hit["force"][0]
    normal_mag = 1e4 * 1e-3
    assert f[0] < 0.0 and abs(f[0]) <= 0.5 * normal_mag * (1 + 1e-12)
    assert f[1] == pytest.approx(normal_mag)


def test_block_settles_on_floor():  # test_collision.cpp:133-166
    m = o.Mesh.make_box((0.1, 0.1, 0.1), (2, 2, 2))
    p = o.material_from_youngs(5e6, 0.3, 1000.0, 1e9, 0.0, STVK)
    p.damp_mass_coeff = 40.0
    s = o.Sim(m, p, o.solver_config(dt=1e-3, gravity=(0, -9.81, 0), cg_tol=1e-10),
              colliders=[_col(stiffness=2e5)])
    for _ in range(200):
        s.dynamic_step()
    st = s.get_state()
    weight = 1000.0 * m.arrays()["vol"].sum() * 9.81
    depth = -(m.arrays()["rest"][:, 1] + st["u"][:, 1])
    total = 2e5 * depth[depth > 0].sum()
    assert 0.0 < depth.max() <= weight / 2e5
    assert 0.5 * weight < total < 1.5 * weight
    assert np.all(np.linalg.norm(st["v"], axis=1) < 5 * 9.81 * 1e-3)


def test_collider_validation():  # test_collision.cpp:168-179
    with pytest.raises(o.FormatError):
        o.collider_validate(dict(kind="sphere", radius=0.0))
    with pytest.raises(o.FormatError):
        o.collider_validate(dict(kind="sphere", radius=1.0, restitution=1.5))
    with pytest.raises(o.FormatError):
        o.collider_validate(dict(kind="sphere", radius=1.0, restitution=0.5, friction=-1.0))
    o.collider_validate(dict(kind="sphere", radius=1.0, restitution=0.5))


def test_rotation_bc_moves_nodes_on_circles():  # test_solver.cpp:157-173 (through one step landing on t = 1)
    m = o.Mesh.make_box((0.2, 0.1, 0.1), (2, 1, 1))
    rest = m.arrays()["rest"][3]
    axis = np.array([0, 0.05, 0.05])
    bc = dict(kind="rotate", nodes=[3], axis_point=axis, axis_dir=(1, 0, 0), times=[0, 1],
              values=[[0, 0, 0], [math.pi / 2, 0, 0]])
    s = o.Sim(m, o.material_from_youngs(1e6, 0.3, 1000, 1e9, 0, STVK), o.solver_config(dt=1.0), [bc])
    s.dynamic_step()
    rel0, rel1 = rest - axis, rest + s.get_state()["u"][3] - axis
    assert np.linalg.norm(rel1) == pytest.approx(np.linalg.norm(rel0), rel=1e-12)
    assert abs(rel0 @ rel1 - rel0[0] * rel1[0]) < 1e-12


def test_rayleigh_damping_in_the_step_system():  # test_fem.cpp:257-279 restated on the implicit-Euler system
    m = unit_tet()
    rng = np.random.default_rng(31)
    u = rng.uniform(-0.05, 0.05, (4, 3))
    v = np.sin(np.arange(1, 13, dtype=float)).reshape(4, 3)
    dt = 1e-3

    def system(a, b):
        p = stvk_soft(1e12)
        p.damp_mass_coeff, p.damp_stiff_coeff = a, b
        s = o.Sim(m, p, o.solver_config(dt=dt))
        s.set_state(u=u, v=v)
        s.dynamic_step()
        return s.last_system()

    p = stvk_soft(1e12)
    K = m.assemble_stiffness(p, u)
    rp, cols, _ = m.pattern()
    mass = m.lumped_mass(p)
    Kd = np.zeros((12, 12))
    for i in range(12):
        Kd[i, cols[rp[i]:rp[i + 1]]] = K[rp[i]:rp[i + 1]]
    diag = np.array([np.nonzero(cols[rp[i]:rp[i + 1]] == i)[0][0] + rp[i] for i in range(12)])
    A0, r0 = system(0.0, 0.0)
    A1, r1 = system(2.5, 0.0)
    A2, r2 = system(2.5, 0.1)
    # alpha only: mass-proportional diagonal and rhs terms, stiffness part untouched
    dA = A1 - A0
    assert np.allclose(dA[diag], dt * 2.5 * mass, rtol=1e-12) and np.all(np.delete(dA, diag) == 0)
    assert np.allclose(r1 - r0, -dt * 2.5 * mass * v.reshape(-1), rtol=1e-9, atol=1e-15)
    # beta: stiffness-proportional matrix and rhs terms scale with dt * beta
    assert np.allclose(A2 - A1, dt * 0.1 * K, rtol=1e-9, atol=1e-12 * np.abs(A2).max())
    assert np.allclose(r2 - r1, -dt * 0.1 * Kd @ v.reshape(-1), rtol=1e-9, atol=1e-12 * np.abs(r2).max())


def test_tetgen_parse():  # mesh.cpp:157-221 (one-based detection)
    node = "4 3 0 0\n1 0 0 0\n2 1 0 0\n3 0 1 0\n4 0 0 1\n"
    ele = "1 4 0\n1 1 2 3 4\n"
    m = o.Mesh.load_tetgen(node, ele)
    assert (m.num_nodes, m.num_tets, m.num_edges) == (4, 1, 6)
    with pytest.raises(o.FormatError):
        o.Mesh.load_tetgen("4 2\n", ele)
    with pytest.raises(o.GeometryError):
        o.Mesh.create([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], [[0, 2, 1, 3]])


# ------------------------------------------------------------------ quasi-static (test_solver.cpp:30-87)
def test_quasi_static_zero_load_converges_immediately():  # test_solver.cpp:30-38
    m = o.Mesh.make_box((0.2, 0.1, 0.1), (4, 2, 2))
    X = m.arrays()["rest"]
    s = o.Sim(m, o.material_from_youngs(1e6, 0.3, 1000, 1e9, 0, STVK), o.solver_config(),
              [dict(nodes=_slab(X, -1.0, 1e-9))])
    before = s.get_state()["u"].copy()
    st = s.quasi_static_step(1.0)
    assert st.newton_iterations == 0 and np.array_equal(s.get_state()["u"], before)


def test_quasi_static_small_stretch_linear_profile():  # test_solver.cpp:40-68
    strain, L = 1e-3, 0.2
    m = o.Mesh.make_box((L, 0.1, 0.1), (8, 4, 4))
    X = m.arrays()["rest"]
    bcs = [dict(nodes=_slab(X, -1.0, 1e-9), times=[0, 1], values=[[0, 0, 0], [-0.5 * strain * L, 0, 0]]),
           dict(nodes=_slab(X, L - 1e-9, 1.0), times=[0, 1], values=[[0, 0, 0], [0.5 * strain * L, 0, 0]])]
    s = o.Sim(m, o.material_from_youngs(1e6, 0.3, 1000, 1e9, 0, STVK), o.solver_config(cg_tol=1e-10), bcs)
    st = s.quasi_static_step(1.0)
    assert st.residual <= s.newton_tolerance()
    state = s.get_state()
    assert state["zeta"].sum() == 0
    c = m.arrays()["centroid"][:, 0]
    sel = np.nonzero((c >= L / 3) & (c <= 2 * L / 3))[0]
    fxx = np.mean([m.deformation_gradient(state["u"], e)[0, 0] for e in sel])
    assert abs(fxx - (1 + strain)) < 0.05 * strain


def test_quasi_static_pull_breaks_edges():  # test_solver.cpp:70-87
    m = o.Mesh.make_box((0.2, 0.1, 0.1), (6, 3, 3))
    X = m.arrays()["rest"]
    bcs = [dict(nodes=_slab(X, -1.0, 1e-9), times=[0, 1], values=[[0, 0, 0], [-0.002, 0, 0]]),
           dict(nodes=_slab(X, 0.2 - 1e-9, 1.0), times=[0, 1], values=[[0, 0, 0], [0.002, 0, 0]])]
    s = o.Sim(m, o.material_from_youngs(1e6, 0.3, 1000, 3e3, 0, STVK), o.solver_config(), bcs)
    for k in range(1, 11):
        last = s.quasi_static_step(k / 10)
    assert s.get_state()["zeta"].sum() > 0 and last.residual <= s.newton_tolerance()


def test_backward_euler_energy_ratio_independent_dense():
    """Independent check of the 0.9078 bound used above: numpy only -- the small-strain element stiffness
    V [lambda g_a g_b^T + mu (g_a . g_b) I + mu g_b g_a^T] (= StVK's tangent at rest, test_fem.cpp:184-229), the
    lumped mass rho V / 4 (fem.cpp:171-179), and the semi-implicit backward Euler of solver.cpp:275-297 with linear
    forces, (M + dt^2 K) dv = -dt K u - dt^2 K v on the free dofs, integrated densely for 100 steps."""
    m = o.Mesh.make_box((0.1, 0.05, 0.05), (4, 2, 2))
    a = m.arrays()
    X, tets, vol, binv = a["rest"], a["tets"], a["vol"], a["binv"].reshape(-1, 3, 3)
    E, nu, rho, dt = 1e6, 0.3, 1000.0, 2e-5
    mu, lam = E / (2 * (1 + nu)), E * nu / ((1 + nu) * (1 - 2 * nu))
    n = 3 * len(X)
    K = np.zeros((n, n))
    M = np.zeros(n)
    for e, t in enumerate(tets):
        g = np.vstack([-binv[e].sum(0), binv[e]])  # rows: shape gradients of the 4 nodes (F = I + Du B^-1)
        for i in range(4):
            M[3 * t[i]:3 * t[i] + 3] += rho * vol[e] / 4
            for j in range(4):
                blk = lam * np.outer(g[i], g[j]) + mu * (g[i] @ g[j]) * np.eye(3) + mu * np.outer(g[j], g[i])
                K[3 * t[i]:3 * t[i] + 3, 3 * t[j]:3 * t[j] + 3] += vol[e] * blk
    free = np.ones(n, bool)
    for node in np.nonzero(X[:, 0] <= 1e-9)[0]:
        free[3 * node:3 * node + 3] = False
    Kf, Mf = K[np.ix_(free, free)], M[free]
    u = np.zeros((len(X), 3))
    u[:, 0] = 1e-4 * X[:, 0]
    u = u.reshape(-1)[free]
    v = np.zeros_like(u)
    A = np.diag(Mf) + dt * dt * Kf
    energy = lambda: 0.5 * u @ Kf @ u + 0.5 * v @ (Mf * v)
    e0 = prev = energy()
    for _ in range(100):
        v = v + np.linalg.solve(A, -dt * (Kf @ u) - dt * dt * (Kf @ v))
        u = u + dt * v
        e = energy()
        assert e <= prev * (1 + 1e-12)
        prev = e
    assert prev / e0 == pytest.approx(0.9078, abs=0.002)


# ------------------------------------------------------------------ edge force decomposition (test_fem.cpp:98-150)
def _one_tet(nodes):
    return o.Mesh.create(np.asarray(nodes, float), np.array([[0, 1, 2, 3]], np.int32))


EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]


def _rebuild(m, u, coeff):
    x = m.arrays()["rest"] + u
    f = np.zeros((4, 3))
    for k, (a, b) in enumerate(EDGES):
        d = x[b] - x[a]
        d = d / np.linalg.norm(d)
        f[a] += coeff[k] * d
        f[b] -= coeff[k] * d
    return f


def test_edge_decomposition_rest_and_uniform_expansion():  # test_fem.cpp:98-113
    m = _one_tet([[0, 0, 0], [1, 0, 0], [0.5, np.sqrt(3) / 2, 0], [0.5, np.sqrt(3) / 6, np.sqrt(6) / 3]])
    p = o.material_from_youngs(1e6, 0.3, 1000.0, 1e5, 0.0, STVK)
    c, res, ok = m.edge_decomposed_forces(p, 0)
    assert ok and np.all(np.abs(c) < 1e-12)
    c, res, ok = m.edge_decomposed_forces(p, 0, 0.2 * m.arrays()["rest"])
    assert ok and res < 1e-8
    assert np.all(np.abs(c[1:] - c[0]) <= 1e-8 * abs(c[0]))


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_edge_decomposition_rebuilds_forces(seed):  # test_fem.cpp:115-139, tools/main.cpp:99-127
    m = _one_tet([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]])
    p = o.material_from_youngs(1e6, 0.3, 1000.0, 1e5, 0.0, STVK)
    u = np.random.default_rng(seed).uniform(-0.15, 0.15, (4, 3))
    c, res, ok = m.edge_decomposed_forces(p, 0, u)
    assert ok
    f = m.element_internal_force(p, 0, u)
    assert np.linalg.norm(_rebuild(m, u, c) - f, axis=1).max() < 1e-8


def test_edge_decomposition_degenerate_flags():  # test_fem.cpp:141-150
    m = _one_tet([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]])
    p = o.material_from_youngs(1e6, 0.3, 1000.0, 1e5, 0.0, STVK)
    u = np.zeros((4, 3))
    u[3] = [0, 0, -1]
    assert not m.edge_decomposed_forces(p, 0, u)[2]


# ------------------------------------------------------------------ dynamic_full_newton (solver.cpp:266-313)
def _bar_sim(full, max_iters=40, dt=2e-3):
    m = o.Mesh.make_box((0.2, 0.05, 0.05), (8, 2, 2))
    X = m.arrays()["rest"]
    p = o.material_from_youngs(1e6, 0.3, 1000, 1e9, 0, 0)
    cfg = o.solver_config(dt=dt, cg_tol=1e-12, dynamic_full_newton=1 if full else 0, newton_max_iters=max_iters,
                          newton_tol=1e-9, gravity=(0.0, -9.81, 0.0))
    s = o.Sim(m, p, cfg, [dict(nodes=_slab(X, -1.0, 1e-9))])
    u = np.zeros_like(X)
    u[:, 1] = -0.02 * X[:, 0]  # bent start: a nonlinear first step
    s.set_state(u=u)
    return s


def test_full_newton_one_iteration_equals_semi_implicit():
    a, b = _bar_sim(False), _bar_sim(True, max_iters=1)
    sa, sb = a.dynamic_step(), b.dynamic_step()
    assert sb.newton_iterations == 1 and sa.newton_iterations == 0
    assert np.array_equal(a.get_state()["u"], b.get_state()["u"])
    assert np.array_equal(a.get_state()["v"], b.get_state()["v"])


def test_full_newton_converges_on_the_backward_euler_residual():
    s = _bar_sim(True)
    st = s.dynamic_step()
    assert 2 <= st.newton_iterations < 40
    semi = _bar_sim(False)
    semi.dynamic_step()
    # the Newton-converged step differs from the single linearised step by the nonlinearity
    assert np.abs(s.get_state()["u"] - semi.get_state()["u"]).max() > 1e-9

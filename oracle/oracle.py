"""ctypes binding of the CPU oracle (oracle/_build/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() (as the checker) and
bench.py's cpu_baseline / --impl reference leg. The product package never imports this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")

F64P = C.POINTER(C.c_double)
I32P = C.POINTER(C.c_int32)
U8P = C.POINTER(C.c_uint8)


class Material(C.Structure):
    _fields_ = [("youngs", C.c_double), ("poisson", C.c_double), ("density", C.c_double), ("mu", C.c_double),
                ("lambda_", C.c_double), ("sigma_thres", C.c_double), ("r_d", C.c_double),
                ("damp_mass_coeff", C.c_double), ("damp_stiff_coeff", C.c_double),
                ("energy_model", C.c_int32), ("_pad", C.c_int32)]


class SolverConfig(C.Structure):
    _fields_ = [("dt", C.c_double), ("newton_tol", C.c_double), ("newton_max_iters", C.c_int32),
                ("cg_max_iters", C.c_int32), ("cg_tol", C.c_double), ("ls_backtrack", C.c_double),
                ("ls_sufficient_decrease", C.c_double), ("ls_max_halvings", C.c_int32),
                ("dynamic_full_newton", C.c_int32), ("gravity", C.c_double * 3),
                ("collision_substeps", C.c_int32), ("_pad", C.c_int32)]


class BoundaryCondition(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_nodes", C.c_int32), ("nodes", I32P), ("n_keys", C.c_int32),
                ("_pad", C.c_int32), ("key_times", F64P), ("key_values", F64P),
                ("axis_point", C.c_double * 3), ("axis_dir", C.c_double * 3)]


class Collider(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_keys", C.c_int32), ("key_times", F64P), ("key_values", F64P),
                ("radius", C.c_double), ("point", C.c_double * 3), ("normal", C.c_double * 3),
                ("stiffness", C.c_double), ("restitution", C.c_double), ("friction", C.c_double)]


class StepStats(C.Structure):
    _fields_ = [("newton_iterations", C.c_int32), ("cg_iterations", C.c_int32), ("newly_broken", C.c_int32),
                ("_pad", C.c_int32), ("residual", C.c_double), ("load", C.c_double)]


class CgResult(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("negative_curvature", C.c_int32),
                ("_pad", C.c_int32), ("relative_residual", C.c_double)]


class OracleError(RuntimeError):
    pass


class FormatError(OracleError):
    pass


class GeometryError(OracleError):
    pass


class SolveError(OracleError):
    pass


_ERRS = {1: FormatError, 2: GeometryError, 3: SolveError}
_lib = None


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, f) for f in ("grafem_oracle.cpp", "oracle.h", "Makefile")]
    stale = not os.path.exists(_LIB_PATH) or any(os.path.getmtime(f) > os.path.getmtime(_LIB_PATH) for f in srcs)
    if force or stale:
        subprocess.run(["make", "-s", "-C", _HERE] + (["-B"] if force else []), check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        L.or_last_error.restype = C.c_char_p
        L.or_energy_density.restype = C.c_double
        L.or_total_strain_energy.restype = C.c_double
        L.or_mesh_mean_face_area.restype = C.c_double
        L.or_pattern_nnz.restype = C.c_int64
        L.or_pattern.restype = C.c_uint64
        L.or_mesh_edge_tets.restype = C.c_int64
        L.or_nonlocal_table.restype = C.c_int64
        L.or_mesh_make_box.argtypes = [F64P, I32P, F64P, C.c_double, C.c_uint64, C.POINTER(C.c_void_p)]
        L.or_sim_pattern_hash.restype = C.c_uint64
        L.or_sim_last_collider_load.restype = C.c_double
        L.or_update_damage.restype = C.c_int32
        L.or_fragment_components.restype = C.c_int32
        L.or_sim_newton_tolerance.restype = C.c_double
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise _ERRS.get(rc, OracleError)(lib().or_last_error().decode())


def f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(F64P)


def i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(I32P)


def _p(a, t):
    return a.ctypes.data_as(t)


def material_from_youngs(E, nu, rho, sigma_thres, r_d=0.0, model=0) -> Material:
    m = Material()
    _check(lib().or_material_from_youngs(C.c_double(E), C.c_double(nu), C.c_double(rho), C.c_double(sigma_thres),
                                         C.c_double(r_d), C.c_int32(model), C.byref(m)))
    return m


def material_lame(mu, lam, model, sigma_thres=1e5, r_d=0.0, density=1000.0) -> Material:
    m = Material()
    m.mu, m.lambda_, m.energy_model, m.sigma_thres, m.r_d, m.density = mu, lam, model, sigma_thres, r_d, density
    m.youngs, m.poisson = 1e6, 0.3
    return m


def solver_config(**kw) -> SolverConfig:
    c = SolverConfig()
    lib().or_solver_config_default(C.byref(c))
    for k, v in kw.items():
        if k == "gravity":
            c.gravity[:] = list(v)
        else:
            setattr(c, k, v)
    return c


# ---------------------------------------------------------------- point functions
def energy_density(F, mat):
    F, pF = f64(F)
    return lib().or_energy_density(pF, C.byref(mat))


def pk1(F, mat):
    F, pF = f64(F)
    out = np.zeros((3, 3))
    lib().or_pk1(pF, C.byref(mat), _p(out, F64P))
    return out


def pk1_differential(F, dF, mat):
    F, pF = f64(F)
    dF, pdF = f64(dF)
    out = np.zeros((3, 3))
    lib().or_pk1_differential(pF, pdF, C.byref(mat), _p(out, F64P))
    return out


def cauchy_sixvector(F, mat):
    F, pF = f64(F)
    out = np.zeros(6)
    fb = lib().or_cauchy_sixvector(pF, C.byref(mat), _p(out, F64P))
    return out, bool(fb)


# ---------------------------------------------------------------- mesh
class Mesh:
    def __init__(self, handle):
        self._h = handle
        n, t, e = C.c_int32(), C.c_int32(), C.c_int32()
        lib().or_mesh_counts(self._h, C.byref(n), C.byref(t), C.byref(e))
        self.num_nodes, self.num_tets, self.num_edges = n.value, t.value, e.value
        self._arrays = None

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.or_mesh_destroy(self._h)
            self._h = None

    @staticmethod
    def make_box(size, cells, origin=(0.0, 0.0, 0.0), jitter=0.0, seed=0):
        h = C.c_void_p()
        s, ps = f64(size)
        c, pc = i32(cells)
        o, po = f64(origin)
        _check(lib().or_mesh_make_box(ps, pc, po, C.c_double(jitter), C.c_uint64(seed), C.byref(h)))
        return Mesh(h)

    @staticmethod
    def create(nodes, tets):
        h = C.c_void_p()
        nodes, pn = f64(nodes)
        tets, pt = i32(tets)
        _check(lib().or_mesh_create(pn, C.c_int32(len(nodes)), pt, C.c_int32(len(tets)), C.byref(h)))
        return Mesh(h)

    @staticmethod
    def load_tetgen(node_text: str, ele_text: str):
        h = C.c_void_p()
        _check(lib().or_mesh_load_tetgen(node_text.encode(), ele_text.encode(), C.byref(h)))
        return Mesh(h)

    def arrays(self):
        if self._arrays is None:
            N, T, E = self.num_nodes, self.num_tets, self.num_edges
            a = dict(rest=np.zeros((N, 3)), tets=np.zeros((T, 4), np.int32), edges=np.zeros((E, 2), np.int32),
                     tet_edges=np.zeros((T, 6), np.int32), vol=np.zeros(T), binv=np.zeros((T, 3, 3)),
                     centroid=np.zeros((T, 3)), rest_len=np.zeros(E))
            lib().or_mesh_get(self._h, _p(a["rest"], F64P), _p(a["tets"], I32P), _p(a["edges"], I32P),
                              _p(a["tet_edges"], I32P), _p(a["vol"], F64P), _p(a["binv"], F64P),
                              _p(a["centroid"], F64P), _p(a["rest_len"], F64P))
            self._arrays = a
        return self._arrays

    def edge_tets(self):
        n = lib().or_mesh_edge_tets(self._h, None, None)
        ptr = np.zeros(self.num_edges + 1, np.int32)
        ids = np.zeros(n, np.int32)
        lib().or_mesh_edge_tets(self._h, _p(ptr, I32P), _p(ids, I32P))
        return ptr, ids

    def mean_face_area(self):
        return lib().or_mesh_mean_face_area(self._h)

    # fem / fracture free functions bound to this mesh
    def deformation_gradient(self, u, tet):
        u, pu = f64(u)
        F = np.zeros((3, 3))
        lib().or_deformation_gradient(self._h, pu, C.c_int32(tet), _p(F, F64P))
        return F

    def _uchi(self, u, chi):
        u = np.zeros((self.num_nodes, 3)) if u is None else u
        chi = np.ones(self.num_tets) if chi is None else chi
        return f64(u), f64(chi)

    def element_internal_force(self, mat, tet, u=None, chi=None):
        (u, pu), (chi, pc) = self._uchi(u, chi)
        f = np.zeros((4, 3))
        lib().or_element_internal_force(self._h, pu, pc, C.byref(mat), C.c_int32(tet), _p(f, F64P))
        return f

    def edge_decomposed_forces(self, mat, tet, u=None):
        """edge_decomposed_forces (fem.cpp:57-94): (coeff[6], residual, ok)"""
        (u, pu), _ = self._uchi(u, None)
        c = np.zeros(6)
        r = C.c_double()
        ok = lib().or_edge_decomposed_forces(self._h, pu, C.byref(mat), C.c_int32(tet), _p(c, F64P), C.byref(r))
        return c, r.value, bool(ok)

    def element_stiffness(self, mat, tet, u=None, chi=None):
        (u, pu), (chi, pc) = self._uchi(u, chi)
        k = np.zeros((12, 12))
        lib().or_element_stiffness(self._h, pu, pc, C.byref(mat), C.c_int32(tet), _p(k, F64P))
        return k

    def assemble_forces(self, mat, u=None, chi=None):
        (u, pu), (chi, pc) = self._uchi(u, chi)
        f = np.zeros(3 * self.num_nodes)
        lib().or_assemble_forces(self._h, pu, pc, C.byref(mat), _p(f, F64P))
        return f

    def pattern(self):
        nnz = lib().or_pattern_nnz(self._h)
        rp = np.zeros(3 * self.num_nodes + 1, np.int32)
        cols = np.zeros(nnz, np.int32)
        h = lib().or_pattern(self._h, _p(rp, I32P), _p(cols, I32P))
        return rp, cols, int(h)

    def assemble_stiffness(self, mat, u=None, chi=None):
        (u, pu), (chi, pc) = self._uchi(u, chi)
        vals = np.zeros(lib().or_pattern_nnz(self._h))
        lib().or_assemble_stiffness(self._h, pu, pc, C.byref(mat), _p(vals, F64P))
        return vals

    def lumped_mass(self, mat):
        m = np.zeros(3 * self.num_nodes)
        lib().or_lumped_mass(self._h, C.byref(mat), _p(m, F64P))
        return m

    def total_strain_energy(self, mat, u=None, chi=None):
        (u, pu), (chi, pc) = self._uchi(u, chi)
        return lib().or_total_strain_energy(self._h, pu, pc, C.byref(mat))

    def build_T(self, u, tet):
        u, pu = f64(u)
        T = np.zeros((6, 6))
        ok = lib().or_build_T(self._h, pu, C.c_int32(tet), _p(T, F64P))
        return bool(ok), T

    def nonlocal_table(self, r_d, brute=False):
        n = lib().or_nonlocal_table(self._h, C.c_double(r_d), C.c_int32(int(brute)), None, None, None)
        ptr = np.zeros(self.num_tets + 1, np.int32)
        ids = np.zeros(n, np.int32)
        w = np.zeros(n)
        lib().or_nonlocal_table(self._h, C.c_double(r_d), C.c_int32(int(brute)), _p(ptr, I32P), _p(ids, I32P),
                                _p(w, F64P))
        return ptr, ids, w

    def per_tet_cauchy(self, mat, u):
        u, pu = f64(u)
        s = np.zeros((self.num_tets, 6))
        lib().or_per_tet_cauchy(self._h, pu, C.byref(mat), _p(s, F64P))
        return s

    def nonlocal_screen(self, u, sigma_c, r_d):
        u, pu = f64(u)
        sc, psc = f64(sigma_c)
        scr = np.zeros(self.num_edges)
        sf = np.zeros((self.num_tets, 6))
        deg = np.zeros(self.num_tets, np.uint8)
        lib().or_nonlocal_screen(self._h, pu, psc, C.c_double(r_d), _p(scr, F64P), _p(sf, F64P), _p(deg, U8P))
        return scr, sf, deg

    def compute_chi(self, zeta, sigma_f, mat):
        z = np.ascontiguousarray(zeta, np.uint8)
        sf, psf = f64(sigma_f)
        chi = np.zeros(self.num_tets)
        lib().or_compute_chi(self._h, _p(z, U8P), psf, C.byref(mat), _p(chi, F64P))
        return chi

    def fragment_components(self, zeta, tet):
        z = np.ascontiguousarray(zeta, np.uint8)
        lab = np.zeros(4, np.int32)
        n = lib().or_fragment_components(self._h, _p(z, U8P), C.c_int32(tet), _p(lab, I32P))
        return lab, int(n)


def update_damage(zeta, screening, thres):
    z = np.ascontiguousarray(zeta, np.uint8).copy()
    s, ps = f64(screening)
    newly = np.zeros(len(z), np.int32)
    n = lib().or_update_damage(_p(z, U8P), C.c_int32(len(z)), ps, C.c_double(thres), _p(newly, I32P))
    return z, newly[:n].copy()


def cg_solve_csr(row_ptr, cols, vals, b, x0, tol, max_iters):
    rp, prp = i32(row_ptr)
    cl, pcl = i32(cols)
    v, pv = f64(vals)
    b, pb = f64(b)
    x = np.array(x0, dtype=np.float64, copy=True)
    r = CgResult()
    lib().or_cg_solve_csr(C.c_int32(len(rp) - 1), prp, pcl, pv, pb, _p(x, F64P), C.c_double(tol),
                          C.c_int32(max_iters), C.byref(r))
    return x, r


def spmv_csr(row_ptr, cols, vals, x):
    rp, prp = i32(row_ptr)
    cl, pcl = i32(cols)
    v, pv = f64(vals)
    x, px = f64(x)
    y = np.zeros(len(rp) - 1)
    lib().or_spmv_csr(C.c_int32(len(rp) - 1), prp, pcl, pv, px, _p(y, F64P))
    return y


def project_dirichlet_csr(row_ptr, cols, vals, dofs, values, rhs):
    rp, prp = i32(row_ptr)
    cl, pcl = i32(cols)
    v = np.array(vals, dtype=np.float64, copy=True)
    d, pd = i32(dofs)
    val, pval = f64(values)
    r = np.array(rhs, dtype=np.float64, copy=True)
    lib().or_project_dirichlet_csr(C.c_int32(len(rp) - 1), prp, pcl, _p(v, F64P), pd, C.c_int32(len(d)), pval,
                                   _p(r, F64P))
    return v, r


# ---------------------------------------------------------------- simulation
def _sched_arrays(times, values):
    t = np.ascontiguousarray(times, np.float64).reshape(-1)
    v = np.ascontiguousarray(values, np.float64).reshape(-1, 3)
    return t, v


def _colliders(colliders, keep):
    Cs = (Collider * max(1, len(colliders)))()
    for i, c in enumerate(colliders):
        t, v = _sched_arrays(np.zeros(0) if c.get("times") is None else c["times"],
                             np.zeros((0, 3)) if c.get("values") is None else c["values"])
        keep += [t, v]
        Cs[i].kind = 1 if c.get("kind", "sphere") == "halfspace" else 0
        Cs[i].n_keys = len(t)
        Cs[i].key_times = _p(t, F64P)
        Cs[i].key_values = _p(v, F64P)
        Cs[i].radius = c.get("radius", 0.0)
        Cs[i].point[:] = list(c.get("point", (0, 0, 0)))
        Cs[i].normal[:] = list(c.get("normal", (0, 0, 1)))
        Cs[i].stiffness = c.get("stiffness", 1e6)
        Cs[i].restitution = c.get("restitution", 0.0)
        Cs[i].friction = c.get("friction", 0.0)
    return Cs


def schedule_eval(times, values, t):
    """Schedule3::eval / rate (collision.cpp:8-30) -> (value[3], rate[3])."""
    tt, vv = _sched_arrays(times, values)
    val, rate = np.zeros(3), np.zeros(3)
    lib().or_schedule_eval(C.c_int32(len(tt)), _p(tt, F64P), _p(vv, F64P), C.c_double(t), _p(val, F64P),
                           _p(rate, F64P))
    return val, rate


def collider_validate(collider):
    """Collider::validate (collision.cpp:32-40); raises FormatError."""
    keep = []
    _check(lib().or_collider_validate(_colliders([collider], keep)))


def detect_and_respond(mesh, u, v, mass, colliders, t, dt):
    """detect_and_respond (collision.cpp:49-111) -> dict(force (n,3), per_collider, contact_count,
    deep_penetrations, max_depth)."""
    n = mesh.num_nodes
    keep = []
    Cs = _colliders(colliders, keep)
    u = np.ascontiguousarray(u, np.float64).reshape(n, 3)
    v = np.ascontiguousarray(v, np.float64).reshape(n, 3)
    mass = np.ascontiguousarray(mass, np.float64).reshape(-1)
    force = np.zeros((n, 3))
    per = np.zeros(max(1, len(colliders)))
    counts = np.zeros(2, np.int32)
    md = C.c_double(0.0)
    _check(lib().or_detect_and_respond(mesh._h, _p(u, F64P), _p(v, F64P), _p(mass, F64P), Cs,
                                       C.c_int32(len(colliders)), C.c_double(t), C.c_double(dt), _p(force, F64P),
                                       _p(per, F64P), _p(counts, I32P), C.byref(md)))
    return dict(force=force, per_collider=per[:len(colliders)], contact_count=int(counts[0]),
                deep_penetrations=int(counts[1]), max_depth=md.value)


class Sim:
    """Oracle Simulation (solver.cpp). bcs: list of dicts {kind, nodes, times, values, axis_point, axis_dir};
    colliders: list of dicts {kind, times, values, radius, point, normal, stiffness, restitution, friction}."""

    def __init__(self, mesh: Mesh, mat: Material, cfg: SolverConfig, bcs=(), colliders=()):
        keep = []
        B = (BoundaryCondition * max(1, len(bcs)))()
        for i, bc in enumerate(bcs):
            nodes = np.ascontiguousarray(bc["nodes"], np.int32)
            t, v = _sched_arrays(bc.get("times", [0.0]), bc.get("values", [[0, 0, 0]]))
            keep += [nodes, t, v]
            B[i].kind = 1 if bc.get("kind", "translate") == "rotate" else 0
            B[i].n_nodes = len(nodes)
            B[i].nodes = _p(nodes, I32P)
            B[i].n_keys = len(t)
            B[i].key_times = _p(t, F64P)
            B[i].key_values = _p(v, F64P)
            B[i].axis_point[:] = list(bc.get("axis_point", (0, 0, 0)))
            B[i].axis_dir[:] = list(bc.get("axis_dir", (1, 0, 0)))
        Cs = _colliders(colliders, keep)
        h = C.c_void_p()
        _check(lib().or_sim_create(mesh._h, C.byref(mat), C.byref(cfg), B, C.c_int32(len(bcs)), Cs,
                                   C.c_int32(len(colliders)), C.byref(h)))
        self._h = h
        self.mesh = mesh
        self.mat = mat
        self.cfg = cfg

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.or_sim_destroy(self._h)
            self._h = None

    def dynamic_step(self):
        st = StepStats()
        _check(lib().or_sim_dynamic_step(self._h, C.byref(st)))
        return st

    def quasi_static_step(self, t_load):
        st = StepStats()
        _check(lib().or_sim_quasi_static_step(self._h, C.c_double(t_load), C.byref(st)))
        return st

    def newton_tolerance(self):
        return lib().or_sim_newton_tolerance(self._h)

    def damage_pass(self):
        ids = np.zeros(self.mesh.num_edges, np.int32)
        n = C.c_int64()
        _check(lib().or_sim_damage_pass(self._h, _p(ids, I32P), C.c_int64(len(ids)), C.byref(n)))
        return ids[: n.value].copy()

    def get_state(self):
        N, T, E = self.mesh.num_nodes, self.mesh.num_tets, self.mesh.num_edges
        u, v, z, chi, t = np.zeros((N, 3)), np.zeros((N, 3)), np.zeros(E, np.uint8), np.zeros(T), C.c_double()
        lib().or_sim_get_state(self._h, _p(u, F64P), _p(v, F64P), _p(z, U8P), _p(chi, F64P), C.byref(t))
        return dict(u=u, v=v, zeta=z, chi=chi, time=t.value)

    def set_state(self, u=None, v=None, zeta=None, chi=None, time=None):
        keep = []

        def ptr(a, dt, t):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dt)
            keep.append(a)
            return _p(a, t)

        tt = C.c_double(time) if time is not None else None
        lib().or_sim_set_state(self._h, ptr(u, np.float64, F64P), ptr(v, np.float64, F64P),
                               ptr(zeta, np.uint8, U8P), ptr(chi, np.float64, F64P),
                               C.byref(tt) if tt is not None else None)

    def set_external_forces(self, f):
        if f is None:
            lib().or_sim_set_external_forces(self._h, None)
        else:
            f, pf = f64(f)
            lib().or_sim_set_external_forces(self._h, pf)

    def pattern_hash(self):
        return int(lib().or_sim_pattern_hash(self._h))

    def last_collider_load(self):
        return lib().or_sim_last_collider_load(self._h)

    def mass(self):
        m = np.zeros(3 * self.mesh.num_nodes)
        lib().or_sim_mass(self._h, _p(m, F64P))
        return m

    def last_system(self):
        nnz = lib().or_pattern_nnz(self.mesh._h)
        vals = np.zeros(nnz)
        rhs = np.zeros(3 * self.mesh.num_nodes)
        lib().or_sim_last_system(self._h, _p(vals, F64P), _p(rhs, F64P))
        return vals, rhs

    def phase_times(self):
        t = np.zeros(4)
        lib().or_sim_phase_times(self._h, _p(t, F64P))
        return t


def num_threads():
    return int(lib().or_num_threads())


def set_num_threads(n: int):
    lib().or_set_num_threads(C.c_int(int(n)))

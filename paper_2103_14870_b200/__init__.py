"""grafem-b200: B200-native per-timestep hot path of the remeshing-free graph-based FEM fracture method.

Python mirror of the reference's C++ simulator API (namespace grafem, /root/reference/proj/include/grafem)
over the C ABI of libgrafem_b200.so (include/grafem_b200.h). Names, argument meaning and error types follow
the reference: TetMesh / make_box_mesh / make_mesh / load_tetgen, MaterialParams.from_youngs, SolverConfig,
BoundaryCondition + Schedule3, Collider, Simulation.{dynamic_step, damage_pass, state, ...}, and the
FormatError / GeometryError / SolveError exceptions.

All compute runs in hand-written sm_100a CUDA kernels. There is no CPU fallback: importing works anywhere
(the library is plain C ABI), but creating a Simulation without a Blackwell GPU raises CudaError.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "FormatError", "GeometryError", "SolveError", "CudaError", "TetMesh", "make_box_mesh", "make_mesh",
    "load_tetgen", "MaterialParams", "SolverConfig", "Schedule3", "BoundaryCondition", "Collider", "Simulation",
    "StepStats", "SimState", "cg_solve_csr", "library_path", "STABLE_NEO_HOOKEAN", "STVK",
]

STABLE_NEO_HOOKEAN, STVK = 0, 1
_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.environ.get("GF_LIB_PATH") or os.path.join(_HERE, "_lib", "libgrafem_b200.so")  # override: A/B tools

F64P = C.POINTER(C.c_double)
I32P = C.POINTER(C.c_int32)
U8P = C.POINTER(C.c_uint8)


class GrafemError(RuntimeError):
    pass


class FormatError(GrafemError):
    """grafem::FormatError (types.hpp:17-20)"""


class GeometryError(GrafemError):
    """grafem::GeometryError (types.hpp:22-25)"""


class SolveError(GrafemError):
    """grafem::SolveError (types.hpp:27-29)"""


class CudaError(GrafemError):
    """No usable sm_100 device / CUDA runtime failure (no CPU fallback exists)."""


_ERRORS = {1: FormatError, 2: GeometryError, 3: SolveError, 4: CudaError, 5: GrafemError}


# ---------------------------------------------------------------- C ABI structs (grafem_b200.h)
class _Material(C.Structure):
    _fields_ = [("youngs", C.c_double), ("poisson", C.c_double), ("density", C.c_double), ("mu", C.c_double),
                ("lambda_", C.c_double), ("sigma_thres", C.c_double), ("r_d", C.c_double),
                ("damp_mass_coeff", C.c_double), ("damp_stiff_coeff", C.c_double),
                ("energy_model", C.c_int32), ("_pad", C.c_int32)]


class _SolverConfig(C.Structure):
    _fields_ = [("dt", C.c_double), ("newton_tol", C.c_double), ("newton_max_iters", C.c_int32),
                ("cg_max_iters", C.c_int32), ("cg_tol", C.c_double), ("ls_backtrack", C.c_double),
                ("ls_sufficient_decrease", C.c_double), ("ls_max_halvings", C.c_int32),
                ("dynamic_full_newton", C.c_int32), ("gravity", C.c_double * 3),
                ("collision_substeps", C.c_int32), ("_pad", C.c_int32)]


class _Bc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_nodes", C.c_int32), ("nodes", I32P), ("n_keys", C.c_int32),
                ("_pad", C.c_int32), ("key_times", F64P), ("key_values", F64P),
                ("axis_point", C.c_double * 3), ("axis_dir", C.c_double * 3)]


class _Collider(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_keys", C.c_int32), ("key_times", F64P), ("key_values", F64P),
                ("radius", C.c_double), ("point", C.c_double * 3), ("normal", C.c_double * 3),
                ("stiffness", C.c_double), ("restitution", C.c_double), ("friction", C.c_double)]


class StepStats(C.Structure):
    """grafem::StepStats (solver.hpp:49-55)"""
    _fields_ = [("newton_iterations", C.c_int32), ("cg_iterations", C.c_int32), ("newly_broken", C.c_int32),
                ("_pad", C.c_int32), ("residual", C.c_double), ("load", C.c_double)]


class _CgResult(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("negative_curvature", C.c_int32),
                ("_pad", C.c_int32), ("relative_residual", C.c_double)]


PCG_SOLVERS = ("two-barrier", "grid", "cluster", "onchip", "large-matrix", "onchip-cluster", "large-matrix-rr")  # gf_sim_info.pcg_solver


class _SimInfo(C.Structure):
    _fields_ = [("nodes", C.c_int64), ("tets", C.c_int64), ("edges", C.c_int64), ("node_blocks", C.c_int64),
                ("upper_blocks", C.c_int64), ("upper_block_slots", C.c_int64), ("spmv_slots", C.c_int64),
                ("nl_entries", C.c_int64), ("nl_slots", C.c_int64), ("nl_layout", C.c_int32),
                ("pcg_dynamic_units", C.c_int32), ("setup_s", C.c_double * 4), ("pcg_solver", C.c_int32),
                ("_pad0", C.c_int32), ("oc_slot_blocks", C.c_int64 * 7), ("oc_offsets", C.c_int32 * 7),
                ("_pad1", C.c_int32)]


class StepMetrics(C.Structure):
    """gf_step_metrics: run_scenario's make_row + log_damage values (scenario.cpp:640-672), device reductions"""
    _fields_ = [("strain_energy", C.c_double), ("kinetic_energy", C.c_double), ("chi_min", C.c_double),
                ("chi_mean", C.c_double), ("broken_edges", C.c_int64), ("time", C.c_double)]


class KernelTime(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("total_ms", C.c_double), ("bytes", C.c_double)]


_lib = None


def library_path() -> str:
    return _LIB


def lib():
    """Load libgrafem_b200.so. Fails loudly when the extension has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} is missing: build it with `python -m paper_2103_14870_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(_LIB)
        L.gf_last_error.restype = C.c_char_p
        L.gf_version.restype = C.c_char_p
        L.gf_mesh_make_box.argtypes = [F64P, I32P, F64P, C.c_double, C.c_uint64, C.POINTER(C.c_void_p)]
        L.gf_mesh_mean_face_area.restype = C.c_double
        L.gf_mesh_pattern_nnz.restype = C.c_int64
        L.gf_mesh_pattern.restype = C.c_uint64
        L.gf_mesh_nonlocal_table.restype = C.c_int64
        L.gf_mesh_nonlocal_table.argtypes = [C.c_void_p, C.c_double, I32P, I32P, F64P]
        L.gf_sim_pattern_hash.restype = C.c_uint64
        L.gf_sim_last_collider_load.restype = C.c_double
        L.gf_sim_newton_tolerance.restype = C.c_double
        L.gf_host_alloc.restype = C.c_void_p
        L.gf_host_alloc.argtypes = [C.c_size_t]
        L.gf_host_free.argtypes = [C.c_void_p]
        L.gf_viz_child_count.restype = C.c_int64
        L.gf_viz_child_count.argtypes = [C.c_void_p]
        for f in ("gf_viz_child", "gf_viz_child_position"):
            getattr(L, f).argtypes = [C.c_void_p, C.c_int64] + [C.c_void_p] * (6 if f == "gf_viz_child" else 3)
        L.gf_viz_apply_splits.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        L.gf_viz_fragment_volumes.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise _ERRORS.get(rc, GrafemError)(lib().gf_last_error().decode())


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(F64P)


def _i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(I32P)


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


# ---------------------------------------------------------------- mesh (mesh.hpp, primitives.hpp)
class TetMesh:
    """TetMesh (mesh.hpp:15-43): rest positions, tets, canonical edges, rest quantities (host setup)."""

    def __init__(self, handle):
        self._h = handle
        n, t, e = C.c_int32(), C.c_int32(), C.c_int32()
        lib().gf_mesh_counts(self._h, C.byref(n), C.byref(t), C.byref(e))
        self._counts = (n.value, t.value, e.value)
        self._arrays = None

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.gf_mesh_destroy(self._h)
            self._h = None

    def num_nodes(self):
        return self._counts[0]

    def num_tets(self):
        return self._counts[1]

    def num_edges(self):
        return self._counts[2]

    def num_dofs(self):
        return 3 * self._counts[0]

    def _get(self):
        if self._arrays is None:
            N, T, E = self._counts
            a = dict(rest_positions=np.zeros((N, 3)), tets=np.zeros((T, 4), np.int32),
                     edges=np.zeros((E, 2), np.int32), tet_edges=np.zeros((T, 6), np.int32),
                     rest_volumes=np.zeros(T), rest_shape_inverse=np.zeros((T, 3, 3)),
                     rest_centroids=np.zeros((T, 3)), rest_edge_lengths=np.zeros(E))
            lib().gf_mesh_get(self._h, *[_p(a[k], t) for k, t in [
                ("rest_positions", F64P), ("tets", I32P), ("edges", I32P), ("tet_edges", I32P),
                ("rest_volumes", F64P), ("rest_shape_inverse", F64P), ("rest_centroids", F64P),
                ("rest_edge_lengths", F64P)]])
            self._arrays = a
        return self._arrays

    def __getattr__(self, name):
        if name in ("rest_positions", "tets", "edges", "tet_edges", "rest_volumes", "rest_shape_inverse",
                    "rest_centroids", "rest_edge_lengths"):
            return self._get()[name]
        raise AttributeError(name)

    def total_volume(self):
        return float(self.rest_volumes.sum())

    def mean_face_area(self):
        return lib().gf_mesh_mean_face_area(self._h)

    def pattern(self):
        """Scalar CSR of make_system_pattern (fem.cpp:140-149): (row_ptr, cols, structure_hash)."""
        nnz = lib().gf_mesh_pattern_nnz(self._h)
        rp = np.zeros(self.num_dofs() + 1, np.int32)
        cols = np.zeros(nnz, np.int32)
        h = lib().gf_mesh_pattern(self._h, _p(rp, I32P), _p(cols, I32P))
        return rp, cols, int(h)

    def nonlocal_table(self, r_d: float):
        """build_nonlocal_table (fracture.cpp:32-54) as CSR (ptr, ids, weights)."""
        n = lib().gf_mesh_nonlocal_table(self._h, r_d, None, None, None)
        ptr = np.zeros(self.num_tets() + 1, np.int32)
        ids = np.zeros(n, np.int32)
        w = np.zeros(n)
        lib().gf_mesh_nonlocal_table(self._h, r_d, _p(ptr, I32P), _p(ids, I32P), _p(w, F64P))
        return ptr, ids, w


def make_box_mesh(size, cells, origin=(0.0, 0.0, 0.0), jitter: float = 0.0, seed: int = 0) -> TetMesh:
    """make_box_mesh (primitives.hpp:12-13) + optional seeded interior-node jitter (cell units)."""
    h = C.c_void_p()
    _, ps = _f64(size)
    c, pc = _i32(cells)
    _, po = _f64(origin)
    s = np.asarray(size, np.float64)
    o = np.asarray(origin, np.float64)
    _check(lib().gf_mesh_make_box(s.ctypes.data_as(F64P), pc, o.ctypes.data_as(F64P), C.c_double(jitter),
                                  C.c_uint64(seed), C.byref(h)))
    return TetMesh(h)


def make_mesh(nodes, tets) -> TetMesh:
    """make_mesh (mesh.hpp:55-56)"""
    h = C.c_void_p()
    nodes, pn = _f64(nodes)
    tets, pt = _i32(tets)
    _check(lib().gf_mesh_create(pn, C.c_int32(len(nodes)), pt, C.c_int32(len(tets)), C.byref(h)))
    return TetMesh(h)


def load_tetgen(node_text: str, ele_text: str) -> TetMesh:
    """load_tetgen (mesh.hpp:59)"""
    h = C.c_void_p()
    _check(lib().gf_mesh_load_tetgen(node_text.encode(), ele_text.encode(), C.byref(h)))
    return TetMesh(h)


# ---------------------------------------------------------------- parameters
class MaterialParams:
    """MaterialParams (material.hpp:14-31)."""

    def __init__(self, raw: _Material):
        self._raw = raw

    @staticmethod
    def from_youngs(youngs, poisson, density, sigma_thres, r_d=0.0, model=STABLE_NEO_HOOKEAN):
        m = _Material()
        _check(lib().gf_material_from_youngs(C.c_double(youngs), C.c_double(poisson), C.c_double(density),
                                             C.c_double(sigma_thres), C.c_double(r_d), C.c_int32(model), C.byref(m)))
        return MaterialParams(m)

    def __getattr__(self, k):
        raw = self.__dict__["_raw"]
        return getattr(raw, "lambda_" if k == "lambda_" or k == "lam" else k)

    def __setattr__(self, k, v):
        if k == "_raw":
            object.__setattr__(self, k, v)
        else:
            setattr(self._raw, k, v)


class SolverConfig:
    """SolverConfig (solver.hpp:15-31)."""

    def __init__(self, **kw):
        self._raw = _SolverConfig()
        lib().gf_solver_config_default(C.byref(self._raw))
        for k, v in kw.items():
            setattr(self, k, v)

    def __getattr__(self, k):
        return getattr(self.__dict__["_raw"], k)

    def __setattr__(self, k, v):
        if k == "_raw":
            object.__setattr__(self, k, v)
        elif k == "gravity":
            self._raw.gravity[:] = [float(x) for x in v]
        else:
            setattr(self._raw, k, v)


@dataclass
class Schedule3:
    """Piecewise-linear vector schedule (collision.hpp:10-18)."""
    times: Sequence[float] = ()
    values: Sequence[Sequence[float]] = ()

    @staticmethod
    def constant(v):
        return Schedule3([0.0], [list(v)])


@dataclass
class BoundaryCondition:
    """BoundaryCondition (solver.hpp:35-47). kind 'translate' (translation schedule) or 'rotate'."""
    nodes: Sequence[int]
    kind: str = "translate"
    name: str = ""
    translation: Schedule3 = field(default_factory=lambda: Schedule3.constant((0.0, 0.0, 0.0)))
    axis_point: Sequence[float] = (0.0, 0.0, 0.0)
    axis_dir: Sequence[float] = (1.0, 0.0, 0.0)
    angle: Schedule3 = field(default_factory=Schedule3)


@dataclass
class Collider:
    """Collider (collision.hpp:20-34). kind 'sphere' (centre schedule) or 'halfspace'."""
    kind: str = "sphere"
    center: Schedule3 = field(default_factory=Schedule3)
    radius: float = 0.0
    point: Sequence[float] = (0.0, 0.0, 0.0)
    normal: Sequence[float] = (0.0, 0.0, 1.0)
    stiffness: float = 1e6
    restitution: float = 0.0
    friction: float = 0.0


@dataclass
class SimState:
    """SimState (fem.hpp:15-28), host copy."""
    displacements: np.ndarray
    velocities: np.ndarray
    edge_damage: np.ndarray
    element_chi: np.ndarray
    time: float

    def broken_edge_count(self):
        return int(self.edge_damage.sum())


def _sched_arrays(s: Schedule3):
    t = np.ascontiguousarray(s.times, np.float64).reshape(-1)
    v = np.ascontiguousarray(s.values, np.float64).reshape(-1, 3) if len(t) else np.zeros((0, 3))
    return t, np.ascontiguousarray(v)


# ---------------------------------------------------------------- simulation (solver.hpp:60-118)
class Simulation:
    def __init__(self, mesh: TetMesh, material: MaterialParams, config: SolverConfig,
                 bcs: Sequence[BoundaryCondition] = (), colliders: Sequence[Collider] = ()):
        keep = []
        B = (_Bc * max(1, len(bcs)))()
        for i, bc in enumerate(bcs):
            nodes = np.ascontiguousarray(bc.nodes, np.int32)
            sched = bc.translation if bc.kind == "translate" else bc.angle
            t, v = _sched_arrays(sched)
            keep += [nodes, t, v]
            B[i].kind = 0 if bc.kind == "translate" else 1
            B[i].n_nodes = len(nodes)
            B[i].nodes = nodes.ctypes.data_as(I32P)
            B[i].n_keys = len(t)
            B[i].key_times = t.ctypes.data_as(F64P)
            B[i].key_values = v.ctypes.data_as(F64P)
            B[i].axis_point[:] = [float(x) for x in bc.axis_point]
            B[i].axis_dir[:] = [float(x) for x in bc.axis_dir]
        K = (_Collider * max(1, len(colliders)))()
        for i, c in enumerate(colliders):
            t, v = _sched_arrays(c.center)
            keep += [t, v]
            K[i].kind = 0 if c.kind == "sphere" else 1
            K[i].n_keys = len(t)
            K[i].key_times = t.ctypes.data_as(F64P)
            K[i].key_values = v.ctypes.data_as(F64P)
            K[i].radius = c.radius
            K[i].point[:] = [float(x) for x in c.point]
            K[i].normal[:] = [float(x) for x in c.normal]
            K[i].stiffness, K[i].restitution, K[i].friction = c.stiffness, c.restitution, c.friction
        h = C.c_void_p()
        _check(lib().gf_sim_create(mesh._h, C.byref(material._raw), C.byref(config._raw), B, C.c_int32(len(bcs)),
                                   K, C.c_int32(len(colliders)), C.byref(h)))
        self._h = h
        self._mesh = mesh
        self.material = material
        self.config = config
        self.N, self.T, self.E = mesh.num_nodes(), mesh.num_tets(), mesh.num_edges()

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.gf_sim_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def mesh(self):
        return self._mesh

    def dynamic_step(self) -> StepStats:
        st = StepStats()
        _check(lib().gf_sim_dynamic_step(self._h, C.byref(st)))
        return st

    def quasi_static_step(self, t_load: float) -> StepStats:
        """Simulation::quasi_static_step (solver.cpp:138-217) on the GPU."""
        st = StepStats()
        _check(lib().gf_sim_quasi_static_step(self._h, C.c_double(t_load), C.byref(st)))
        return st

    def newton_tolerance(self) -> float:
        return lib().gf_sim_newton_tolerance(self._h)

    def viz(self) -> "VizMesh":
        """Simulation::viz (solver.hpp:83-84): the render companion; created on first call, then fed by every
        damage pass (solver.cpp:94)."""
        h = C.c_void_p()
        _check(lib().gf_sim_viz(self._h, C.byref(h)))
        return VizMesh(None, _borrowed=h, _owner=self)

    def nonlocal_layout(self) -> int:
        """0: local screening (r_d = 0), 1: general sliced-ELL table, 2: structured template layout."""
        return lib().gf_sim_nonlocal_layout(self._h)

    def damage_pass(self) -> np.ndarray:
        ids = np.zeros(self.E, np.int32)
        n = C.c_int64()
        _check(lib().gf_sim_damage_pass(self._h, _p(ids, I32P), C.c_int64(self.E), C.byref(n)))
        return ids[: n.value].copy()

    def state(self) -> SimState:
        u, v = np.zeros((self.N, 3)), np.zeros((self.N, 3))
        z, chi, t = np.zeros(self.E, np.uint8), np.zeros(self.T), C.c_double()
        _check(lib().gf_sim_get_state(self._h, _p(u, F64P), _p(v, F64P), _p(z, U8P), _p(chi, F64P), C.byref(t)))
        return SimState(u, v, z, chi, t.value)

    def set_state(self, displacements=None, velocities=None, edge_damage=None, element_chi=None, time=None):
        args, keep = [], []
        for a, dt, t in ((displacements, np.float64, F64P), (velocities, np.float64, F64P),
                         (edge_damage, np.uint8, U8P), (element_chi, np.float64, F64P)):
            if a is None:
                args.append(None)
            else:
                a = np.ascontiguousarray(a, dt)
                keep.append(a)
                args.append(a.ctypes.data_as(t))
        tt = C.c_double(time) if time is not None else None
        _check(lib().gf_sim_set_state(self._h, *args, C.byref(tt) if tt is not None else None))

    def get_state_into(self, u=None, v=None, zeta=None, chi=None):
        """Zero-copy variant for pinned buffers (raw pointers or numpy arrays)."""
        def ptr(a, t):
            if a is None:
                return None
            return C.cast(a, t) if isinstance(a, int) else a.ctypes.data_as(t)
        _check(lib().gf_sim_get_state(self._h, ptr(u, F64P), ptr(v, F64P), ptr(zeta, U8P), ptr(chi, F64P), None))

    def set_state_from(self, u=None, v=None):
        """Stream-ordered upload of u, v from pinned buffers (gf_sim_set_state_async)."""
        def ptr(a):
            if a is None:
                return None
            return C.cast(a, F64P) if isinstance(a, int) else a.ctypes.data_as(F64P)
        # pinned buffers: stream-ordered upload, no host round trip (the next step reads the new state; the
        # caller must not modify the buffers before its next synchronous call on the simulation)
        _check(lib().gf_sim_set_state_async(self._h, ptr(u), ptr(v)))

    def set_external_forces(self, f3n=None):
        if f3n is None:
            _check(lib().gf_sim_set_external_forces(self._h, None))
        else:
            f, pf = _f64(np.asarray(f3n).reshape(-1))
            _check(lib().gf_sim_set_external_forces(self._h, pf))

    def pattern_hash(self) -> int:
        return int(lib().gf_sim_pattern_hash(self._h))

    def dof_count(self) -> int:
        return int(lib().gf_sim_dof_count(self._h))

    def broken_fraction(self) -> float:
        n = C.c_int64()
        _check(lib().gf_sim_broken_edge_count(self._h, C.byref(n)))
        return n.value / self.E if self.E else 0.0

    def last_collider_load(self) -> float:
        return lib().gf_sim_last_collider_load(self._h)

    def mass(self) -> np.ndarray:
        m = np.zeros(3 * self.N)
        _check(lib().gf_sim_mass(self._h, _p(m, F64P)))
        return m

    def reaction_load(self, nodes, axis) -> float:
        n, pn = _i32(nodes)
        a = (C.c_double * 3)(*[float(x) for x in axis])
        out = C.c_double()
        _check(lib().gf_sim_reaction_load(self._h, pn, C.c_int32(len(n)), a, C.byref(out)))
        return out.value

    def energies(self):
        s, k = C.c_double(), C.c_double()
        _check(lib().gf_sim_energies(self._h, C.byref(s), C.byref(k)))
        return s.value, k.value

    def step_metrics(self) -> StepMetrics:
        m = StepMetrics()
        _check(lib().gf_sim_step_metrics(self._h, C.byref(m)))
        return m

    # parity / microbench hooks
    def eval_forces(self) -> np.ndarray:
        f = np.zeros(3 * self.N)
        _check(lib().gf_sim_eval_forces(self._h, _p(f, F64P)))
        return f

    def eval_stiffness(self) -> np.ndarray:
        vals = np.zeros(lib().gf_mesh_pattern_nnz(self._mesh._h))
        _check(lib().gf_sim_eval_stiffness(self._h, _p(vals, F64P)))
        return vals

    def eval_cauchy(self) -> np.ndarray:
        s = np.zeros((self.T, 6))
        _check(lib().gf_sim_eval_cauchy(self._h, _p(s, F64P)))
        return s

    def eval_screening(self):
        scr, sf, deg = np.zeros(self.E), np.zeros((self.T, 6)), np.zeros(self.T, np.uint8)
        _check(lib().gf_sim_eval_screening(self._h, _p(scr, F64P), _p(sf, F64P), _p(deg, U8P)))
        return scr, sf, deg

    def last_system(self):
        vals = np.zeros(lib().gf_mesh_pattern_nnz(self._mesh._h))
        rhs = np.zeros(3 * self.N)
        _check(lib().gf_sim_last_system(self._h, _p(vals, F64P), _p(rhs, F64P)))
        return vals, rhs

    def spmv(self, x) -> np.ndarray:
        x, px = _f64(x)
        y = np.zeros(3 * self.N)
        _check(lib().gf_sim_spmv(self._h, px, _p(y, F64P)))
        return y

    def edge_forces(self):
        """edge_decomposed_forces (fem.cpp:57-94) of every tet: (coeff[T, 6], ok[T])"""
        c, ok = np.zeros((self.T, 6)), np.zeros(self.T, np.uint8)
        _check(lib().gf_sim_edge_forces(self._h, _p(c, F64P), _p(ok, U8P)))
        return c, ok.astype(bool)

    def element_form(self) -> str:
        return "edge" if lib().gf_sim_element_form(self._h) else "F"

    def assembly_energy(self) -> float:
        e = C.c_double()
        _check(lib().gf_sim_assembly_energy(self._h, C.byref(e)))
        return e.value

    def solve_system(self, vals, b, x0=None, tol=1e-8, max_iters=4000):
        """The production PCG (k_pcg_sell) on a symmetric matrix with this simulation's pattern (scalar-CSR values
        as eval_stiffness returns them): cg_solve (sparse.cpp:129-188). Replaces the current system."""
        v, pv = _f64(vals)
        bb, pb = _f64(np.asarray(b).reshape(-1))
        xx = None if x0 is None else _f64(np.asarray(x0).reshape(-1))
        x = np.zeros(3 * self.N)
        r = _CgResult()
        _check(lib().gf_sim_solve_system(self._h, pv, pb, None if xx is None else xx[1], C.c_double(tol),
                                         C.c_int32(max_iters), _p(x, F64P), C.byref(r)))
        return x, dict(iterations=r.iterations, converged=bool(r.converged),
                       negative_curvature=bool(r.negative_curvature), relative_residual=r.relative_residual)

    # runtime utilities
    def set_profiling(self, level):
        """0 / False off, 1 / True events around every kernel, 2 events around the PCG solve only."""
        _check(lib().gf_sim_set_profiling(self._h, C.c_int32(int(level))))

    def kernel_times(self):
        arr = (KernelTime * 64)()
        n = C.c_int32()
        _check(lib().gf_sim_kernel_times(self._h, arr, C.c_int32(64), C.byref(n)))
        return {arr[i].name.decode(): dict(launches=arr[i].launches, total_ms=arr[i].total_ms, bytes=arr[i].bytes)
                for i in range(n.value)}

    def reset_kernel_times(self):
        _check(lib().gf_sim_reset_kernel_times(self._h))

    def synchronize(self):
        _check(lib().gf_sim_synchronize(self._h))

    def info(self) -> dict:
        """gf_sim_info: storage sizes of the device formats (roofline byte models) and the setup wall times."""
        i = _SimInfo()
        _check(lib().gf_sim_info_get(self._h, C.byref(i)))
        out = {k: getattr(i, k) for k, _ in _SimInfo._fields_
               if k not in ("setup_s", "_pad0", "_pad1", "oc_slot_blocks", "oc_offsets")}
        out["oc_slot_blocks"] = list(i.oc_slot_blocks)
        out["oc_offsets"] = list(i.oc_offsets)
        out["pcg_solver_name"] = PCG_SOLVERS[i.pcg_solver]
        out["setup_s"] = dict(pattern_and_layouts=i.setup_s[0], nonlocal_table=i.setup_s[1],
                              device_layout_and_upload=i.setup_s[2], total=i.setup_s[3])
        return out

    def timer_record(self, slot: int):
        _check(lib().gf_sim_timer_record(self._h, C.c_int32(slot)))

    def timer_elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_double()
        _check(lib().gf_sim_timer_elapsed(self._h, C.c_int32(a), C.c_int32(b), C.byref(ms)))
        return ms.value


class VizMesh:
    """VizMesh (viz.hpp:17-82): render-only companion mesh that splits at broken edges (host code, SURVEY
    §8(f)-4). It consumes the ascending newly-broken lists of Simulation.damage_pass / dynamic_step and the
    state read back from the GPU; neither the mesh nor the simulation state is touched."""
    EDGE, FACE, TET = 0, 1, 2

    def __init__(self, mesh: TetMesh, _borrowed=None, _owner=None):
        if _borrowed is not None:  # Simulation.viz(): the simulation's own companion
            self._h, self._owner, self._own = _borrowed, _owner, False
            return
        h = C.c_void_p()
        _check(lib().gf_viz_create(mesh._h, C.byref(h)))
        self._h, self._mesh, self._own = h, mesh, True

    def __del__(self):
        if getattr(self, "_own", False) and getattr(self, "_h", None) and _lib is not None:
            _lib.gf_viz_destroy(self._h)
            self._h = None

    @staticmethod
    def _state(state):
        u = np.ascontiguousarray(state.displacements, dtype=np.float64)
        z = np.ascontiguousarray(state.edge_damage, dtype=np.uint8)
        return u, z

    def apply_splits(self, newly_broken_edges, state):
        """VizMesh::apply_splits (viz.cpp:183-195)."""
        ids = np.ascontiguousarray(newly_broken_edges, dtype=np.int32)
        _, z = self._state(state)
        _check(lib().gf_viz_apply_splits(self._h, ids.ctypes.data, C.c_int64(len(ids)), z.ctypes.data))

    def children(self):
        """VizMesh::children (viz.hpp:62): list of dicts kind / entity / rep / rest_pos / parents_at_creation."""
        out = []
        for c in range(lib().gf_viz_child_count(self._h)):
            k, e, r, n = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
            rest = np.zeros(3)
            par = np.zeros(4, np.int32)
            _check(lib().gf_viz_child(self._h, C.c_int64(c), C.byref(k), C.byref(e), C.byref(r), rest.ctypes.data,
                                      par.ctypes.data, C.byref(n)))
            out.append(dict(kind=k.value, entity=e.value, rep=r.value, rest_pos=rest,
                            parents_at_creation=par[:n.value].tolist()))
        return out

    def child_position(self, child: int, state) -> np.ndarray:
        """VizMesh::child_position (viz.cpp:197-203)."""
        u, z = self._state(state)
        out = np.zeros(3)
        _check(lib().gf_viz_child_position(self._h, C.c_int64(child), u.ctypes.data, z.ctypes.data, out.ctypes.data))
        return out

    def build_surface(self, state):
        """VizMesh::build_surface (viz.cpp:222-317) -> (vertices (V, 3), triangles (F, 3) 0-based,
        original_vertex_count)."""
        u, z = self._state(state)
        nv, nt, no = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().gf_viz_build_surface(self._h, _p(u, F64P), _p(z, U8P), C.byref(nv), C.byref(nt), C.byref(no)))
        v = np.zeros((nv.value, 3))
        t = np.zeros((nt.value, 3), np.int32)
        _check(lib().gf_viz_surface(self._h, _p(v, F64P), _p(t, I32P)))
        return v, t, no.value

    def export_frame(self, path: str, state):
        """VizMesh::export_frame (viz.cpp:319-331): Wavefront OBJ."""
        u, z = self._state(state)
        _check(lib().gf_viz_export_frame(self._h, os.fsencode(path), _p(u, F64P), _p(z, U8P)))

    def fragment_volumes(self, tet: int, state) -> np.ndarray:
        """VizMesh::fragment_volumes (viz.cpp:333-412)."""
        u, z = self._state(state)
        out = np.zeros(4)
        _check(lib().gf_viz_fragment_volumes(self._h, C.c_int32(tet), u.ctypes.data, z.ctypes.data, out.ctypes.data))
        return out


def cg_solve_csr(row_ptr, cols, vals, b, x0, tol, max_iters):
    """cg_solve (sparse.cpp:129-188) on the GPU for a scalar CSR; returns (x, result dict)."""
    rp, prp = _i32(row_ptr)
    cl, pcl = _i32(cols)
    v, pv = _f64(vals)
    b, pb = _f64(b)
    x = np.array(x0, dtype=np.float64, copy=True)
    r = _CgResult()
    _check(lib().gf_cg_solve_csr(C.c_int32(len(rp) - 1), prp, pcl, pv, pb, _p(x, F64P), C.c_double(tol),
                                 C.c_int32(max_iters), C.byref(r)))
    return x, dict(iterations=r.iterations, converged=bool(r.converged),
                   negative_curvature=bool(r.negative_curvature), relative_residual=r.relative_residual)


def set_device(device: int):
    _check(lib().gf_set_device(C.c_int32(device)))


def host_alloc(nbytes: int) -> int:
    """Pinned host memory (cudaMallocHost) as a raw pointer; free with host_free."""
    p = lib().gf_host_alloc(C.c_size_t(nbytes))
    if not p:
        raise CudaError("gf_host_alloc failed")
    return p


def host_free(p: int):
    lib().gf_host_free(C.c_void_p(p))


def measure_bandwidth(kind: str, nbytes: int, reps: int = 20) -> float:
    """GB/s of the current device: kind "l2" = reads of an L2-resident buffer, "hbm" = copy (read + write)."""
    out = C.c_double()
    _check(lib().gf_measure_bandwidth(C.c_int32({"l2": 0, "hbm": 1}[kind]), C.c_int64(int(nbytes)),
                                      C.c_int32(reps), C.byref(out)))
    return out.value


def device_info():
    sm, ma, mi = C.c_int32(), C.c_int32(), C.c_int32()
    name = C.create_string_buffer(128)
    _check(lib().gf_device_info(C.byref(sm), C.byref(ma), C.byref(mi), name, C.c_int32(128)))
    return dict(sm_count=sm.value, cc=(ma.value, mi.value), name=name.value.decode())

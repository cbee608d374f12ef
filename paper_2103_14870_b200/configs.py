"""The BASELINE.json workloads as plain data (shared by bench.py, the tests and smoke()).

Every config uses the reference's own box generator (make_box_mesh, primitives.cpp:71-79) with 1 cm cells;
the config features the reference does not have are mapped identically for the GPU path and the oracle
(DESIGN.md §2 "Config mappings"):
  * seeded interior-node jitter (cell units, splitmix64; applied before rest quantities);
  * energy-density-ratio thresholds -> sigma_thres = E * sqrt(2 * ratio) (uniaxial equivalence);
  * "ductile, yield ratio 0.7" -> the reference's brittle criterion at 0.7 x the c1 base ratio 1e-3
    (no plastic model exists in the reference);
  * "non-local over 2 edge hops" -> the reference's metric radius r_d = 2 h (fracture.cpp:32-54);
  * c1's 500 N point load -> a constant nodal external force (the f_ext hook);
  * c4's initial velocity -> state().velocities, ground -> halfspace Collider (collision.hpp:20-34).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

H = 0.01  # cell size (m)


@dataclass
class BcSpec:
    select: Tuple  # ("plane", axis, value)
    velocity: Tuple[float, float, float] = (0.0, 0.0, 0.0)  # translate schedule u(t) = v t


@dataclass
class Scenario:
    name: str
    cells: Tuple[int, int, int]
    jitter: float = 0.0
    seed: int = 0
    youngs: float = 1e6
    poisson: float = 0.3
    density: float = 1000.0
    sigma_thres: float = 1e5
    r_d: float = 0.0
    model: int = 0  # stable neo-hookean
    dt: float = 1e-3
    steps: int = 100
    cg_tol: float = 1e-8
    cg_max_iters: int = 4000
    gravity: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    bcs: List[BcSpec] = field(default_factory=list)
    colliders: List[dict] = field(default_factory=list)
    initial_velocity: Optional[Tuple[float, float, float]] = None
    point_load: Optional[Tuple[Tuple, Tuple[float, float, float]]] = None  # (selector, total force)
    origin: Tuple[float, float, float] = (0.0, 0.0, 0.0)

    @property
    def size(self):
        return tuple(c * H for c in self.cells)

    @property
    def num_tets(self):
        return 6 * self.cells[0] * self.cells[1] * self.cells[2]


def select_nodes(X: np.ndarray, sel: Tuple, size) -> np.ndarray:
    tol = 1e-9 * max(size)
    kind = sel[0]
    if kind == "plane":
        _, axis, value = sel
        return np.nonzero(np.abs(X[:, axis] - value) <= tol)[0].astype(np.int32)
    if kind == "line":  # intersection of two planes
        _, a0, v0, a1, v1 = sel
        return np.nonzero((np.abs(X[:, a0] - v0) <= tol) & (np.abs(X[:, a1] - v1) <= tol))[0].astype(np.int32)
    raise ValueError(sel)


def threshold_from_ratio(E: float, ratio: float) -> float:
    return E * math.sqrt(2.0 * ratio)


def _c1():
    L = 32 * H
    return Scenario(
        name="c1_bending_bar_8x8x32", cells=(8, 8, 32), youngs=1e7, poisson=0.3, density=1000.0,
        sigma_thres=threshold_from_ratio(1e7, 1e-3), dt=1e-3, steps=200, cg_tol=1e-8,
        bcs=[BcSpec(("plane", 2, 0.0)), BcSpec(("plane", 2, L))],
        point_load=(("line", 1, 8 * H, 2, 16 * H), (0.0, -500.0, 0.0)))


def _c2():
    L = 32 * H
    return Scenario(
        name="c2_tension_cube_32", cells=(32, 32, 32), jitter=0.2, seed=1, youngs=5e6, poisson=0.4, density=1100.0,
        sigma_thres=0.7 * threshold_from_ratio(5e6, 1e-3), dt=5e-4, steps=300,
        bcs=[BcSpec(("plane", 2, 0.0)), BcSpec(("plane", 2, L), (0.0, 0.0, 0.5))])


def _c3():
    Lx = 48 * H
    return Scenario(
        name="c3_tearing_slab_48x48x45", cells=(48, 48, 45), jitter=0.15, seed=2, youngs=2e5, poisson=0.35,
        density=300.0, sigma_thres=0.7 * threshold_from_ratio(2e5, 1e-3), r_d=2 * H, dt=1e-3, steps=200,
        cg_tol=1e-8, bcs=[BcSpec(("plane", 0, 0.0), (-0.3, 0.0, 0.0)), BcSpec(("plane", 0, Lx), (0.3, 0.0, 0.0))])


def _c4():
    return Scenario(
        name="c4_impact_block_96", cells=(96, 96, 96), jitter=0.1, seed=3, youngs=7e10, poisson=0.22,
        density=2500.0, sigma_thres=threshold_from_ratio(7e10, 5e-4), dt=1e-5, steps=100,
        initial_velocity=(0.0, 0.0, -5.0),
        colliders=[dict(kind="halfspace", point=(0.0, 0.0, 0.0), normal=(0.0, 0.0, 1.0), stiffness=1e9,
                        restitution=0.0, friction=0.0)])


CONFIGS = {"c1": _c1, "c2": _c2, "c3": _c3, "c4": _c4}


def get(name: str, **overrides) -> Scenario:
    s = CONFIGS[name]()
    for k, v in overrides.items():
        setattr(s, k, v)
    return s


def scaled(name: str, cells, **overrides) -> Scenario:
    """Same physics/BC layout on a smaller grid (for parity tests); planes follow the new extents."""
    s = CONFIGS[name]()
    old = s.cells
    s.cells = tuple(cells)
    new_bcs = []
    for b in s.bcs:
        kind, axis, value = b.select
        value = value / (old[axis] * H) * (cells[axis] * H) if value else 0.0
        new_bcs.append(BcSpec((kind, axis, value), b.velocity))
    s.bcs = new_bcs
    if s.point_load is not None:
        (_, a0, v0, a1, v1), f = s.point_load
        s.point_load = (("line", a0, cells[a0] * H, a1, round(cells[a1] / 2) * H), f)
    for k, v in overrides.items():
        setattr(s, k, v)
    return s


def bc_dicts(s: Scenario, X: np.ndarray):
    """BCs as plain dicts {nodes, times, values} (oracle/product neutral)."""
    out = []
    for b in s.bcs:
        nodes = select_nodes(X, b.select, s.size)
        out.append(dict(nodes=nodes, times=[0.0, 1.0], values=[[0.0, 0.0, 0.0], list(b.velocity)]))
    return out


def point_load_vector(s: Scenario, X: np.ndarray) -> Optional[np.ndarray]:
    if s.point_load is None:
        return None
    sel, total = s.point_load
    nodes = select_nodes(X, sel, s.size)
    f = np.zeros((len(X), 3))
    f[nodes] = np.asarray(total) / len(nodes)
    return f.reshape(-1)


def build_gpu(s: Scenario):
    """Construct the product Simulation for a scenario (mesh, material, BCs, colliders, loads, v0)."""
    import paper_2103_14870_b200 as g
    mesh = g.make_box_mesh(s.size, s.cells, s.origin, s.jitter, s.seed)
    X = mesh.rest_positions
    mat = g.MaterialParams.from_youngs(s.youngs, s.poisson, s.density, s.sigma_thres, s.r_d, s.model)
    cfg = g.SolverConfig(dt=s.dt, cg_tol=s.cg_tol, cg_max_iters=s.cg_max_iters, gravity=s.gravity)
    bcs = [g.BoundaryCondition(nodes=d["nodes"], translation=g.Schedule3(d["times"], d["values"]))
           for d in bc_dicts(s, X)]
    cols = [g.Collider(kind=c["kind"], point=c["point"], normal=c["normal"], stiffness=c["stiffness"],
                       restitution=c["restitution"], friction=c["friction"]) for c in s.colliders]
    sim = g.Simulation(mesh, mat, cfg, bcs, cols)
    f = point_load_vector(s, X)
    if f is not None:
        sim.set_external_forces(f)
    if s.initial_velocity is not None:
        sim.set_state(velocities=np.tile(np.asarray(s.initial_velocity, np.float64), (mesh.num_nodes(), 1)))
    return sim, mesh

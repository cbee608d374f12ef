"""CPU-side checks of the product library (no GPU needed): the C ABI loads and exports every symbol the
header declares, the host setup (mesh, rest quantities, pattern, non-local table) is bit-identical to the
oracle's, errors map to the reference's exception types, and there is no CPU fallback."""
import os
import re

import numpy as np
import pytest

import paper_2103_14870_b200 as g
from paper_2103_14870_b200 import configs as cf
from oracle import oracle as o
from tests.conftest import ROOT, gpu_available


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64) if a.dtype == np.float64 else a


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "grafem_b200.h")).read()
    names = sorted(set(re.findall(r"\b(gf_[a-z0-9_]+)\s*\(", hdr)))
    assert len(names) > 40
    L = g.lib()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {g.library_path()} 2>&1").read()
    assert "sm_100a" in out, out
    assert not re.search(r"sm_(80|86|89|90)\b", out)


MESHES = [
    dict(size=(0.08, 0.08, 0.32), cells=(8, 8, 32), jitter=0.0, seed=0),
    dict(size=(0.05, 0.06, 0.07), cells=(5, 6, 7), jitter=0.2, seed=1),
    dict(size=(0.1, 0.1, 0.09), cells=(10, 10, 9), jitter=0.15, seed=2),
    dict(size=(1.0, 2.0, 3.0), cells=(3, 4, 5), jitter=0.1, seed=3, origin=(-0.5, 0.25, 1.0)),
]


@pytest.mark.parametrize("spec", MESHES)
def test_mesh_setup_bit_identical_to_oracle(spec):
    origin = spec.get("origin", (0.0, 0.0, 0.0))
    gm = g.make_box_mesh(spec["size"], spec["cells"], origin, spec["jitter"], spec["seed"])
    om = o.Mesh.make_box(spec["size"], spec["cells"], origin, spec["jitter"], spec["seed"])
    a = om.arrays()
    assert (gm.num_nodes(), gm.num_tets(), gm.num_edges()) == (om.num_nodes, om.num_tets, om.num_edges)
    for gk, ok in [("rest_positions", "rest"), ("tets", "tets"), ("edges", "edges"), ("tet_edges", "tet_edges"),
                   ("rest_volumes", "vol"), ("rest_shape_inverse", "binv"), ("rest_centroids", "centroid"),
                   ("rest_edge_lengths", "rest_len")]:
        assert np.array_equal(bits(getattr(gm, gk)), bits(a[ok])), gk
    grp, gcols, gh = gm.pattern()
    orp, ocols, oh = om.pattern()
    assert np.array_equal(grp, orp) and np.array_equal(gcols, ocols) and gh == oh
    assert gm.mean_face_area() == om.mean_face_area()


@pytest.mark.parametrize("r_d_cells", [0.0, 0.9, 1.5, 2.0])
def test_nonlocal_table_bit_identical(r_d_cells):
    spec = MESHES[2]
    gm = g.make_box_mesh(spec["size"], spec["cells"], (0, 0, 0), spec["jitter"], spec["seed"])
    om = o.Mesh.make_box(spec["size"], spec["cells"], (0, 0, 0), spec["jitter"], spec["seed"])
    r_d = r_d_cells * 0.01
    gp, gi, gw = gm.nonlocal_table(r_d)
    op, oi, ow = om.nonlocal_table(r_d, brute=r_d_cells in (0.9, 2.0))
    assert np.array_equal(gp, op) and np.array_equal(gi, oi) and np.array_equal(bits(gw), bits(ow))


def test_random_mesh_and_tetgen_parity():
    rng = np.random.default_rng(4)
    X = rng.uniform(0, 1, (5, 3))
    X[4] = X[:4].mean(0) + [0.0, 0.0, 0.5]
    tets = [[0, 1, 2, 3], [0, 1, 2, 4]]
    # orient both tets positively as make_mesh requires
    for t in tets:
        d = np.linalg.det(np.stack([X[t[1]] - X[t[0]], X[t[2]] - X[t[0]], X[t[3]] - X[t[0]]], 1))
        if d < 0:
            t[2], t[3] = t[3], t[2]
    gm, om = g.make_mesh(X, tets), o.Mesh.create(X, tets)
    assert np.array_equal(bits(gm.rest_shape_inverse), bits(om.arrays()["binv"]))
    node = "4 3 0 0\n1 0 0 0\n2 1 0 0\n3 0 1 0\n4 0 0 1\n"
    ele = "1 4 0\n1 1 2 3 4\n"
    gt, ot = g.load_tetgen(node, ele), o.Mesh.load_tetgen(node, ele)
    assert np.array_equal(bits(gt.rest_shape_inverse), bits(ot.arrays()["binv"]))


def test_error_types():
    with pytest.raises(g.GeometryError):
        g.make_mesh([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], [[0, 2, 1, 3]])
    with pytest.raises(g.GeometryError):
        g.make_mesh([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], [[0, 1, 1, 3]])
    with pytest.raises(g.FormatError):
        g.load_tetgen("4 2\n", "1 4\n1 1 2 3 4\n")
    with pytest.raises(g.FormatError):
        g.MaterialParams.from_youngs(1e6, 0.5, 1000, 1e5)
    p = g.MaterialParams.from_youngs(2.1e9, 0.3, 7800.0, 1e6)
    q = o.material_from_youngs(2.1e9, 0.3, 7800.0, 1e6)
    assert (p.mu, p.lambda_) == (q.mu, q.lambda_)


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU path")
def test_no_cpu_fallback_without_gpu():
    s = cf.get("c1")
    with pytest.raises(g.CudaError):
        cf.build_gpu(s)


def test_config_selections():
    s = cf.get("c1")
    m = g.make_box_mesh(s.size, s.cells)
    X = m.rest_positions
    f = cf.point_load_vector(s, X).reshape(-1, 3)
    assert (np.abs(f[:, 1]) > 0).sum() == 9 and f[:, 1].sum() == pytest.approx(-500.0)
    bcs = cf.bc_dicts(s, X)
    assert [len(b["nodes"]) for b in bcs] == [81, 81]
    s3 = cf.get("c3")
    assert s3.num_tets == 622080 and s3.r_d == pytest.approx(0.02)
    assert cf.get("c4").num_tets == 5308416


@pytest.mark.parametrize("src", ["facade_smoke.cpp", "facade_reference_style.cpp"])
def test_cpp_facade_compiles_and_links(tmp_path, src):
    """include/grafem_b200.hpp (reference-shaped C++ API: MaterialParams, SolverConfig, BoundaryCondition, Schedule3,
    Collider, StepStats, Simulation with material()/config()) builds against the library -- facade_reference_style.cpp
    is a reference call site with only the include and namespace changed; on a CPU-only host the Simulation
    constructor must raise CudaError (exit 10), on a GPU host the steps must run (exit 0)."""
    import subprocess
    from paper_2103_14870_b200 import build as b
    exe = tmp_path / "facade"
    libdir = os.path.dirname(g.library_path())
    subprocess.run([b._host_cxx(), "-std=c++17", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", src), "-L", libdir, "-lgrafem_b200",
                    f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == (0 if gpu_available() else 10), r.stdout + r.stderr

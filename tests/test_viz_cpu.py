"""Render-side consumer (VizMesh, host code): the known answers of the reference's
proj/tests/test_viz.cpp restated, plus OBJ format / determinism / error checks. CPU only."""
from types import SimpleNamespace

import numpy as np
import pytest

import paper_2103_14870_b200 as g


def unit_tet():
    return g.make_mesh([(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)], [(0, 1, 2, 3)])


def rest_state(mesh):
    return SimpleNamespace(displacements=np.zeros((mesh.num_nodes(), 3)),
                           edge_damage=np.zeros(mesh.num_edges(), np.uint8))


def edge_id(mesh, a, b):
    key = (min(a, b), max(a, b))
    for e, ed in enumerate(mesh.edges):
        if tuple(ed) == key:
            return e
    raise AssertionError(key)


def boundary_faces(mesh):
    count = {}
    for t in mesh.tets:
        for f in ((t[1], t[2], t[3]), (t[0], t[2], t[3]), (t[0], t[1], t[3]), (t[0], t[1], t[2])):
            k = tuple(sorted(int(x) for x in f))
            count[k] = count.get(k, 0) + 1
    return [k for k, c in count.items() if c == 1]


def obj_counts(path):
    v = f = 0
    with open(path) as fh:
        for line in fh:
            v += line.startswith("v ")
            f += line.startswith("f ")
    return v, f


def test_pre_fracture_surface_equals_the_computational_boundary():  # test_viz.cpp:39-58
    mesh = g.make_box_mesh((1, 1, 1), (2, 2, 2))
    viz = g.VizMesh(mesh)
    verts, tris, n_orig = viz.build_surface(rest_state(mesh))
    bf = boundary_faces(mesh)
    assert len(tris) == len(bf)
    bnodes = sorted({n for f in bf for n in f})
    assert len(verts) == len(bnodes) == n_orig
    assert np.array_equal(verts, mesh.rest_positions[bnodes])  # ascending node order, bit-equal
    # every triangle is a boundary face, oriented outward (away from the mesh centre for this convex box)
    centre = mesh.rest_positions.mean(axis=0)
    for t in tris:
        a, b, c = verts[t]
        assert tuple(sorted(bnodes[i] for i in t)) in set(bf)
        assert np.dot(np.cross(b - a, c - a), (a + b + c) / 3 - centre) > 0


def test_no_broken_edges_leaves_the_render_mesh_unchanged():  # test_viz.cpp:60-69
    mesh = unit_tet()
    viz = g.VizMesh(mesh)
    st = rest_state(mesh)
    viz.apply_splits([], st)
    assert viz.children() == []
    verts, tris, _ = viz.build_surface(st)
    assert len(verts) == 4 and len(tris) == 4


def test_breaking_one_edge_creates_two_midpoint_children_bound_to_its_endpoints():  # test_viz.cpp:71-91
    mesh = unit_tet()
    st = rest_state(mesh)
    viz = g.VizMesh(mesh)
    e01 = edge_id(mesh, 0, 1)
    st.edge_damage[e01] = 1
    viz.apply_splits([e01], st)
    mid = 0.5 * (mesh.rest_positions[0] + mesh.rest_positions[1])
    at_mid = [c for c in viz.children() if np.linalg.norm(c["rest_pos"] - mid) < 1e-14]
    assert len(at_mid) == 2
    assert sorted(c["parents_at_creation"][0] for c in at_mid) == [0, 1]
    assert all(len(c["parents_at_creation"]) == 1 for c in at_mid)


def test_partial_face_split_lone_corner_separates():  # test_viz.cpp:93-118
    mesh = unit_tet()
    st = rest_state(mesh)
    viz = g.VizMesh(mesh)
    broken = [edge_id(mesh, 0, 1), edge_id(mesh, 0, 2), edge_id(mesh, 0, 3)]
    st.edge_damage[broken] = 1
    viz.apply_splits(broken, st)
    st.displacements[1] = (0.1, 0, 0)
    st.displacements[2] = (-0.1, 0, 0)
    st.displacements[0] = (0, 0, 0.25)
    seen = set()
    for c, ch in enumerate(viz.children()):
        pos = viz.child_position(c, st)
        if ch["parents_at_creation"] == [1, 2]:
            assert np.linalg.norm(pos - ch["rest_pos"]) < 1e-15  # the mean of +/- cancels
            seen.add("pair")
        if ch["parents_at_creation"] == [0]:
            assert np.linalg.norm(pos - (ch["rest_pos"] + (0, 0, 0.25))) < 1e-15
            seen.add("lone")
    assert seen == {"pair", "lone"}


def test_advection_rigid_translation_and_single_parent_offset():  # test_viz.cpp:120-148
    mesh = unit_tet()
    st = rest_state(mesh)
    viz = g.VizMesh(mesh)
    st.edge_damage[:] = 1
    viz.apply_splits(list(range(mesh.num_edges())), st)
    ch = viz.children()
    assert ch
    shift = np.array([0.3, -0.2, 0.9])
    st.displacements[:] = shift
    for c, x in enumerate(ch):
        assert np.linalg.norm(viz.child_position(c, st) - (x["rest_pos"] + shift)) < 1e-15
    st.displacements[2] = (0.5, 0.1, -0.3)
    single = [c for c, x in enumerate(ch) if x["parents_at_creation"] == [2]]
    assert single
    for c in single:
        off = viz.child_position(c, st) - (mesh.rest_positions[2] + st.displacements[2])
        assert np.linalg.norm(off - (ch[c]["rest_pos"] - mesh.rest_positions[2])) < 1e-14


def test_fully_split_tet_fragment_volumes_sum_to_the_tet_volume():  # test_viz.cpp:150-177
    mesh = unit_tet()
    st = rest_state(mesh)
    viz = g.VizMesh(mesh)
    st.edge_damage[:] = 1
    viz.apply_splits(list(range(mesh.num_edges())), st)
    vols = viz.fragment_volumes(0, st)
    assert np.all(vols > 0)
    assert abs(vols.sum() - mesh.rest_volumes[0]) < 1e-9
    st.displacements[0] = (-1, 0, 0)  # fragments fly apart rigidly: volumes unchanged
    st.displacements[1] = (1, 1, 0)
    st.displacements[2] = (0, -2, 1)
    vols2 = viz.fragment_volumes(0, st)
    assert np.allclose(vols2, vols, rtol=1e-9, atol=0)
    assert abs(vols2.sum() - mesh.rest_volumes[0]) < 1e-9


def test_intact_tet_single_fragment_carries_the_whole_volume():
    """With no broken edge every corner's group is the whole tet: the corner pieces still partition it."""
    mesh = g.make_box_mesh((1, 1, 1), (1, 1, 1), jitter=0.0)
    st = rest_state(mesh)
    viz = g.VizMesh(mesh)
    for t in range(mesh.num_tets()):
        assert abs(viz.fragment_volumes(t, st).sum() - mesh.rest_volumes[t]) < 1e-12


def test_splitting_touches_neither_mesh_nor_state():  # test_viz.cpp:179-198
    mesh = g.make_box_mesh((1, 1, 1), (2, 1, 1))
    st = rest_state(mesh)
    viz = g.VizMesh(mesh)
    X0, T0 = mesh.rest_positions.copy(), mesh.tets.copy()
    st.edge_damage[0] = 1
    u0, z0 = st.displacements.copy(), st.edge_damage.copy()
    viz.apply_splits([0], st)
    viz.build_surface(st)
    assert np.array_equal(mesh.rest_positions, X0) and np.array_equal(mesh.tets, T0)
    assert np.array_equal(st.displacements, u0) and np.array_equal(st.edge_damage, z0)


def test_obj_export_counts_determinism_and_fracture_surfaces(tmp_path):  # test_viz.cpp:200-235
    mesh = unit_tet()
    st = rest_state(mesh)
    viz = g.VizMesh(mesh)
    viz.export_frame(str(tmp_path / "intact.obj"), st)
    assert obj_counts(tmp_path / "intact.obj") == (4, 4)
    e01 = edge_id(mesh, 0, 1)
    st.edge_damage[e01] = 1
    viz.apply_splits([e01], st)
    viz.export_frame(str(tmp_path / "split.obj"), st)
    v1, f1 = obj_counts(tmp_path / "split.obj")
    assert v1 > 4 and f1 > 4
    viz.export_frame(str(tmp_path / "split2.obj"), st)
    assert (tmp_path / "split.obj").read_bytes() == (tmp_path / "split2.obj").read_bytes()
    # the record format of export_frame (viz.cpp:323-330): %.17g coordinates, 1-based faces
    verts, tris, _ = viz.build_surface(st)
    lines = (tmp_path / "split.obj").read_text().splitlines()
    assert lines[0] == "v %.17g %.17g %.17g" % tuple(verts[0])
    assert lines[len(verts)] == "f %d %d %d" % tuple(tris[0] + 1)
    assert (v1, f1) == (len(verts), len(tris))
    # one broken edge of a single tet (test_viz.cpp:214-216): 2 midpoint children of that edge, one shared
    # centroid child per split face and one tet child (the other five edges keep both groups connected)
    kinds = [c["kind"] for c in viz.children()]
    assert kinds.count(g.VizMesh.TET) == 1 and kinds.count(g.VizMesh.FACE) == 2
    assert sum(1 for c in viz.children() if c["kind"] == g.VizMesh.EDGE and c["entity"] == e01) == 2


def test_split_requests_are_validated_and_idempotent():
    mesh = unit_tet()
    st = rest_state(mesh)
    viz = g.VizMesh(mesh)
    with pytest.raises(g.GeometryError):
        viz.apply_splits([mesh.num_edges()], st)
    st.edge_damage[:] = 1
    viz.apply_splits([0, 1], st)
    n = len(viz.children())
    viz.apply_splits([0, 1], st)
    assert len(viz.children()) == n
    # build_surface needs the children of every broken edge: a missing split is an error, not a silent hole
    viz2 = g.VizMesh(mesh)
    with pytest.raises(g.GeometryError):
        viz2.build_surface(st)
    with pytest.raises(g.FormatError):
        viz2.export_frame("/nonexistent-dir/x.obj", rest_state(mesh))


def test_closed_fracture_surface_is_watertight():
    """Every edge of the exported triangle soup is shared by exactly two triangles: the exterior pieces and
    the fracture quads of a fully shattered block close up (orientation-consistent: each directed edge once)."""
    mesh = g.make_box_mesh((1, 1, 1), (2, 2, 1))
    st = rest_state(mesh)
    st.edge_damage[:] = 1
    viz = g.VizMesh(mesh)
    viz.apply_splits(list(range(mesh.num_edges())), st)
    _, tris, _ = viz.build_surface(st)
    directed = {}
    for a, b, c in tris:
        for e in ((a, b), (b, c), (c, a)):
            directed[e] = directed.get(e, 0) + 1
    assert all(v == 1 for v in directed.values())
    assert all((b, a) in directed for (a, b) in directed)

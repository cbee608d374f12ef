"""Mesh known answers (test_mesh.cpp) for BOTH the oracle and the product's host mesh setup.

The mesh data model (canonical edges, tet->edge map, rest volumes / shape inverses / centroids / edge lengths)
feeds every kernel on the path, so the product's setup code (csrc host side, no GPU needed) is pinned against
the reference's own unit-test answers here, next to the oracle. Boundary-face extraction (viz) is out of scope.
"""
import itertools
import random

import numpy as np
import pytest

import paper_2103_14870_b200 as g
from oracle import oracle as o

UNIT_NODE = "# unit right tet\n4 3 0 0\n1 0.0 0.0 0.0\n2 1.0 0.0 0.0\n3 0.0 1.0 0.0\n4 0.0 0.0 1.0\n"
UNIT_ELE = "1 4 0\n1 1 2 3 4\n"
TWO_TET = ([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 1]], [[0, 1, 2, 3], [1, 2, 3, 4]])


class _Oracle:
    FormatError, GeometryError = o.FormatError, o.GeometryError

    def __init__(self, m):
        a = m.arrays()
        self.rest, self.tets, self.edges, self.tet_edges = a["rest"], a["tets"], a["edges"], a["tet_edges"]
        self.vol, self.binv, self.centroid, self.edge_len = a["vol"], a["binv"], a["centroid"], a["rest_len"]

    @classmethod
    def create(cls, nodes, tets):
        return cls(o.Mesh.create(nodes, tets))

    @classmethod
    def tetgen(cls, n, e):
        return cls(o.Mesh.load_tetgen(n, e))

    @classmethod
    def box(cls, size, cells):
        return cls(o.Mesh.make_box(size, cells))


class _Product(_Oracle):
    FormatError, GeometryError = g.FormatError, g.GeometryError

    def __init__(self, m):
        self.rest, self.tets, self.edges, self.tet_edges = m.rest_positions, m.tets, m.edges, m.tet_edges
        self.vol, self.binv = m.rest_volumes, m.rest_shape_inverse
        self.centroid, self.edge_len = m.rest_centroids, m.rest_edge_lengths

    @classmethod
    def create(cls, nodes, tets):
        return cls(g.make_mesh(nodes, tets))

    @classmethod
    def tetgen(cls, n, e):
        return cls(g.load_tetgen(n, e))

    @classmethod
    def box(cls, size, cells):
        return cls(g.make_box_mesh(size, cells))


@pytest.fixture(params=["oracle", "product"])
def M(request):
    return _Oracle if request.param == "oracle" else _Product


def edge_tets(m):
    out = [[] for _ in range(len(m.edges))]
    for t, te in enumerate(m.tet_edges):
        for e in te:
            out[e].append(t)
    return out


def edge_index(m, a, b):
    hit = np.nonzero((m.edges[:, 0] == a) & (m.edges[:, 1] == b))[0]
    assert len(hit) == 1
    return int(hit[0])


def test_load_tetgen_unit_tet(M):  # test_mesh.cpp:32-38
    m = M.tetgen(UNIT_NODE, UNIT_ELE)
    assert (len(m.rest), len(m.tets), len(m.edges)) == (4, 1, 6)
    assert m.vol[0] == pytest.approx(1 / 6, rel=1e-14)


def test_load_tetgen_zero_based(M):  # test_mesh.cpp:40-46
    m = M.tetgen("4 3 0 0\n0 0.0 0.0 0.0\n1 1.0 0.0 0.0\n2 0.0 1.0 0.0\n3 0.0 0.0 1.0\n", "1 4 0\n0 0 1 2 3\n")
    assert len(m.tets) == 1


def test_two_tets_share_three_edges(M):  # test_mesh.cpp:48-56
    m = M.create(*TWO_TET)
    assert len(m.edges) == 9
    assert sum(len(ts) == 2 for ts in edge_tets(m)) == 3


def test_out_of_range_node_is_format_error_with_line(M):  # test_mesh.cpp:58-66
    with pytest.raises(M.FormatError, match="line 2"):
        M.tetgen(UNIT_NODE, "1 4 0\n1 1 2 3 9\n")


def test_inverted_element_is_geometry_error_naming_tet(M):  # test_mesh.cpp:68-76
    with pytest.raises(M.GeometryError, match="tet 0"):
        M.tetgen(UNIT_NODE, "1 4 0\n1 1 3 2 4\n")


def test_single_tet_edges_incident_to_tet0(M):  # test_mesh.cpp:78-84
    m = M.tetgen(UNIT_NODE, UNIT_ELE)
    assert edge_tets(m) == [[0]] * 6


def test_three_tet_fan_edge(M):  # test_mesh.cpp:86-96
    m = M.create([[0, 0, 0], [0, 0, 1], [1, 0, 0], [0.3, 1, 0.5], [-1, 0.2, 0.5], [0.2, -1, 0.5]],
                 [[0, 1, 2, 3], [0, 1, 3, 4], [0, 1, 4, 5]])
    assert edge_tets(m)[edge_index(m, 0, 1)] == [0, 1, 2]


def test_empty_tet_list_rejected(M):  # test_mesh.cpp:98-102
    with pytest.raises(M.GeometryError):
        M.create([[0, 0, 0]], np.zeros((0, 4), np.int32))


def test_repeated_node_rejected(M):  # test_mesh.cpp:104-108
    with pytest.raises(M.GeometryError):
        M.create([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], [[0, 1, 2, 2]])


def test_rest_quantities_unit_tet(M):  # test_mesh.cpp:110-122
    m = M.tetgen(UNIT_NODE, UNIT_ELE)
    assert m.vol[0] == pytest.approx(1 / 6, rel=1e-14)
    assert np.linalg.norm(m.centroid[0] - 0.25) < 1e-15
    assert m.edge_len[edge_index(m, 0, 1)] == pytest.approx(1.0)
    dm = (m.rest[1:4] - m.rest[0]).T
    assert np.linalg.norm(dm @ m.binv[0] - np.eye(3)) < 1e-14


def test_similarity_scaling(M):  # test_mesh.cpp:124-132
    nodes = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    base, scaled = M.create(nodes, [[0, 1, 2, 3]]), M.create(2 * nodes, [[0, 1, 2, 3]])
    assert scaled.vol[0] == pytest.approx(8 * base.vol[0], rel=1e-13)
    assert np.allclose(scaled.edge_len, 2 * base.edge_len, rtol=1e-12)


def test_edge_set_equals_bruteforce_pairs(M):  # test_mesh.cpp:134-143
    m = M.box((1, 1, 1), (2, 2, 1))
    brute = sorted({(min(t[i], t[j]), max(t[i], t[j])) for t in m.tets.tolist()
                    for i, j in itertools.combinations(range(4), 2)})
    assert [tuple(e) for e in m.edges.tolist()] == brute


def test_rest_volume_sum(M):  # test_mesh.cpp:145-156
    m = M.box((0.3, 0.2, 0.1), (3, 2, 2))
    X = m.rest
    signed = sum(np.dot(X[t[1]] - X[t[0]], np.cross(X[t[2]] - X[t[0]], X[t[3]] - X[t[0]])) / 6 for t in m.tets)
    assert m.vol.sum() == pytest.approx(signed, rel=1e-12)
    assert m.vol.sum() == pytest.approx(0.3 * 0.2 * 0.1, rel=1e-12)


def test_edge_graph_invariant_under_tet_permutation(M):  # test_mesh.cpp:158-165
    m = M.box((1, 1, 1), (2, 2, 2))
    tets = m.tets.tolist()
    random.Random(99).shuffle(tets)
    assert np.array_equal(M.create(m.rest, tets).edges, m.edges)


def test_tet_edges_and_edge_tets_consistent(M):  # test_mesh.cpp:167-184
    m = M.create(*TWO_TET)
    et = edge_tets(m)
    for t, te in enumerate(m.tet_edges.tolist()):
        assert len(set(te)) == 6 and all(t in et[e] for e in te)
    for e, ts in enumerate(et):
        assert all(e in m.tet_edges[t] for t in ts)


def test_generated_box_is_valid(M):  # test_mesh.cpp:200+ (make_box_mesh)
    m = M.box((0.2, 0.1, 0.1), (4, 2, 2))
    assert len(m.tets) == 6 * 16 and len(m.rest) == 5 * 3 * 3
    assert np.all(m.vol > 0) and m.vol.sum() == pytest.approx(0.002, rel=1e-12)

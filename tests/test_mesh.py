"""Host mesh generators (csrc/meshgen.cpp) against the reference builder and
the reference's own known-answer tests."""
import numpy as np
import pytest

from paper_2106_07154_b200.mesh import Mesh


@pytest.mark.parametrize("level", [0, 1, 2, 3, 4, 5])
def test_icosahedral_tables_bitwise_equal_reference(ref_lib, level):
    mine = Mesh.icosahedral(level, 6371220.0)
    ref = ref_lib.RefMesh.icosahedral(level, 6371220.0).as_mesh()
    for name, arr in mine.tables.items():
        assert np.array_equal(arr.view(np.uint8), ref.tables[name].view(np.uint8)), name
    for a, b in [(mine.cell_xyz, ref.cell_xyz), (mine.vertex_xyz, ref.vertex_xyz),
                 (mine.edge_xyz, ref.edge_xyz), (mine.kite_area, ref.kite_area)]:
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_level0_weights_are_tenths():
    # test_mesh.cpp:121-128 / SPEC.md:113-114: all-pentagon mesh, |w| in {0.1, 0.3}
    m = Mesh.icosahedral(0, 1.0)
    w = np.abs(m.edge_weight)
    assert np.all((np.abs(w - 0.1) < 1e-12) | (np.abs(w - 0.3) < 1e-12))


def test_icosahedral_counts():
    for level in range(4):
        m = Mesh.icosahedral(level, 1.0)
        nC = 10 * 4 ** level + 2
        assert (m.n_cells, m.n_edges, m.n_vertices) == (nC, 3 * (nC - 2), 2 * (nC - 2))
        assert np.sum(m.ring_size() == 5) == 12


def _reverse_walk_weights(m, e):
    """oracles.hpp:139-160: the stencil rebuilt by a clockwise walk."""
    out = []
    co, ce, cv = m.cell_offset, m.cell_edges, m.cell_vertices
    ec, ecs, ev, evs = m.edge_cells, m.edge_cell_sign, m.edge_vertices, m.edge_vertex_sign
    ka, A = m.kite_area, m.cell_area

    def csign(edge, cell):
        return float(ecs[edge][0] if ec[edge][0] == cell else ecs[edge][1])

    def vsign(edge, v):
        return float(evs[edge][0] if ev[edge][0] == v else evs[edge][1])

    for side in range(2):
        i = ec[e][side]
        off, mm = co[i], co[i + 1] - co[i]
        ring = list(ce[off:off + mm])
        p = ring.index(e)
        anchor = vsign(e, cv[off + (p + mm - 1) % mm])
        frac = 0.0
        cw = []
        for k in range(1, mm):
            frac += ka[off + (p + mm - k) % mm] / A[i]
            ep = ring[(p + mm - k) % mm]
            cw.append((ep, csign(ep, i) * anchor * (frac - 0.5)))
        out.extend(reversed(cw))
    return out


@pytest.mark.parametrize("make", [lambda: Mesh.planar_hex(12, 10, 10e3),
                                  lambda: Mesh.icosahedral(2, 6371220.0)])
def test_weights_match_reverse_walk_oracle(make):
    m = make()
    for e in range(0, m.n_edges, 7):
        rev = _reverse_walk_weights(m, e)
        off = m.edge_edge_offset[e]
        ids = m.edge_edges[off:off + len(rev)]
        ws = m.edge_weight[off:off + len(rev)]
        assert list(ids) == [r[0] for r in rev]
        assert np.max(np.abs(ws - np.array([r[1] for r in rev]))) < 1e-13


def test_planar_hex_known_answers():
    dc = 10e3
    m = Mesh.planar_hex(16, 12, dc)
    assert (m.n_cells, m.n_edges, m.n_vertices) == (192, 576, 384)
    assert np.all(m.ring_size() == 6)
    np.testing.assert_allclose(m.edge_dual_len, dc, rtol=1e-14)
    np.testing.assert_allclose(m.edge_len, dc / np.sqrt(3), rtol=1e-12)
    np.testing.assert_allclose(m.cell_area, np.sqrt(3) / 2 * dc * dc, rtol=1e-12)
    np.testing.assert_allclose(m.vertex_area, np.sqrt(3) / 4 * dc * dc, rtol=1e-12)
    # kites at a vertex sum to its area (test_mesh.cpp:135-149)
    np.testing.assert_allclose(m.vertex_kite.sum(axis=1), m.vertex_area, rtol=1e-12)
    # regular hexagon: w = +-(k/6 - 1/2) -> |w| in {1/3, 1/6, 0}
    w = np.abs(m.edge_weight)
    near = lambda x: np.abs(w - x) < 1e-12
    assert np.all(near(1 / 3) | near(1 / 6) | near(0.0))
    assert np.all(np.diff(m.edge_edge_offset) == 10)


def test_planar_weight_antisymmetry():
    # test_operators.cpp:107-142: w_{e,e'} l_e'/d_e' ... antisymmetric: w_ee' = -w_e'e
    m = Mesh.planar_hex(10, 8, 3e3)
    W = {}
    for e in range(m.n_edges):
        off, end = m.edge_edge_offset[e], m.edge_edge_offset[e + 1]
        for j in range(off, end):
            W[(e, m.edge_edges[j])] = m.edge_weight[j] * m.edge_len[m.edge_edges[j]]
    worst = max(abs(v + W[(b, a)] * 1.0) for (a, b), v in W.items() if (b, a) in W)
    assert worst < 1e-9


def test_planar_tables_rederived_by_reference(ref_lib):
    """The reference's own rebuild_edge_stencil + assign_orientation_signs
    (mesh_build.cpp:133-183) reproduce the planar builder's tables."""
    m = Mesh.planar_hex(16, 12, 10e3)
    r = ref_lib.RefMesh.from_mesh(m)
    r.rederive()
    back = r.as_mesh()
    for name in ("edge_edge_offset", "edge_edges", "edge_cell_sign", "edge_vertex_sign"):
        assert np.array_equal(m.tables[name], back.tables[name]), name


def test_planar_rejects_bad_shapes():
    with pytest.raises(RuntimeError):
        Mesh.planar_hex(8, 7, 1e3)

"""The CPU restatement oracle (oracle/mswm_oracle.c) is pinned two ways:
bitwise against the committed golden fixtures made from the unmodified
reference (tests/make_golden.py), and bitwise against the reference itself
(oracle/_ref) on fresh inputs when that library is present."""
import numpy as np
import pytest

from helpers import bits_equal, golden_mesh, load_golden
from oracle.oracle import Oracle, orc_lts_coeffs
from paper_2106_07154_b200 import workloads as W
from paper_2106_07154_b200.api import LTS3_MASKS, Scheme, kMaskAll
from make_golden import mesh_digest

FIXTURES = ["planar24", "sphereL3"]


@pytest.mark.parametrize("name", FIXTURES)
def test_restatement_matches_golden(name):
    g = load_golden(name)
    mesh = golden_mesh(name)
    assert mesh_digest(mesh) == str(g["digest"]), "mesh generator drifted from the fixture"
    o = Oracle(mesh, g["b"], g["f"], float(g["gravity"]))
    o.set_regions(g["fine"], 1)
    cl, cs, el = o.labels()
    assert np.array_equal(cl, g["cell_label"])
    assert np.array_equal(cs, g["cell_sub"])
    assert np.array_equal(el, g["edge_label"])
    for gi, ids in enumerate(o.groups()):
        assert np.array_equal(ids, g[f"group{gi}"]), gi
    for mask in LTS3_MASKS + [kMaskAll]:
        dh = np.full(mesh.n_cells, np.nan)
        du = np.full(mesh.n_edges, np.nan)
        o.eval(g["h"], g["u"], mask, dh, du)
        assert bits_equal(dh, g[f"dh_{mask}"]), mask
        assert bits_equal(du, g[f"du_{mask}"]), mask
        for kind in range(4):
            assert np.array_equal(np.sort(o.last_closure(kind)), g[f"closure_{mask}_{kind}"])
    M = int(g["M"])
    dt = float(g["dt"])
    for scheme, n in [(Scheme.LTS3, 3), (Scheme.RK4, 2), (Scheme.SSPRK3, 2)]:
        o2 = Oracle(mesh, g["b"], g["f"], float(g["gravity"]))
        o2.set_regions(g["fine"], 1)
        h, u, _ = o2.step(int(scheme), g["h"], g["u"], 0.0, dt if scheme == Scheme.LTS3 else dt / M,
                          M, n)
        assert bits_equal(h, g[f"h_{scheme.name}"]), scheme
        assert bits_equal(u, g[f"u_{scheme.name}"]), scheme
        c, e, _ = o2.ledger()
        assert np.array_equal(c, g[f"ledger_cell_{scheme.name}"])
        assert np.array_equal(e, g[f"ledger_edge_{scheme.name}"])


def test_lts_coefficient_table():
    # test_integrators.cpp:85-122 pins these closed forms; x~ per stage
    for M in (1, 2, 4, 7):
        for k in range(M):
            for stage in (1, 2, 3):
                c = orc_lts_coeffs(3, stage, k, M)
                assert abs(c.sum() - 1.0) < 1e-15
    assert np.array_equal(orc_lts_coeffs(3, 1, 0, 4), [1.0, 0.0, 0.0])
    c = orc_lts_coeffs(3, 3, 0, 1)  # x = 1/2, x~ = 1/2
    assert np.array_equal(c, [1.0 - 0.5 - 0.5, 0.0, 1.0])


def test_lts_coeffs_match_reference(ref_lib):
    for order in (2, 3):
        for M in (1, 3, 8):
            for k in range(M):
                for stage in range(1, order + 1):
                    assert bits_equal(orc_lts_coeffs(order, stage, k, M),
                                      ref_lib.ref_lts_coeffs(order, stage, k, M))


def _both(wl):
    from oracle.oracle import RefEvaluator, RefMesh, RefRegions
    rm = RefMesh.from_mesh(wl.mesh)
    rr = RefRegions(rm, wl.fine_mask, wl.width)
    ev = RefEvaluator(rm, rr, wl.b, wl.f, wl.gravity)
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, wl.width)
    return rm, rr, ev, o


@pytest.mark.parametrize("make", [lambda: W.config1(n_steps=4), lambda: W.small_sphere(4)])
def test_restatement_matches_reference(ref_lib, make):
    wl = make()
    m = wl.mesh
    rm, rr, ev, o = _both(wl)
    for a, b in zip(rr.groups(), o.groups()):
        assert np.array_equal(a, b)
    for mask in LTS3_MASKS + [kMaskAll, 0x21, 0x401]:
        dh1 = np.full(m.n_cells, 7.0)
        du1 = np.full(m.n_edges, 7.0)
        dh2, du2 = dh1.copy(), du1.copy()
        ev.eval(wl.h, wl.u, mask, dh1, du1)
        o.eval(wl.h, wl.u, mask, dh2, du2)
        assert bits_equal(dh1, dh2) and bits_equal(du1, du2), hex(mask)
    for scheme in (Scheme.LTS3, Scheme.RK4, Scheme.SSPRK3, Scheme.SSPRK2, Scheme.LTS2):
        h1, u1, t1, _ = ev.step(int(scheme), wl.h, wl.u, 0.0, wl.dt, wl.M, 3)
        h2, u2, t2 = o.step(int(scheme), wl.h, wl.u, 0.0, wl.dt, wl.M, 3)
        assert bits_equal(h1, h2) and bits_equal(u1, u2) and t1 == t2, scheme


def test_restatement_region_errors():
    wl = W.config1(n_steps=1)
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    from oracle.oracle import OracleError
    with pytest.raises(OracleError):
        o.set_regions(np.zeros(wl.mesh.n_cells, np.uint8), 1)      # no fine cell
    with pytest.raises(OracleError):
        o.set_regions(np.ones(wl.mesh.n_cells, np.uint8), 1)       # all fine
    with pytest.raises(OracleError):
        o.set_regions(wl.fine_mask, 40)                            # no coarse left


def test_restatement_dry_vertex(ref_lib):
    # test_operators.cpp:222-242 on a level-0 mesh, via both libraries
    from oracle.oracle import OracleError, RefEvaluator, RefMesh
    from paper_2106_07154_b200.mesh import Mesh
    mesh = Mesh.icosahedral(0, 1.0)
    h = np.ones(mesh.n_cells)
    h[4] = -40.0
    u = np.full(mesh.n_edges, 0.1)
    b = np.zeros(mesh.n_cells)
    f = np.zeros(mesh.n_vertices)
    o = Oracle(mesh, b, f, 9.80616)
    with pytest.raises(OracleError) as e1:
        o.eval(h, u, kMaskAll, np.zeros(mesh.n_cells), np.zeros(mesh.n_edges))
    ev = RefEvaluator(RefMesh.from_mesh(mesh), None, b, f, 9.80616)
    with pytest.raises(OracleError) as e2:
        ev.eval(h, u, kMaskAll, np.zeros(mesh.n_cells), np.zeros(mesh.n_edges))
    assert e1.value.vertex == e2.value.vertex
    assert 4 in mesh.vertex_cells[e1.value.vertex]


@pytest.mark.parametrize("make", [lambda: W.config1(n_steps=4), lambda: W.small_sphere(4)])
def test_diagnostics_match_reference(ref_lib, make):
    """total_mass / total_energy (harness.cpp:99-123) and courant_numbers
    (integrators.cpp:632-659), with and without a region map."""
    wl = make()
    rm, rr, ev, o = _both(wl)
    h, u, _ = o.step(int(Scheme.LTS3), wl.h, wl.u, 0.0, wl.dt, wl.M, 2)
    assert o.total_mass(h) == rm.total_mass(h)
    assert o.total_energy(h, u) == rm.total_energy(h, u, wl.b, wl.gravity)
    for M in (1, 4):
        assert o.courant(u, wl.dt, M) == rm.courant(rr, u, wl.dt, M)
    o2 = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    assert o2.courant(u, wl.dt, 3) == rm.courant(None, u, wl.dt, 3)
    f, c = o2.courant(u, wl.dt, 3)
    assert f == c > 0


@pytest.mark.parametrize("width", [2, 3])
def test_restatement_wide_interfaces_match_reference(ref_lib, width):
    """make_regions with interface bands of `width` layers (regions.cpp:69-105)
    and the LTS steps on them: restatement = reference, bitwise."""
    from oracle.oracle import RefEvaluator, RefMesh, RefRegions
    wl = W.small_sphere(4, seed=9, cap_deg=35.0)
    rm = RefMesh.from_mesh(wl.mesh)
    rr = RefRegions(rm, wl.fine_mask, width)
    ev = RefEvaluator(rm, rr, wl.b, wl.f, wl.gravity)
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, width)
    assert all(np.array_equal(a, b) for a, b in zip(rr.groups(), o.groups()))
    for scheme in (Scheme.LTS3, Scheme.LTS2):
        h1, u1, _, _ = ev.step(int(scheme), wl.h, wl.u, 0.0, wl.dt, wl.M, 3)
        h2, u2, _ = o.step(int(scheme), wl.h, wl.u, 0.0, wl.dt, wl.M, 3)
        assert bits_equal(h1, h2) and bits_equal(u1, u2), scheme

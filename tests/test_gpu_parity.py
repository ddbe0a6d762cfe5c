"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Bar: bitwise equality for region labels, group lists, closure sets,
tendencies and prognostic states (the path keeps the reference's IEEE
operation order and is built with --fmad=false), which is stricter than
north_star's 1e-11 relative max-norm after 100 coarse steps; the 1e-11
bound is asserted too where north_star states it.
"""
import numpy as np
import pytest

from helpers import bits_equal, golden_mesh, load_golden, max_rel, workload
from make_golden import mesh_digest
from oracle.oracle import Oracle
from paper_2106_07154_b200 import workloads as W
from paper_2106_07154_b200.api import (LTS3_MASKS, ConfigError, CudaContext, CudaEvaluator,
                                       CudaStepper, DryVertexError, Scheme, SchemeConfig, State,
                                       UsageError, kMaskAll)
from paper_2106_07154_b200.mesh import Mesh

pytestmark = pytest.mark.gpu

FIXTURES = ["planar24", "sphereL3"]
SENTINEL = 123456789.0


def _ctx(wl_or_mesh, b, f, g, fine=None, width=1):
    ctx = CudaContext(wl_or_mesh, b, f, g)
    if fine is not None:
        ctx.make_regions(fine, width)
    return ctx


@pytest.mark.parametrize("name", FIXTURES)
def test_golden_regions_tendencies_steps(name):
    g = load_golden(name)
    mesh = golden_mesh(name)
    assert mesh_digest(mesh) == str(g["digest"])
    ctx = _ctx(mesh, g["b"], g["f"], float(g["gravity"]), g["fine"])
    rm = ctx.regions
    assert np.array_equal(rm.cell_label, g["cell_label"])
    assert np.array_equal(rm.cell_sublabel, g["cell_sub"])
    assert np.array_equal(rm.edge_label, g["edge_label"])
    for gi in range(11):
        assert np.array_equal(rm.groups[gi], g[f"group{gi}"]), gi
    ev = CudaEvaluator(ctx)
    for mask in LTS3_MASKS + [kMaskAll]:
        dh = np.full(mesh.n_cells, np.nan)
        du = np.full(mesh.n_edges, np.nan)
        ev.eval(g["h"], g["u"], mask, dh, du)
        assert bits_equal(dh, g[f"dh_{mask}"]), hex(mask)
        assert bits_equal(du, g[f"du_{mask}"]), hex(mask)
        for kind in range(4):
            assert np.array_equal(ctx.closure(mask, kind), g[f"closure_{mask}_{kind}"]), (mask, kind)
    M, dt = int(g["M"]), float(g["dt"])
    for scheme, n in [(Scheme.LTS3, 3), (Scheme.RK4, 2), (Scheme.SSPRK3, 2)]:
        c2 = _ctx(mesh, g["b"], g["f"], float(g["gravity"]), g["fine"])
        c2.upload(State(g["h"], g["u"], 0.0))
        c2.advance(scheme, dt if scheme == Scheme.LTS3 else dt / M, M, n)
        st = c2.download()
        assert bits_equal(st.h, g[f"h_{scheme.name}"]), scheme
        assert bits_equal(st.u, g[f"u_{scheme.name}"]), scheme
        lg = c2.ledger()
        assert np.array_equal(lg.cell_evals, g[f"ledger_cell_{scheme.name}"])
        assert np.array_equal(lg.edge_evals, g[f"ledger_edge_{scheme.name}"])


def _oracle_for(wl):
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, wl.width)
    return o


def test_c1_lts3_100_steps_bitwise():
    """BASELINE configs[0]: 100 LTS3 coarse steps on 1 GPU vs the CPU oracle."""
    wl = W.config1()
    o = _oracle_for(wl)
    h_ref, u_ref, t_ref = o.step(int(Scheme.LTS3), wl.h, wl.u, 0.0, wl.dt, wl.M, wl.n_steps)
    ctx = _ctx(wl.mesh, wl.b, wl.f, wl.gravity, wl.fine_mask)
    for a, b in zip(ctx.regions.groups, o.groups()):
        assert np.array_equal(a, b)
    ctx.upload(State(wl.h, wl.u, 0.0))
    ctx.advance(Scheme.LTS3, wl.dt, wl.M, wl.n_steps)
    st = ctx.download()
    assert max_rel(st.h, h_ref) <= 1e-11 and max_rel(st.u, u_ref, 1.0) <= 1e-11
    assert bits_equal(st.h, h_ref) and bits_equal(st.u, u_ref)
    assert st.time == pytest.approx(t_ref)
    c, e, s = o.ledger()
    lg = ctx.ledger()
    assert np.array_equal(lg.cell_evals, c) and np.array_equal(lg.edge_evals, e)
    assert lg.steps_taken == s == wl.n_steps


@pytest.mark.parametrize("M", [1, 2, 5])
def test_sphere_lts3_and_rk4_bitwise(M):
    wl = W.small_sphere(5, seed=7, cap_deg=25.0, M=M)
    o = _oracle_for(wl)
    ctx = _ctx(wl.mesh, wl.b, wl.f, wl.gravity, wl.fine_mask)
    for scheme, n, dt in [(Scheme.LTS3, 6, wl.dt), (Scheme.RK4, 3, wl.dt / M),
                          (Scheme.SSPRK3, 3, wl.dt / M), (Scheme.LTS2, 6, wl.dt),
                          (Scheme.SSPRK2, 3, wl.dt / M)]:
        h_ref, u_ref, _ = o.step(int(scheme), wl.h, wl.u, 0.0, dt, M, n)
        ctx.upload(State(wl.h, wl.u, 0.0))
        ctx.advance(scheme, dt, M, n)
        st = ctx.download()
        assert bits_equal(st.h, h_ref) and bits_equal(st.u, u_ref), scheme


def test_c1_lts2_bitwise():
    """Second-order LTS (Stepper::lts_step(2, ...)) on the device: coarse
    steps and the ledger against the oracle (40 steps: at C1's LTS3 time step
    the second-order scheme dries a vertex by step 100)."""
    wl = W.config1(n_steps=40)
    o = _oracle_for(wl)
    h_ref, u_ref, t_ref = o.step(int(Scheme.LTS2), wl.h, wl.u, 0.0, wl.dt, wl.M, wl.n_steps)
    ctx = _ctx(wl.mesh, wl.b, wl.f, wl.gravity, wl.fine_mask)
    ctx.upload(State(wl.h, wl.u, 0.0))
    ctx.advance(Scheme.LTS2, wl.dt, wl.M, wl.n_steps)
    st = ctx.download()
    assert bits_equal(st.h, h_ref) and bits_equal(st.u, u_ref)
    assert st.time == pytest.approx(t_ref)
    c, e, s = o.ledger()
    lg = ctx.ledger()
    assert np.array_equal(lg.cell_evals, c) and np.array_equal(lg.edge_evals, e)
    assert lg.steps_taken == s == wl.n_steps


def test_c2_full_size_parity():
    """BASELINE configs[1] at full size: regions bit-exact, all masks bitwise,
    5 coarse steps bitwise against the oracle."""
    wl = W.config2(n_steps=5)
    o = _oracle_for(wl)
    ctx = _ctx(wl.mesh, wl.b, wl.f, wl.gravity, wl.fine_mask)
    cl, cs, el = o.labels()
    assert np.array_equal(ctx.regions.cell_label, cl)
    assert np.array_equal(ctx.regions.cell_sublabel, cs)
    assert np.array_equal(ctx.regions.edge_label, el)
    for a, b in zip(ctx.regions.groups, o.groups()):
        assert np.array_equal(a, b)
    ev = CudaEvaluator(ctx)
    for mask in LTS3_MASKS:
        dh1 = np.full(wl.mesh.n_cells, SENTINEL)
        du1 = np.full(wl.mesh.n_edges, SENTINEL)
        dh2, du2 = dh1.copy(), du1.copy()
        ev.eval(wl.h, wl.u, mask, dh1, du1)
        o.eval(wl.h, wl.u, mask, dh2, du2)
        assert bits_equal(dh1, dh2) and bits_equal(du1, du2)
    h_ref, u_ref, _ = o.step(int(Scheme.LTS3), wl.h, wl.u, 0.0, wl.dt, wl.M, wl.n_steps)
    ctx.upload(State(wl.h, wl.u, 0.0))
    ctx.advance(Scheme.LTS3, wl.dt, wl.M, wl.n_steps)
    st = ctx.download()
    assert bits_equal(st.h, h_ref) and bits_equal(st.u, u_ref)


def test_restricted_evaluation_bitwise_equal_full():
    # test_operators.cpp:164-202 through the masked-group interface
    wl = W.small_sphere(4, seed=5)
    ctx = _ctx(wl.mesh, wl.b, wl.f, wl.gravity, wl.fine_mask)
    ev = CudaEvaluator(ctx)
    m = wl.mesh
    dh_full = np.full(m.n_cells, SENTINEL)
    du_full = np.full(m.n_edges, SENTINEL)
    ev.eval(wl.h, wl.u, kMaskAll, dh_full, du_full)
    for mask in [0x1, 0x20, 0x400, 0x41, 0x28 | 0x500, 0x7FF & ~0x21, 0x5 | 0x280]:
        dh = np.full(m.n_cells, SENTINEL)
        du = np.full(m.n_edges, SENTINEL)
        ev.eval(wl.h, wl.u, mask, dh, du)
        in_c = np.zeros(m.n_cells, bool)
        in_e = np.zeros(m.n_edges, bool)
        for gi in range(6):
            if mask & (1 << gi):
                in_c[ctx.regions.groups[gi]] = True
        for gi in range(6, 11):
            if mask & (1 << gi):
                in_e[ctx.regions.groups[gi]] = True
        assert bits_equal(dh, np.where(in_c, dh_full, SENTINEL))
        assert bits_equal(du, np.where(in_e, du_full, SENTINEL))


def test_m1_lts3_reduces_to_ssprk3():
    # acceptance criterion 1 (acceptance.cpp:98-118), both on the device
    wl = W.small_sphere(4, seed=9, M=1)
    ctx = _ctx(wl.mesh, wl.b, wl.f, wl.gravity, wl.fine_mask)
    ctx.upload(State(wl.h, wl.u, 0.0))
    ctx.advance(Scheme.LTS3, wl.dt, 1, 10)
    a = ctx.download()
    ctx.upload(State(wl.h, wl.u, 0.0))
    ctx.advance(Scheme.SSPRK3, wl.dt, 1, 10)
    b = ctx.download()
    assert max_rel(a.h, b.h) <= 1e-12
    assert np.max(np.abs(a.u - b.u) / np.maximum(np.abs(b.u), 1.0)) <= 1e-12


def test_mass_conservation_100_steps():
    # acceptance criterion 3 (acceptance.cpp:147-166): drift <= 1e-11
    wl = W.config1()
    ctx = _ctx(wl.mesh, wl.b, wl.f, wl.gravity, wl.fine_mask)
    ctx.upload(State(wl.h, wl.u, 0.0))
    m0 = ctx.total_mass()
    assert m0 == wl.mesh.total_mass(wl.h)
    ctx.advance(Scheme.LTS3, wl.dt, wl.M, 100)
    m1 = ctx.total_mass()
    assert abs(m1 - m0) / abs(m0) <= 1e-11


def test_ledger_matches_hand_derived_formulas():
    # test_integrators.cpp:254-276
    wl = W.small_sphere(4, seed=3)
    ctx = _ctx(wl.mesh, wl.b, wl.f, wl.gravity, wl.fine_mask)
    G = [len(x) for x in ctx.regions.groups]
    Fc, U1, U2, I1, I2, Cc = G[0] + G[1] + G[2], G[1], G[2], G[3], G[4], G[5]
    Fe, Ue, E1, E2, Ce = G[6] + G[7], G[7], G[8], G[9], G[10]
    for M in (1, 2, 4):
        ctx.reset_ledger()
        ctx.upload(State(wl.h, wl.u, 0.0))
        ctx.advance(Scheme.LTS3, wl.dt, M, 1)
        lg = ctx.ledger()
        assert lg.cell_evals[0][0] == U1 + U2 + M * Fc
        assert lg.edge_evals[0][0] == Ue + M * Fe
        assert lg.cell_evals[1][0] == I1 + M * I1
        assert lg.cell_evals[3][0] == Cc
        assert lg.cell_evals[2][1] == I2 + M * I2
        assert lg.cell_evals[3][2] == Cc
        assert lg.total_cell_evals() == (U1 + U2 + I1 + I2 + Cc) + (I1 + I2 + Cc) + Cc \
            + 3 * M * (Fc + I1 + I2)
        assert lg.total_edge_evals() == (Ue + E1 + E2 + Ce) + (E1 + E2 + Ce) + Ce \
            + 3 * M * (Fe + E1 + E2)


def test_dry_vertex_reported():
    # test_operators.cpp:222-242
    m = Mesh.icosahedral(0, 1.0)
    h = np.ones(m.n_cells)
    h[4] = -40.0
    u = np.full(m.n_edges, 0.1)
    ctx = CudaContext(m, np.zeros(m.n_cells), np.zeros(m.n_vertices), 9.80616)
    with pytest.raises(DryVertexError) as err:
        CudaEvaluator(ctx).eval(h, u, kMaskAll, np.zeros(m.n_cells), np.zeros(m.n_edges))
    v = err.value.vertex
    assert 0 <= v < m.n_vertices and 4 in m.vertex_cells[v]


def _draining_workload():
    """A fine cell with a strong outward flow: the reference's LTS3 raises
    DryVertexError in step 3 (found with the oracle)."""
    wl = W.small_sphere(4, seed=5, cap_deg=30.0)
    T = wl.mesh.tables
    i = int(np.nonzero(wl.fine_mask)[0][len(np.nonzero(wl.fine_mask)[0]) // 2])
    off, ce = T["cell_offset"], T["cell_edges"]
    ec, es = T["edge_cells"].reshape(-1, 2), T["edge_cell_sign"].reshape(-1, 2)
    u = wl.u.copy()
    for k in range(off[i], off[i + 1]):
        e = ce[k]
        u[e] = 250.0 * (es[e, 0] if ec[e, 0] == i else es[e, 1])
    return wl, u


@pytest.mark.parametrize("sync", [True, False])
def test_dry_vertex_step_reported(sync):
    """harness.cpp:183-190: the error names the step of the batch in which
    the vertex went dry (kernel A records (step, vertex) on the device); an
    asynchronous batch reports it at the next synchronous call, once."""
    from oracle.oracle import OracleError
    wl, u = _draining_workload()
    o = _oracle_for(wl)
    hh, uu, k_ref, v_ref = wl.h, u, None, None
    for k in range(1, 7):
        try:
            hh, uu, _ = o.step(int(Scheme.LTS3), hh, uu, 0.0, wl.dt, wl.M, 1)
        except OracleError as ex:
            k_ref, v_ref = k, ex.vertex
            break
    assert k_ref == 3
    ctx = _ctx(wl.mesh, wl.b, wl.f, wl.gravity, wl.fine_mask)
    ctx.upload(State(wl.h, u, 0.0))
    ctx.advance(Scheme.LTS3, wl.dt, wl.M, 1)   # a clean batch first: steps are per batch
    with pytest.raises(DryVertexError) as err:
        ctx.advance(Scheme.LTS3, wl.dt, wl.M, 5, sync=sync)
        if not sync:
            ctx.download()
    assert err.value.step == k_ref - 1, str(err.value)
    assert f"during step {k_ref - 1} of 5" in str(err.value)
    v = err.value.vertex
    vc = wl.mesh.tables["vertex_cells"].reshape(-1, 3)
    assert 0 <= v < wl.mesh.n_vertices
    assert set(vc[v]) & set(vc[v_ref]), (v, v_ref)   # next to the drained cell
    ctx.sync()                                        # reported once, then cleared


def test_usage_and_config_errors():
    wl = W.small_sphere(3)
    ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity)
    ev = CudaEvaluator(ctx)
    z = (np.zeros(wl.mesh.n_cells), np.zeros(wl.mesh.n_edges))
    with pytest.raises(UsageError):          # integrators.cpp:139-142
        ev.eval(wl.h, wl.u, 0x21, *z)
    ctx.upload(State(wl.h, wl.u, 0.0))
    with pytest.raises(ConfigError):         # integrators.cpp:413-421
        ctx.advance(Scheme.LTS3, wl.dt, 4, 1)
    with pytest.raises(ConfigError):
        ctx.advance(Scheme.RK4, -1.0, 1, 1)
    with pytest.raises(ConfigError):         # regions.cpp:77-79
        ctx.make_regions(np.zeros(wl.mesh.n_cells, np.uint8))
    ctx.make_regions(wl.fine_mask)
    with pytest.raises(ConfigError):
        ctx.advance(Scheme.LTS3, wl.dt, 0, 1)


def test_stepper_drop_in_interface():
    wl = W.small_sphere(3, seed=4)
    ctx = _ctx(wl.mesh, wl.b, wl.f, wl.gravity, wl.fine_mask)
    o = _oracle_for(wl)
    st = State(wl.h.copy(), wl.u.copy(), 0.0)
    CudaStepper(ctx).step(st, SchemeConfig(Scheme.LTS3, wl.dt, wl.M))
    h_ref, u_ref, _ = o.step(int(Scheme.LTS3), wl.h, wl.u, 0.0, wl.dt, wl.M, 1)
    assert bits_equal(st.h, h_ref) and bits_equal(st.u, u_ref)


@pytest.mark.parametrize("kout,env", [("explicit", {"MSWM_ST16": "1"}),
                                      ("explicit", {"MSWM_ST16": "0"}),
                                      ("explicit", {"MSWM_ST16": "1", "MSWM_PACK16": "0"})])
def test_layouts_are_bitwise_equivalent(kout, env, monkeypatch):
    """Results are independent of the device numbering (input, Hilbert,
    region-major, random) and of the stencil-id table (16-bit offsets or the
    int32 table)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    st16 = env.get("MSWM_ST16", "1")
    wl = W.small_sphere(5, seed=13, cap_deg=20.0)
    o = _oracle_for(wl)
    h_ref, u_ref, _ = o.step(int(Scheme.LTS3), wl.h, wl.u, 0.0, wl.dt, wl.M, 4)
    rng = np.random.default_rng(0)
    for order in ["input", "hilbert", "regions",
                  rng.permutation(wl.mesh.n_cells).astype(np.int32)]:
        ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, order=order, fine_mask=wl.fine_mask)
        assert ctx.layout_info()["kernel_path"] == kout
        assert ctx.stencil_info()["offsets16"] == (st16 == "1")
        ctx.make_regions(wl.fine_mask, wl.width)
        for a, b in zip(ctx.regions.groups, o.groups()):
            assert np.array_equal(a, b)
        for mask in LTS3_MASKS:
            for kind in range(4):
                o_dh = np.zeros(wl.mesh.n_cells)
                o_du = np.zeros(wl.mesh.n_edges)
                o.eval(wl.h, wl.u, mask, o_dh, o_du)
                assert np.array_equal(ctx.closure(mask, kind), np.sort(o.last_closure(kind)))
        ctx.upload(State(wl.h, wl.u, 0.0))
        ctx.advance(Scheme.LTS3, wl.dt, wl.M, 4)
        st = ctx.download()
        assert bits_equal(st.h, h_ref) and bits_equal(st.u, u_ref), str(order)[:20]


def test_planar_rk4_full_mesh():
    wl = W.config1(n_steps=3)
    o = _oracle_for(wl)
    ctx = _ctx(wl.mesh, wl.b, wl.f, wl.gravity, wl.fine_mask)
    assert ctx.layout_info()["input_order"] is False
    h_ref, u_ref, _ = o.step(int(Scheme.RK4), wl.h, wl.u, 0.0, wl.dt / 4, 1, 5)
    ctx.upload(State(wl.h, wl.u, 0.0))
    ctx.advance(Scheme.RK4, wl.dt / 4, 1, 5)
    st = ctx.download()
    assert bits_equal(st.h, h_ref) and bits_equal(st.u, u_ref)


def test_reference_stepper_drives_cuda_evaluator():
    """The C++ drop-in: the reference's own Stepper::lts_step with its
    evaluator slot filled by mswm::CudaEvaluator (oracle/drop_in_evaluator.hpp
    over the C ABI) reproduces the reference with SerialEvaluator bitwise."""
    from oracle.oracle import RefEvaluator, RefMesh, RefRegions, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    wl = W.small_sphere(4, seed=17, cap_deg=30.0)
    rm = RefMesh.from_mesh(wl.mesh)
    rr = RefRegions(rm, wl.fine_mask, wl.width)
    serial = RefEvaluator(rm, rr, wl.b, wl.f, wl.gravity)
    cuda = RefEvaluator.cuda(rm, rr, wl.b, wl.f, wl.gravity)
    for scheme, dt in [(Scheme.LTS3, wl.dt), (Scheme.RK4, wl.dt / wl.M)]:
        h1, u1, _, _ = serial.step(int(scheme), wl.h, wl.u, 0.0, dt, wl.M, 3)
        h2, u2, _, _ = cuda.step(int(scheme), wl.h, wl.u, 0.0, dt, wl.M, 3)
        assert bits_equal(h1, h2) and bits_equal(u1, u2), scheme
    c1, e1, _ = serial.ledger()
    c2, e2, _ = cuda.ledger()
    assert np.array_equal(c1, c2) and np.array_equal(e1, e2)


@pytest.mark.parametrize("order", ["hilbert", "input"])
def test_device_diagnostics(order):
    """total_mass / total_energy (harness.cpp:99-123) and courant_numbers
    (integrators.cpp:632-659) of the device state: exact mode and Courant
    numbers bitwise the oracle, the device tree sum within 1e-13."""
    wl = W.small_sphere(5, seed=41, cap_deg=25.0)
    o = _oracle_for(wl)
    h, u, _ = o.step(int(Scheme.LTS3), wl.h, wl.u, 0.0, wl.dt, wl.M, 3)
    ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, order=order)
    ctx.upload(State(h, u, 0.0))
    o_nomap = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    assert ctx.courant(wl.dt, 4) == o_nomap.courant(u, wl.dt, 4)
    ctx.make_regions(wl.fine_mask, wl.width)
    m, e = ctx.diagnostics(exact=True)
    assert m == o.total_mass(h) and e == o.total_energy(h, u)
    assert ctx.total_mass() == m
    mf, ef = ctx.diagnostics(exact=False)
    assert abs(mf - m) <= 1e-13 * abs(m) and abs(ef - e) <= 1e-13 * abs(e)
    for M in (1, 4, 7):
        assert ctx.courant(wl.dt, M) == o.courant(u, wl.dt, M)
    with pytest.raises(UsageError):
        ctx.courant(wl.dt, 0)


def test_eval_profile_levels():
    """set_profiling(1) brackets all 3M+3 evaluations of an LTS3 step with
    events, set_profiling(2) only the first one covering half the mesh (the
    bench's roofline kernel); profiling never changes the results."""
    wl = W.small_sphere(5, seed=43, cap_deg=25.0)
    ref = None
    for level, n_evals in [(0, 0), (1, 3 * wl.M + 3), (2, 1)]:
        ctx = _ctx(wl.mesh, wl.b, wl.f, wl.gravity, wl.fine_mask)
        ctx.set_profiling(level)
        ctx.upload(State(wl.h, wl.u, 0.0))
        ctx.advance(Scheme.LTS3, wl.dt, wl.M, 2)
        ms, nc, ne = ctx.eval_profile()
        assert len(ms) == n_evals and np.all(ms > 0)
        if level == 2:
            assert 2 * (nc[0] + ne[0]) >= wl.mesh.n_cells + wl.mesh.n_edges
        st = ctx.download()
        if ref is None:
            ref = st
        assert bits_equal(st.h, ref.h) and bits_equal(st.u, ref.u)
    with pytest.raises(UsageError):
        ctx.set_profiling(3)


@pytest.mark.parametrize("width", [2, 3])
def test_wide_interfaces_bitwise(width):
    """Interface bands of `width` layers each (make_regions width,
    regions.cpp:69-105; the paper widens them to tens of layers): regions,
    every LTS3 mask, LTS3 and LTS2 steps bitwise against the oracle, in the
    Hilbert and region-major layouts."""
    wl = W.small_sphere(5, seed=47, cap_deg=20.0)
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, width)
    for order in ["hilbert", "regions"]:
        ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, order=order, fine_mask=wl.fine_mask,
                          interface_width=width)
        ctx.make_regions(wl.fine_mask, width)
        for a, b in zip(ctx.regions.groups, o.groups()):
            assert np.array_equal(a, b)
        ev = CudaEvaluator(ctx)
        for mask in LTS3_MASKS:
            dh1 = np.full(wl.mesh.n_cells, SENTINEL)
            du1 = np.full(wl.mesh.n_edges, SENTINEL)
            dh2, du2 = dh1.copy(), du1.copy()
            ev.eval(wl.h, wl.u, mask, dh1, du1)
            o.eval(wl.h, wl.u, mask, dh2, du2)
            assert bits_equal(dh1, dh2) and bits_equal(du1, du2), hex(mask)
        for scheme in (Scheme.LTS3, Scheme.LTS2):
            h_ref, u_ref, _ = o.step(int(scheme), wl.h, wl.u, 0.0, wl.dt, wl.M, 3)
            ctx.upload(State(wl.h, wl.u, 0.0))
            ctx.advance(scheme, wl.dt, wl.M, 3)
            st = ctx.download()
            assert bits_equal(st.h, h_ref) and bits_equal(st.u, u_ref), (order, scheme)


@pytest.mark.parametrize("fork", ["1", "0"])
@pytest.mark.parametrize("order", ["regions", "hilbert"])
def test_concurrent_coarse_step_bitwise(fork, order, monkeypatch):
    """LTS3 with the coarse step (step 4) on a second stream concurrent with
    the substeps (default) and in sequence (MSWM_FORK=0): bitwise equal to
    the oracle over several coarse steps, M = 2 and 4."""
    monkeypatch.setenv("MSWM_FORK", fork)
    wl = W.small_sphere(6, seed=41, cap_deg=25.0)
    o = _oracle_for(wl)
    ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, order=order, fine_mask=wl.fine_mask)
    ctx.make_regions(wl.fine_mask, wl.width)
    for M in (4, 2):
        h_ref, u_ref, _ = o.step(int(Scheme.LTS3), wl.h, wl.u, 0.0, wl.dt, M, 5)
        ctx.upload(State(wl.h, wl.u, 0.0))
        ctx.advance(Scheme.LTS3, wl.dt, M, 5)
        st = ctx.download()
        assert bits_equal(st.h, h_ref) and bits_equal(st.u, u_ref), M


@pytest.mark.parametrize("st16", ["1", "0"])
def test_stencil_offsets16_bitwise(st16, monkeypatch):
    """16-bit stencil offsets (default) with edges whose offsets overflow
    int16 (a random numbering of a level-6 sphere: 123k edges, most offsets
    wide, warps mixing both kinds) and the int32-only table: bitwise equal."""
    monkeypatch.setenv("MSWM_ST16", st16)
    wl = W.small_sphere(6, seed=31, cap_deg=20.0)
    o = _oracle_for(wl)
    h_ref, u_ref, _ = o.step(int(Scheme.LTS3), wl.h, wl.u, 0.0, wl.dt, wl.M, 2)
    rng = np.random.default_rng(3)
    for order in ["regions", rng.permutation(wl.mesh.n_cells).astype(np.int32)]:
        ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, order=order, fine_mask=wl.fine_mask)
        info = ctx.stencil_info()
        assert info["offsets16"] == (st16 == "1")
        if not isinstance(order, str):
            assert 0 < info["n_wide"] < wl.mesh.n_edges
        ctx.make_regions(wl.fine_mask, wl.width)
        ev = CudaEvaluator(ctx)
        for mask in LTS3_MASKS:
            dh1 = np.full(wl.mesh.n_cells, SENTINEL)
            du1 = np.full(wl.mesh.n_edges, SENTINEL)
            dh2, du2 = dh1.copy(), du1.copy()
            ev.eval(wl.h, wl.u, mask, dh1, du1)
            o.eval(wl.h, wl.u, mask, dh2, du2)
            assert bits_equal(dh1, dh2) and bits_equal(du1, du2)
        ctx.upload(State(wl.h, wl.u, 0.0))
        ctx.advance(Scheme.LTS3, wl.dt, wl.M, 2)
        st = ctx.download()
        assert bits_equal(st.h, h_ref) and bits_equal(st.u, u_ref)


@pytest.mark.parametrize("pack16", ["1", "0"])
def test_index_records16_bitwise(pack16, monkeypatch):
    """16-bit index records of kernels A, B, C (default) against the int32
    tables: bitwise equal on the region-major numbering (a few wide elements
    at region seams) and on a random numbering (most elements wide, warps
    mixing both kinds), sphere (pentagons: padded ring slots) and plane."""
    monkeypatch.setenv("MSWM_PACK16", pack16)
    rng = np.random.default_rng(5)
    for wl in [W.small_sphere(6, seed=37, cap_deg=20.0), W.config1(n_steps=2)]:
        o = _oracle_for(wl)
        h_ref, u_ref, _ = o.step(int(Scheme.LTS3), wl.h, wl.u, 0.0, wl.dt, wl.M, 2)
        for order in ["regions", rng.permutation(wl.mesh.n_cells).astype(np.int32)]:
            ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, order=order,
                              fine_mask=wl.fine_mask)
            info = ctx.index_info()
            assert info["packed16"] == (pack16 == "1")
            if pack16 == "1":
                assert info["cell_records"]
                if not isinstance(order, str) and wl.mesh.n_edges > 1 << 16:
                    for k in ("n_wide_vertices", "n_wide_cells", "n_wide_edges"):
                        assert 0 < info[k], k
            ctx.make_regions(wl.fine_mask, wl.width)
            ev = CudaEvaluator(ctx)
            for mask in LTS3_MASKS:
                dh1 = np.full(wl.mesh.n_cells, SENTINEL)
                du1 = np.full(wl.mesh.n_edges, SENTINEL)
                dh2, du2 = dh1.copy(), du1.copy()
                ev.eval(wl.h, wl.u, mask, dh1, du1)
                o.eval(wl.h, wl.u, mask, dh2, du2)
                assert bits_equal(dh1, dh2) and bits_equal(du1, du2)
            ctx.upload(State(wl.h, wl.u, 0.0))
            ctx.advance(Scheme.LTS3, wl.dt, wl.M, 2)
            st = ctx.download()
            assert bits_equal(st.h, h_ref) and bits_equal(st.u, u_ref)


@pytest.mark.parametrize("mix,win", [("0", None), ("1", None), ("3", None), ("12", "7"),
                                     ("25", None), ("29", "3"), ("25", "1000")])
def test_chunk_schedules_bitwise(mix, win, monkeypatch):
    """Chunk schedules of the evaluation kernels (MSWM_MIX: none, kernel A /
    C interleaved in proportion, windowed with few / one-chunk windows, ping-pong
    directions; the default is 25): every order of the same elements gives the
    same bits -- every LTS3 mask's tendencies and 3 coarse steps against the
    oracle, on a sphere (hilbert and region-major numbering) and a plane."""
    monkeypatch.setenv("MSWM_MIX", mix)
    if win:
        monkeypatch.setenv("MSWM_MIX_WIN", win)
    for wl in [W.small_sphere(6, seed=41, cap_deg=20.0), W.config1(n_steps=3)]:
        o = _oracle_for(wl)
        h_ref, u_ref, _ = o.step(int(Scheme.LTS3), wl.h, wl.u, 0.0, wl.dt, wl.M, 3)
        for order in ["hilbert", "regions"]:
            ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, order=order,
                              fine_mask=wl.fine_mask)
            ctx.make_regions(wl.fine_mask, wl.width)
            ev = CudaEvaluator(ctx)
            for mask in LTS3_MASKS + [kMaskAll]:
                dh1 = np.full(wl.mesh.n_cells, SENTINEL)
                du1 = np.full(wl.mesh.n_edges, SENTINEL)
                dh2, du2 = dh1.copy(), du1.copy()
                ev.eval(wl.h, wl.u, mask, dh1, du1)
                o.eval(wl.h, wl.u, mask, dh2, du2)
                assert bits_equal(dh1, dh2) and bits_equal(du1, du2), hex(mask)
            ctx.upload(State(wl.h, wl.u, 0.0))
            ctx.advance(Scheme.LTS3, wl.dt, wl.M, 3)
            st = ctx.download()
            assert bits_equal(st.h, h_ref) and bits_equal(st.u, u_ref)


@pytest.mark.parametrize("config", ["c4", "c3"])
def test_full_size_against_reference(config):
    """BASELINE configs at full size against the unmodified reference
    (oracle/_ref, ThreadedEvaluator -- bitwise partition-invariant,
    acceptance.cpp:205-244): C4 = north_star's target mesh (icosahedral level
    10, 10,485,762 cells, 20-degree cap, M = 4), C3 = planar 2048^2 (4.2M
    cells, four fine circles, beta-plane, M = 8).  Region labels and the 11
    group lists bit-exact, every LTS3 mask's tendencies bitwise, h, u after 2
    coarse LTS3 steps bitwise (so within north_star's 1e-11 relative
    max-norm, also asserted)."""
    import os
    from oracle.oracle import RefEvaluator, RefMesh, RefRegions, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    wl = workload(config)
    nC, nE = wl.mesh.n_cells, wl.mesh.n_edges
    rm = RefMesh.from_mesh(wl.mesh)
    rr = RefRegions(rm, wl.fine_mask, wl.width)
    ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, order="regions", fine_mask=wl.fine_mask)
    ctx.make_regions(wl.fine_mask, wl.width)
    cl, cs, el = rr.labels(nC, nE)
    assert np.array_equal(ctx.regions.cell_label, cl)
    assert np.array_equal(ctx.regions.cell_sublabel, cs)
    assert np.array_equal(ctx.regions.edge_label, el)
    for a, b in zip(ctx.regions.groups, rr.groups()):
        assert np.array_equal(a, b)
    # full-size host arrays per rank block: keep the rank count inside host RAM
    ranks = max(1, min(8, len(os.sched_getaffinity(0))))
    ref = RefEvaluator(rm, rr, wl.b, wl.f, wl.gravity, nranks=ranks)
    ev = CudaEvaluator(ctx)
    for mask in LTS3_MASKS:
        dh1 = np.full(nC, SENTINEL)
        du1 = np.full(nE, SENTINEL)
        dh2, du2 = dh1.copy(), du1.copy()
        ev.eval(wl.h, wl.u, mask, dh1, du1)
        ref.eval(wl.h, wl.u, mask, dh2, du2)
        assert bits_equal(dh1, dh2) and bits_equal(du1, du2), mask
    h_ref, u_ref, _, _ = ref.step(int(Scheme.LTS3), wl.h, wl.u, 0.0, wl.dt, wl.M, 2)
    ctx.upload(State(wl.h, wl.u, 0.0))
    ctx.advance(Scheme.LTS3, wl.dt, wl.M, 2)
    st = ctx.download()
    assert max_rel(st.h, h_ref) <= 1e-11 and max_rel(st.u, u_ref) <= 1e-11
    assert bits_equal(st.h, h_ref) and bits_equal(st.u, u_ref)


def test_region_edge_cases_match_reference(ref_lib):
    """make_regions on degenerate inputs (regions.cpp:69-105): every fine
    predicate the reference rejects raises ConfigError on the device too
    (no fine cell, every cell fine, interface layers exhausting the non-fine
    cells, an empty layer, width 0); the ones it accepts -- a single fine
    cell, fine cells that touch no interface (underline layers empty, with
    its warnings) -- give bit-exact labels and groups."""
    wl = W.small_sphere(3, seed=8)
    n = wl.mesh.n_cells
    rm = ref_lib.RefMesh.from_mesh(wl.mesh)
    rng = np.random.default_rng(3)
    one = np.zeros(n, np.uint8)
    one[7] = 1
    almost = np.ones(n, np.uint8)
    almost[rng.choice(n, 3, replace=False)] = 0
    cases = [(np.zeros(n, np.uint8), 1), (np.ones(n, np.uint8), 1), (almost, 1), (one, 1),
             (one, 2), (one, 4), (wl.fine_mask, 3), (wl.fine_mask, 0),
             ((rng.random(n) < 0.3).astype(np.uint8), 1)]
    for mask, width in cases:
        try:
            rr = ref_lib.RefRegions(rm, mask, width)
            ref_err = None
        except ref_lib.OracleError as e:
            ref_err = e
        ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity)
        if ref_err is not None:
            assert ref_err.status == 1
            with pytest.raises(ConfigError):
                ctx.make_regions(mask, width)
            continue
        got = ctx.make_regions(mask, width)
        cl, cs, el = rr.labels(n, wl.mesh.n_edges)
        assert np.array_equal(got.cell_label, cl) and np.array_equal(got.cell_sublabel, cs)
        assert np.array_equal(got.edge_label, el)
        for a, b in zip(got.groups, rr.groups()):
            assert np.array_equal(a, b)
        assert len(got.warnings) == rr.n_warnings, (width, got.warnings)


def _first_ids(msgs):
    """validate_regions messages -> {check kind: first offending id} (regions.cpp:213-286)."""
    import re
    pat = [(1, r"^Interface1 cell (\d+) at distance"), (2, r"^Interface2 cell (\d+) at distance"),
           (3, r"^coarse cell (\d+) at distance"),
           (4, r"^fine cell (\d+) has the wrong underline sublabel"),
           (5, r"^edge (\d+) label disagrees")]
    out = {}
    for m in msgs:
        for kind, p in pat:
            hit = re.match(p, m)
            if hit:
                out.setdefault(kind, int(hit.group(1)))
    return out


@pytest.mark.parametrize("width", [1, 2])
def test_validate_regions_matches_reference(ref_lib, width):
    """validate_regions (regions.cpp:173-288) on the device: a valid map
    passes; labels corrupted one check kind at a time (and all at once) are
    flagged for the kinds the reference flags, naming the same first element."""
    from paper_2106_07154_b200.api import RegionMap
    wl = W.small_sphere(4, seed=5)
    nC, nE = wl.mesh.n_cells, wl.mesh.n_edges
    rm = ref_lib.RefMesh.from_mesh(wl.mesh)
    rr = ref_lib.RefRegions(rm, wl.fine_mask, width)
    for order in ("input", "hilbert"):  # identity and permuted internal numbering
        ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, order=order)
        good = ctx.make_regions(wl.fine_mask, width)
        rep = ctx.validate_regions()
        assert rep.ok() and rep.counts == [0] * 6 and rep.first == [-1] * 6
        assert rr.validate() == 0
        assert (rep.n_fine, rep.n_if1, rep.n_if2, rep.n_coarse, rep.n_uf1, rep.n_uf2) == (
            sum(len(g) for g in good.groups[0:3]), len(good.groups[3]), len(good.groups[4]),
            len(good.groups[5]), len(good.groups[1]), len(good.groups[2]))
        rng = np.random.default_rng(17)

        def corrupt(kinds):
            cl, cs, el = good.cell_label.copy(), good.cell_sublabel.copy(), good.edge_label.copy()
            if 1 in kinds:   # coarse cells relabelled Interface1
                cl[rng.choice(np.flatnonzero(good.cell_label == 3), 3, replace=False)] = 1
            if 2 in kinds:   # Interface1 cells relabelled Interface2
                cl[rng.choice(np.flatnonzero(good.cell_label == 1), 2, replace=False)] = 2
            if 3 in kinds:   # Interface2 cells relabelled coarse
                cl[rng.choice(np.flatnonzero(good.cell_label == 2), 4, replace=False)] = 3
            if 4 in kinds:   # underline layer 1 cells demoted
                cs[rng.choice(np.flatnonzero(good.cell_sublabel == 1), 2, replace=False)] = 0
            if 5 in kinds:   # edge labels changed
                e = rng.choice(nE, 5, replace=False)
                el[e] = (el[e] + 1) % 5
            return cl, cs, el

        for kinds in ([1], [2], [3], [4], [5], [1, 2, 3, 4, 5]):
            cl, cs, el = corrupt(kinds)
            want = _first_ids(rr.validate_labels(cl, cs, el))
            assert want, kinds
            # lists rebuilt from the labels, as the reference shim does
            ckey = np.where(cl == 0, cs, cl + 2)
            groups = [np.flatnonzero(ckey == k).astype(np.int32) for k in range(6)] + \
                     [np.flatnonzero(el == k).astype(np.int32) for k in range(5)]
            rep = ctx.validate_regions(RegionMap(cl, cs, el, width, groups, []))
            got = {k: rep.first[k] for k in range(1, 6) if rep.counts[k]}
            assert got == want, (kinds, got, want)
            assert not rep.ok() and rep.counts[0] == 0
    # value checks: a label outside the enum, a sublabel on a non-fine cell
    cl, cs, el = good.cell_label.copy(), good.cell_sublabel.copy(), good.edge_label.copy()
    cl[11] = 7
    cs[int(np.flatnonzero(good.cell_label == 3)[5])] = 1
    rep = ctx.validate_regions(RegionMap(cl, cs, el, width, good.groups, []))
    assert rep.counts[0] == 2 and rep.first[0] == min(11, int(np.flatnonzero(good.cell_label == 3)[5]))

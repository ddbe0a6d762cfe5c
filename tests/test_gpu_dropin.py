"""The C++ drop-in on the GPU: mswm::CudaStepper (the device-resident
Stepper, integrators.hpp:136-160) and mswm::CudaEvaluator (one C-ABI eval
per stage, integrators.hpp:68-73, inputs and outputs packed to the masked
read / write sets) against the unmodified reference; cost replication
(SchemeConfig::replication, operators.cpp:60)."""
import numpy as np
import pytest

from helpers import bits_equal
from paper_2106_07154_b200 import workloads as W
from paper_2106_07154_b200.api import (LTS3_MASKS, CudaContext, CudaEvaluator, Scheme, State,
                                       kMaskAll)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    from oracle import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    return oracle


@pytest.fixture(scope="module")
def sphere(ref):
    wl = W.small_sphere(5, seed=17, cap_deg=25.0)
    rm = ref.RefMesh.from_mesh(wl.mesh)
    rr = ref.RefRegions(rm, wl.fine_mask, wl.width)
    return wl, rm, rr


@pytest.mark.parametrize("per_call", [True, False])
def test_cuda_stepper_bitwise_reference_stepper(ref, sphere, per_call):
    """CudaStepper::step (state up/down per call) and ::advance (resident
    across steps) reproduce the reference Stepper with SerialEvaluator for
    every scheme, ledger included."""
    wl, rm, rr = sphere
    for scheme, dt in [(Scheme.LTS3, wl.dt), (Scheme.LTS2, wl.dt), (Scheme.RK4, wl.dt / wl.M),
                       (Scheme.SSPRK3, wl.dt / wl.M), (Scheme.SSPRK2, wl.dt / (2 * wl.M))]:
        serial = ref.RefEvaluator(rm, rr, wl.b, wl.f, wl.gravity)
        st = ref.CudaStepperRef(rm, rr, wl.b, wl.f, wl.gravity)
        h1, u1, t1, _ = serial.step(int(scheme), wl.h, wl.u, 0.0, dt, wl.M, 3)
        h2, u2, t2 = st.run(int(scheme), wl.h, wl.u, 0.0, dt, wl.M, 3, per_call=per_call)
        assert bits_equal(h1, h2) and bits_equal(u1, u2) and t1 == t2, scheme
        c1, e1, _ = serial.ledger()
        c2, e2 = st.ledger()
        assert np.array_equal(c1, c2) and np.array_equal(e1, e2), scheme


def test_cuda_stepper_errors_are_reference_exceptions(ref, sphere):
    """dt <= 0 and M < 1 raise the reference's ConfigError
    (integrators.cpp:413-421) through the C++ shim."""
    wl, rm, rr = sphere
    st = ref.CudaStepperRef(rm, rr, wl.b, wl.f, wl.gravity)
    for dt, M in [(0.0, 4), (wl.dt, 0)]:
        with pytest.raises(ref.OracleError) as ei:
            st.run(int(Scheme.LTS3), wl.h, wl.u, 0.0, dt, M, 1)
        assert ei.value.status == 1  # MSWM_E_CONFIG <- ConfigError


@pytest.mark.parametrize("replication", [2, 3])
def test_replication_results_unchanged_ledger_scaled(ref, sphere, replication):
    """Cost replication repeats the arithmetic: h, u bitwise those of
    replication 1 (and of the reference run with the same factor), every
    ledger count scaled by the factor, as the reference's tally
    (integrators.cpp:302-335)."""
    wl, rm, rr = sphere
    serial = ref.RefEvaluator(rm, rr, wl.b, wl.f, wl.gravity, replication=replication)
    h1, u1, _, _ = serial.step(int(Scheme.LTS3), wl.h, wl.u, 0.0, wl.dt, wl.M, 2)
    c1, e1, _ = serial.ledger()
    st = ref.CudaStepperRef(rm, rr, wl.b, wl.f, wl.gravity, replication=replication)
    h2, u2, _ = st.run(int(Scheme.LTS3), wl.h, wl.u, 0.0, wl.dt, wl.M, 2, per_call=False)
    c2, e2 = st.ledger()
    assert bits_equal(h1, h2) and bits_equal(u1, u2)
    assert np.array_equal(c1, c2) and np.array_equal(e1, e2)
    # the Python context: same results as replication 1, counts x factor
    ctx1 = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, fine_mask=wl.fine_mask)
    ctx1.make_regions(wl.fine_mask, wl.width)
    ctxr = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, fine_mask=wl.fine_mask)
    ctxr.make_regions(wl.fine_mask, wl.width)
    ctxr.set_replication(replication)
    for c in (ctx1, ctxr):
        c.upload(State(wl.h, wl.u, 0.0))
        c.advance(Scheme.LTS3, wl.dt, wl.M, 2)
    a, b = ctx1.download(), ctxr.download()
    assert bits_equal(a.h, b.h) and bits_equal(a.u, b.u) and bits_equal(a.h, h1)
    l1, lr = ctx1.ledger(), ctxr.ledger()
    assert np.array_equal(lr.edge_evals, replication * l1.edge_evals)
    assert np.array_equal(lr.cell_evals, replication * l1.cell_evals)


def test_replication_rejects_zero():
    from paper_2106_07154_b200.api import ConfigError
    wl = W.small_sphere(3, seed=1)
    ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity)
    with pytest.raises(ConfigError):
        ctx.set_replication(0)


def test_packed_eval_writes_only_the_mask(ref, sphere):
    """mswm_cuda_eval moves only the masked read set up and the outputs down
    (small masks): every masked entry bitwise the reference's
    shallow_water_tendencies, every other entry untouched (sentinel)."""
    wl, rm, rr = sphere
    serial = ref.RefEvaluator(rm, rr, wl.b, wl.f, wl.gravity)
    ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, fine_mask=wl.fine_mask)
    ctx.make_regions(wl.fine_mask, wl.width)
    rng = np.random.default_rng(5)
    h = wl.h + rng.normal(scale=0.1, size=wl.h.shape)
    u = wl.u + rng.normal(scale=1e-3, size=wl.u.shape)
    for mask in LTS3_MASKS + [kMaskAll, 1 << 3, 1 << 8]:
        dh_r = np.full(wl.mesh.n_cells, 7.25)
        du_r = np.full(wl.mesh.n_edges, -3.5)
        serial.eval(h, u, mask, dh_r, du_r)
        dh = np.full(wl.mesh.n_cells, 7.25)
        du = np.full(wl.mesh.n_edges, -3.5)
        CudaEvaluator(ctx).eval(h, u, mask, dh, du)
        assert bits_equal(dh, dh_r) and bits_equal(du, du_r), hex(mask)

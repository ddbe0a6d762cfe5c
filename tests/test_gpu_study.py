"""Device convergence study (study.py) against the reference's
convergence_study on its TC5 mountain case (harness.cpp:243-309, init_tc5
harness.cpp:35-72): errors, slopes and monotonicity flags equal."""
import numpy as np
import pytest

from paper_2106_07154_b200.api import CudaContext, Scheme, State
from paper_2106_07154_b200.study import convergence_study, l2_error

GRAVITY_TC5 = 9.80616  # TestCaseConfig::gravity (harness.hpp)


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,M", [(Scheme.LTS3, 2), (Scheme.RK4, 1), (Scheme.SSPRK3, 1)])
def test_convergence_study_equals_reference(ref_lib, scheme, M):
    rm = ref_lib.RefMesh.icosahedral(3)
    mesh = rm.as_mesh()
    h, u, b, f = ref_lib.ref_init_tc5(rm)
    fine = (b > 0.0).astype(np.uint8)  # the mountain's cells
    rr = ref_lib.RefRegions(rm, fine, 1)
    dts, duration = [1200.0, 600.0, 300.0], 3600.0
    want = ref_lib.ref_convergence_study(rm, rr, int(scheme), M, dts, duration)
    ctx = CudaContext(mesh, b, f, GRAVITY_TC5, fine_mask=fine)
    ctx.make_regions(fine, 1)
    got = convergence_study(ctx, State(h, u, 0.0), scheme, M, dts, duration)
    assert np.array_equal(np.asarray(got["err_h"]), want["err_h"])
    assert np.array_equal(np.asarray(got["err_u"]), want["err_u"])
    assert got["slope_h"] == want["slope_h"] and got["slope_u"] == want["slope_u"]
    assert (got["monotone_h"], got["monotone_u"]) == (want["monotone_h"], want["monotone_u"])
    if scheme == Scheme.LTS3:
        assert 2.0 < got["slope_h"] < 4.5  # third order in time (acceptance.cpp:120-145)


def test_fit_matches_reference_formula():
    """Least-squares slope of log(err) on log(dt) (harness.cpp:279-297)."""
    from paper_2106_07154_b200.study import _fit
    dts = [4.0, 2.0, 1.0]
    assert _fit(dts, [d ** 3 for d in dts]) == pytest.approx(3.0, abs=1e-12)
    assert _fit([1.0], [1.0]) == 0.0


def test_l2_error_norms():
    from paper_2106_07154_b200 import workloads as W
    wl = W.small_sphere(3, seed=2)
    a = State(wl.h, wl.u, 0.0)
    b = State(wl.h + 1.0, wl.u - 2.0, 0.0)
    rep = l2_error(wl.mesh, a, b)
    assert rep["l2_h"] == pytest.approx(np.sqrt(wl.mesh.n_cells))
    assert rep["l2_u"] == pytest.approx(2.0 * np.sqrt(wl.mesh.n_edges))
    assert rep["linf_h"] == 1.0 and rep["linf_u"] == 2.0

"""Parity at north_star's horizon on the BASELINE configurations (GPU).

north_star: "prognostic h and u within 1e-11 relative max-norm after 100
coarse steps" on the 10.5M-cell mesh.  The reference's CPU LTS3 takes minutes
per hundred C4 steps, so its results are committed as digests
(tests/golden/horizon_<cfg>.json, made by tests/make_horizon_digests.py from
oracle/_ref = the unmodified reference's Stepper::lts_step(3),
integrators.cpp:412-575).  Each test checks the input digest first (mesh
tables, h, u, b, f, fine mask, dt, M), then advances the device state through
the checkpoints and compares sha256 of h and u: bitwise equality, hence the
1e-11 bound.  On a mismatch the stored samples give the relative error.
"""
import hashlib
import json

import numpy as np
import pytest

from helpers import GOLDEN, workload
from paper_2106_07154_b200 import workloads as W
from paper_2106_07154_b200.api import CudaContext, Scheme, State

pytestmark = pytest.mark.gpu


def _load(cfg):
    p = GOLDEN / f"horizon_{cfg}.json"
    if not p.exists():
        pytest.skip(f"{p.name} not generated")
    rec = json.loads(p.read_text())
    if not rec.get("complete"):
        pytest.skip(f"{p.name} incomplete")
    return rec


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.float64).tobytes()).hexdigest()


def _input_digest(wl):
    h = hashlib.sha256()
    h.update(wl.mesh.digest().encode())
    for a in (wl.h, wl.u, wl.b, wl.f):
        h.update(np.ascontiguousarray(a, np.float64).tobytes())
    h.update(np.ascontiguousarray(wl.fine_mask, np.uint8).tobytes())
    h.update(np.array([wl.dt, wl.gravity, wl.M, wl.width], np.float64).tobytes())
    return h.hexdigest()


def _rel(a, ref_sample, stride):
    s = np.asarray(a)[::stride]
    r = np.asarray(ref_sample)
    return float(np.max(np.abs(s - r) / np.maximum(np.abs(r), 1e-300)))


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_lts3_horizon_bitwise_vs_reference(cfg):
    """C4: 100 coarse steps (north_star); C2: its 1000-step horizon; C1 100;
    C3 20; C5 1 -- h and u bitwise the reference at every checkpoint."""
    rec = _load(cfg)
    wl = workload(cfg)
    assert _input_digest(wl) == rec["input_sha256"], "workload or mesh builder changed"
    ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, order="regions", fine_mask=wl.fine_mask,
                      interface_width=wl.width)
    ctx.make_regions(wl.fine_mask, wl.width)
    ctx.upload(State(wl.h, wl.u, 0.0))
    st = State(np.zeros(wl.mesh.n_cells), np.zeros(wl.mesh.n_edges), 0.0)
    done = 0
    for cp in rec["checkpoints"]:
        ctx.advance(Scheme.LTS3, wl.dt, wl.M, cp["step"] - done)
        done = cp["step"]
        ctx.download(st)
        eh = _rel(st.h, cp["h_sample"], rec["sample_stride"])
        eu = _rel(st.u, cp["u_sample"], rec["sample_stride"])
        assert eh <= 1e-11 and eu <= 1e-11, (cfg, done, eh, eu)
        assert _sha(st.h) == cp["h_sha256"] and _sha(st.u) == cp["u_sha256"], (cfg, done, eh, eu)

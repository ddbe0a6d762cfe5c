"""Reference digests of the BASELINE configurations at north_star's horizon.

Runs the UNMODIFIED reference (oracle/_ref: Stepper::lts_step(3) with the
ThreadedEvaluator, bitwise equal to SerialEvaluator, acceptance.cpp:205-244)
from each configuration's seeded initial state and records, at checkpoint
steps, the sha256 of h and u (float64 bytes, original numbering) plus a
strided sample of both for error reporting.  The GPU tests
(tests/test_horizon.py) check the input digest first, then the device state
at every checkpoint against these digests: bitwise, hence within north_star's
1e-11 relative max-norm.

    python tests/make_horizon_digests.py c2 c3 c4      # here (62 GB host)
    python tests/make_horizon_digests.py c5            # on the GPU box (L11 needs ~100 GB)

Outputs tests/golden/horizon_<cfg>.json.
"""
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2106_07154_b200 import workloads as W  # noqa: E402

OUT = ROOT / "tests" / "golden"

# checkpoints (coarse LTS3 steps): north_star's 100 steps on C4, the configs'
# own horizons on C2 (1000) and, bounded by the reference's CPU time, C3/C5
CHECKPOINTS = {"c1": [1, 10, 100], "c2": [1, 10, 100, 1000], "c3": [1, 10, 20],
               "c4": [1, 10, 100], "c5": [1, 10]}
SAMPLE = 4099  # stride of the stored samples (prime: no alignment with the numbering)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, np.float64).tobytes()).hexdigest()


def input_digest(wl) -> str:
    h = hashlib.sha256()
    h.update(wl.mesh.digest().encode())
    for a in (wl.h, wl.u, wl.b, wl.f):
        h.update(np.ascontiguousarray(a, np.float64).tobytes())
    h.update(np.ascontiguousarray(wl.fine_mask, np.uint8).tobytes())
    h.update(np.array([wl.dt, wl.gravity, wl.M, wl.width], np.float64).tobytes())
    return h.hexdigest()


def sample(a: np.ndarray) -> list:
    return [float(x) for x in np.asarray(a)[::SAMPLE]]


def run(cfg: str, ranks: int):
    from oracle.oracle import RefEvaluator, RefMesh, RefRegions
    t0 = time.time()
    wl = W.CONFIGS[cfg]()
    rm = RefMesh.from_mesh(wl.mesh)
    rr = RefRegions(rm, wl.fine_mask, wl.width)
    ev = RefEvaluator(rm, rr, wl.b, wl.f, wl.gravity, nranks=ranks)
    print(f"{cfg}: {wl.mesh.n_cells} cells, set up in {time.time() - t0:.0f} s", flush=True)
    rec = {"config": cfg, "input_sha256": input_digest(wl), "mesh_sha256": wl.mesh.digest(),
           "M": wl.M, "dt": wl.dt, "scheme": "LTS3", "sample_stride": SAMPLE,
           "reference": f"oracle/_ref Stepper::lts_step(3), ThreadedEvaluator {ranks} ranks",
           "checkpoints": []}
    h, u, t, done = wl.h, wl.u, 0.0, 0
    for k in CHECKPOINTS[cfg]:
        t1 = time.time()
        h, u, t, _ = ev.step(4, h, u, t, wl.dt, wl.M, k - done)
        done = k
        rec["checkpoints"].append({"step": k, "h_sha256": sha(h), "u_sha256": sha(u),
                                   "h_sample": sample(h), "u_sample": sample(u),
                                   "h_absmax": float(np.max(np.abs(h))),
                                   "u_absmax": float(np.max(np.abs(u)))})
        print(f"{cfg}: step {k} ({time.time() - t1:.0f} s)", flush=True)
        (OUT / f"horizon_{cfg}.json").write_text(json.dumps(rec, indent=1))
    rec["complete"] = True
    (OUT / f"horizon_{cfg}.json").write_text(json.dumps(rec, indent=1))


def main():
    ranks = int(os.environ.get("REF_RANKS", str(len(os.sched_getaffinity(0)))))
    for cfg in sys.argv[1:]:
        run(cfg, ranks)


if __name__ == "__main__":
    main()

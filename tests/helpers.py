"""Shared test helpers."""
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def bits_equal(a, b) -> bool:
    """Bitwise equality of float64 arrays (NaN payloads and signed zeros included)."""
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.int64), b.view(np.int64))


def max_rel(a, b, floor=1e-300):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor))) if a.size else 0.0


def load_golden(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


def golden_mesh(name):
    """Rebuild the mesh a fixture was made on (digest-checked by the tests)."""
    from paper_2106_07154_b200.mesh import Mesh
    if name == "planar24":
        return Mesh.planar_hex(24, 24, 10e3)
    if name.startswith("sphereL"):
        return Mesh.icosahedral(int(name[len("sphereL"):]), 6371220.0)
    raise KeyError(name)


def workload(cfg: str):
    """A BASELINE configuration's workload, built once per test session for
    the full-size tests (the C4 / C5 meshes take minutes to build)."""
    return _workload(cfg)


def _build(cfg):
    from paper_2106_07154_b200 import workloads as W
    return W.CONFIGS[cfg]()


import functools  # noqa: E402

_workload = functools.lru_cache(maxsize=2)(_build)

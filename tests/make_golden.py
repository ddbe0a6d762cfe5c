"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run here (the reference sources are only in this container):
    python tests/make_golden.py
Each fixture holds the inputs (mesh table digest, h, u, b, f, fine mask)
and the reference's outputs: region labels and the 11 group lists,
tendencies and closure sets for the LTS3 masks and kMaskAll, the state
after a few LTS3 / RK4 / SSPRK3 steps, and the LTS3 ledger.
"""
import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle.oracle import RefEvaluator, RefMesh, RefRegions  # noqa: E402
from paper_2106_07154_b200 import workloads as W  # noqa: E402
from paper_2106_07154_b200.api import LTS3_MASKS, kMaskAll, Scheme  # noqa: E402
from paper_2106_07154_b200.mesh import Mesh  # noqa: E402

OUT = ROOT / "tests" / "golden"


def mesh_digest(mesh) -> str:
    h = hashlib.sha256()
    for name in sorted(mesh.tables):
        h.update(name.encode())
        h.update(np.ascontiguousarray(mesh.tables[name]).tobytes())
    return h.hexdigest()


def planar_small(seed=21):
    mesh = Mesh.planar_hex(24, 24, 10e3)
    rng = np.random.Generator(np.random.PCG64(seed))
    xy = mesh.cell_xyz
    c = np.array([0.4 * mesh.width, 0.55 * mesh.height])
    d = mesh.min_image(xy[:, :2] - c[None, :])
    r = np.hypot(d[:, 0], d[:, 1])
    h = 1000.0 + 10.0 * np.exp(-r * r / (2 * 50e3 ** 2)) + rng.uniform(-0.5, 0.5, mesh.n_cells)
    u = rng.normal(0, 0.5, mesh.n_edges)
    b = rng.uniform(0, 5, mesh.n_cells)
    f = 1e-4 + rng.uniform(-1e-6, 1e-6, mesh.n_vertices)
    fine = (r < 0.2 * mesh.width).astype(np.uint8)
    return "planar24", mesh, h, u, b, f, fine, 9.81, 50.0, 4


def sphere_small(level=3, seed=22):
    wl = W.small_sphere(level, seed=seed, cap_deg=35.0, M=3)
    return (f"sphereL{level}", wl.mesh, wl.h, wl.u, wl.b, wl.f, wl.fine_mask, wl.gravity,
            wl.dt, wl.M)


def make(case):
    name, mesh, h, u, b, f, fine, g, dt, M = case
    rm = RefMesh.from_mesh(mesh)
    rr = RefRegions(rm, fine, 1)
    ev = RefEvaluator(rm, rr, b, f, g)
    out = dict(digest=np.array(mesh_digest(mesh)), h=h, u=u, b=b, f=f, fine=fine,
               gravity=np.float64(g), dt=np.float64(dt), M=np.int64(M))
    cl, cs, el = rr.labels(mesh.n_cells, mesh.n_edges)
    out.update(cell_label=cl, cell_sub=cs, edge_label=el)
    for gi, ids in enumerate(rr.groups()):
        out[f"group{gi}"] = ids
    for mask in LTS3_MASKS + [kMaskAll]:
        dh = np.full(mesh.n_cells, np.nan)
        du = np.full(mesh.n_edges, np.nan)
        ev.eval(h, u, mask, dh, du)
        out[f"dh_{mask}"] = dh
        out[f"du_{mask}"] = du
        for kind in range(4):
            out[f"closure_{mask}_{kind}"] = np.sort(ev.closure(h, u, mask, kind))
    for scheme, n in [(Scheme.LTS3, 3), (Scheme.RK4, 2), (Scheme.SSPRK3, 2)]:
        ev2 = RefEvaluator(rm, rr, b, f, g)
        h2, u2, t2, _ = ev2.step(int(scheme), h, u, 0.0, dt if scheme == Scheme.LTS3 else dt / M,
                                 M, n)
        out[f"h_{scheme.name}"] = h2
        out[f"u_{scheme.name}"] = u2
        c, e, s = ev2.ledger()
        out[f"ledger_cell_{scheme.name}"] = c
        out[f"ledger_edge_{scheme.name}"] = e
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(name, mesh.n_cells, mesh.n_edges, (OUT / f"{name}.npz").stat().st_size, "bytes")


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    make(planar_small())
    make(sphere_small())

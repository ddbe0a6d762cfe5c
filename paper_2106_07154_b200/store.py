"""Binary mesh / workload store (replaces the reference's MSWM1 text container
for the device path, proj/src/mesh_io.cpp:13-25,85-148).

A store is a directory of raw ``.npy`` arrays plus ``header.json``:

* ``mesh/<table>.npy`` -- every ``mswm_mesh_desc`` table (mesh.hpp:31-68), the
  positions (cell / vertex / edge xyz) and the kite areas;
* ``fields/<name>.npy`` -- h, u, b, f, the fine mask and any extra per-element
  arrays (region labels, the cell locality order, ...);
* ``header.json`` -- sizes, domain, scalar workload parameters and the mesh
  digest, checked on load.

Loading memory-maps the arrays (``np.load(mmap_mode="r")``), so N processes
of one node reading the same store under ``/dev/shm`` share one copy in the
page cache: the multi-GPU setup builds the global mesh once (rank 0) and every
rank cuts its own piece from the shared maps (``dist.shard_from_store``)
instead of each rank rebuilding the global mesh.
"""
from __future__ import annotations

import json
import os
import shutil
from pathlib import Path

import numpy as np

from . import _lib
from .mesh import Mesh

FORMAT = "mswm-store-1"
_GEOM = ("cell_xyz", "vertex_xyz", "edge_xyz", "kite_area")
_FIELDS = ("h", "u", "b", "f", "fine_mask")


def _put(path: Path, a) -> None:
    a = np.ascontiguousarray(a)
    with open(path, "wb") as fh:
        np.save(fh, a, allow_pickle=False)


def save_mesh(root, mesh: Mesh) -> None:
    d = Path(root) / "mesh"
    d.mkdir(parents=True, exist_ok=True)
    for name, _p, dtype, _k in _lib.DESC_TABLES:
        _put(d / f"{name}.npy", np.asarray(mesh.tables[name], dtype))
    for name in _GEOM:
        a = getattr(mesh, name)
        if a is not None:
            _put(d / f"{name}.npy", np.asarray(a, np.float64))


def load_mesh(root, header: dict, mmap: bool = True) -> Mesh:
    d = Path(root) / "mesh"
    mode = "r" if mmap else None
    tables = {}
    for name, _p, dtype, _k in _lib.DESC_TABLES:
        a = np.load(d / f"{name}.npy", mmap_mode=mode, allow_pickle=False)
        if a.dtype != dtype:
            raise ValueError(f"store table {name}: dtype {a.dtype}, expected {np.dtype(dtype)}")
        tables[name] = a
    geo = {}
    for name in _GEOM:
        p = d / f"{name}.npy"
        geo[name] = np.load(p, mmap_mode=mode, allow_pickle=False) if p.exists() else None
    m = header["mesh"]
    mesh = Mesh(int(m["n_cells"]), int(m["n_edges"]), int(m["n_vertices"]), tables,
                geo["cell_xyz"], geo["vertex_xyz"], geo["edge_xyz"], geo["kite_area"],
                bool(m["spherical"]), float(m["radius"]), float(m["width"]), float(m["height"]))
    for name, arr in tables.items():
        exp = _lib.table_shape(dict((t[0], t[3]) for t in _lib.DESC_TABLES)[name], mesh.n_cells,
                               mesh.n_edges, mesh.n_vertices, mesh.n_ring, mesh.n_stencil)
        if tuple(arr.shape) != tuple(exp):
            raise ValueError(f"store table {name}: shape {arr.shape}, expected {exp}")
    return mesh


def save_workload(root, wl, extra: dict | None = None, digest: bool = True) -> Path:
    """Write ``wl`` (a workloads.Workload) and ``extra`` arrays to ``root``.
    The directory is written under a temporary name and renamed, so a reader
    never sees a partial store."""
    root = Path(root)
    tmp = root.with_name(root.name + f".tmp{os.getpid()}")
    if tmp.exists():
        shutil.rmtree(tmp)
    save_mesh(tmp, wl.mesh)
    fd = tmp / "fields"
    fd.mkdir(parents=True, exist_ok=True)
    for name in _FIELDS:
        _put(fd / f"{name}.npy", getattr(wl, name))
    for name, a in (extra or {}).items():
        _put(fd / f"{name}.npy", a)
    m = wl.mesh
    header = {
        "format": FORMAT,
        "name": wl.name,
        "mesh": {"n_cells": m.n_cells, "n_edges": m.n_edges, "n_vertices": m.n_vertices,
                 "spherical": bool(m.spherical), "radius": float(m.radius),
                 "width": float(m.width), "height": float(m.height),
                 "sha256": m.digest(geometry=False) if digest else None},
        "gravity": float(wl.gravity), "dt": float(wl.dt), "M": int(wl.M),
        "n_steps": int(wl.n_steps), "width": int(wl.width), "meta": wl.meta,
        "extra": sorted((extra or {}).keys()),
    }
    (tmp / "header.json").write_text(json.dumps(header, indent=1))
    if root.exists():
        shutil.rmtree(root)
    tmp.rename(root)
    return root


def load_workload(root, mmap: bool = True, verify: bool = False):
    """(Workload, extra arrays) from a store.  ``verify`` recomputes the mesh
    digest (reads every table once)."""
    from .workloads import Workload
    root = Path(root)
    header = json.loads((root / "header.json").read_text())
    if header.get("format") != FORMAT:
        raise ValueError(f"{root}: not an {FORMAT} store")
    mesh = load_mesh(root, header, mmap)
    if verify and header["mesh"]["sha256"] and mesh.digest(geometry=False) != header["mesh"]["sha256"]:
        raise ValueError(f"{root}: mesh digest mismatch")
    mode = "r" if mmap else None
    fd = root / "fields"
    f = {n: np.load(fd / f"{n}.npy", mmap_mode=mode, allow_pickle=False) for n in _FIELDS}
    extra = {n: np.load(fd / f"{n}.npy", mmap_mode=mode, allow_pickle=False)
             for n in header["extra"]}
    wl = Workload(header["name"], mesh, f["h"], f["u"], f["b"], f["f"], f["fine_mask"],
                  header["gravity"], header["dt"], header["M"], header["n_steps"],
                  header["width"], header["meta"])
    return wl, extra

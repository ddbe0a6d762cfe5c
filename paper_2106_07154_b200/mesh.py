"""VoronoiMesh tables on the host (proj/include/mswm/mesh.hpp:31-103).

A :class:`Mesh` is the input data contract of the drop-in boundary: the SoA
tables of ``mswm_mesh_desc`` as numpy arrays plus positions for host-side
setup (initial conditions, fine predicates).  Generators live in the native
host library (``csrc/meshgen.cpp``).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib


@dataclass
class Mesh:
    n_cells: int
    n_edges: int
    n_vertices: int
    tables: dict
    cell_xyz: np.ndarray
    vertex_xyz: np.ndarray
    edge_xyz: np.ndarray
    kite_area: np.ndarray | None
    spherical: bool
    radius: float = 1.0
    width: float = 0.0
    height: float = 0.0
    _owner: object = field(default=None, repr=False)

    def __getattr__(self, name):
        tables = self.__dict__.get("tables")
        if tables is not None and name in tables:
            return tables[name]
        raise AttributeError(name)

    # -- construction ------------------------------------------------------
    @classmethod
    def from_desc(cls, desc: _lib.MeshDesc, n_ring: int, n_stencil: int, geometry=None,
                  owner=None, spherical=True, radius=1.0, width=0.0, height=0.0) -> "Mesh":
        nC, nE, nV = desc.n_cells, desc.n_edges, desc.n_vertices
        tables = {}
        for name, _ptype, dtype, kind in _lib.DESC_TABLES:
            shape = _lib.table_shape(kind, nC, nE, nV, n_ring, n_stencil)
            tables[name] = _lib.view(getattr(desc, name), dtype, shape)
        cx = vx = ex = ka = None
        if geometry is not None:
            cx = _lib.view(geometry[0], np.float64, (nC, 3))
            vx = _lib.view(geometry[1], np.float64, (nV, 3))
            ex = _lib.view(geometry[2], np.float64, (nE, 3))
            ka = _lib.view(geometry[3], np.float64, (n_ring,)) if geometry[3] else None
        return cls(nC, nE, nV, tables, cx, vx, ex, ka, spherical, radius, width, height, owner)

    @classmethod
    def _from_host(cls, handle) -> "Mesh":
        lib = _lib.host()
        if not handle:
            raise RuntimeError("mesh generation failed: " + lib.mswm_host_last_error().decode())
        owner = _HostMesh(handle)
        sizes = _lib.MeshSizes()
        lib.mswm_mesh_get_sizes(handle, C.byref(sizes))
        desc = _lib.MeshDesc()
        lib.mswm_mesh_get_desc(handle, C.byref(desc))
        geo = [_lib.f64p() for _ in range(4)]
        lib.mswm_mesh_get_geometry(handle, *[C.byref(g) for g in geo])
        sph = C.c_int()
        r, w, h = C.c_double(), C.c_double(), C.c_double()
        lib.mswm_mesh_get_domain(handle, C.byref(sph), C.byref(r), C.byref(w), C.byref(h))
        return cls.from_desc(desc, sizes.n_ring, sizes.n_stencil, geo, owner, bool(sph.value),
                             r.value, w.value, h.value)

    @classmethod
    def icosahedral(cls, level: int, radius: float = 6371220.0) -> "Mesh":
        """build_voronoi_mesh(subdivide_icosahedron(level), radius) without the
        reference's level clamp (proj/src/mesh_build.cpp:369)."""
        return cls._from_host(_lib.host().mswm_mesh_icosahedral(level, radius))

    @classmethod
    def planar_hex(cls, nx: int, ny: int, dc: float) -> "Mesh":
        """Doubly periodic hexagonal mesh (nx*ny cells, centre spacing dc)."""
        return cls._from_host(_lib.host().mswm_mesh_planar_hex(nx, ny, dc))

    def locality_order(self) -> np.ndarray:
        """Hilbert-curve cell order for the device layout (host library)."""
        owner = self._owner
        if isinstance(owner, _HostMesh):
            out = np.zeros(self.n_cells, np.int32)
            _lib.host().mswm_mesh_locality_order(owner.handle, _lib.as_ptr(out, _lib.i32p))
            return out
        return hilbert_order_py(self)

    # -- boundary ----------------------------------------------------------
    def desc(self) -> _lib.MeshDesc:
        d = _lib.MeshDesc()
        d.n_cells, d.n_edges, d.n_vertices = self.n_cells, self.n_edges, self.n_vertices
        for name, ptype, dtype, _kind in _lib.DESC_TABLES:
            arr = self.tables[name]
            if not isinstance(arr, np.ndarray) or arr.dtype != dtype or not arr.flags.c_contiguous:
                raise ValueError(f"mesh table {name} must be a contiguous {np.dtype(dtype)} array")
            setattr(d, name, _lib.as_ptr(arr, ptype))
        return d

    def digest(self, geometry: bool = True) -> str:
        """sha256 of the hot-path tables (and positions / kite areas): equal
        digests = bitwise equal meshes, whichever builder made them."""
        import hashlib
        h = hashlib.sha256()
        for name in sorted(self.tables):
            h.update(name.encode())
            h.update(np.ascontiguousarray(self.tables[name]).tobytes())
        if geometry:
            for name in ("cell_xyz", "vertex_xyz", "edge_xyz", "kite_area"):
                a = getattr(self, name)
                if a is not None:
                    h.update(name.encode())
                    h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()

    @property
    def n_ring(self) -> int:
        return int(self.tables["cell_offset"][-1])

    @property
    def n_stencil(self) -> int:
        return int(self.tables["edge_edge_offset"][-1])

    def ring_size(self) -> np.ndarray:
        return np.diff(self.tables["cell_offset"])

    # -- geometry helpers (host setup only) --------------------------------
    def min_image(self, d: np.ndarray) -> np.ndarray:
        """Minimum-image difference vectors on the periodic plane."""
        out = np.array(d, dtype=np.float64, copy=True)
        out[..., 0] -= self.width * np.round(out[..., 0] / self.width)
        out[..., 1] -= self.height * np.round(out[..., 1] / self.height)
        return out

    def edge_normals(self) -> np.ndarray:
        """Unit normal per edge, from the higher-id cell toward the lower
        (mesh.hpp:98-101); tangent = position x normal (sphere) or z x n."""
        ec = self.tables["edge_cells"]
        if self.spherical:
            p = self.edge_xyz
            q = self.cell_xyz[ec[:, 0]]
            t = q - p * np.sum(p * q, axis=1, keepdims=True)
            return t / np.linalg.norm(t, axis=1, keepdims=True)
        d = self.min_image(self.cell_xyz[ec[:, 0]] - self.cell_xyz[ec[:, 1]])
        return d / np.linalg.norm(d, axis=1, keepdims=True)

    def total_mass(self, h: np.ndarray) -> float:
        """harness.cpp:99-105 (sequential sum in id order)."""
        return float(sum_in_order(self.tables["cell_area"] * h))


def hilbert_order_py(mesh: "Mesh") -> np.ndarray:
    """Coarse locality order for meshes not built by the host library:
    sort cells by a 3-D Morton key of their positions."""
    p = np.asarray(mesh.cell_xyz, np.float64)
    lo, hi = p.min(0), p.max(0)
    q = ((p - lo) / np.maximum(hi - lo, 1e-300) * 1023).astype(np.uint64)
    key = np.zeros(len(p), np.uint64)
    for b in range(10):
        for a in range(3):
            key |= ((q[:, a] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + a)
    return np.argsort(key, kind="stable").astype(np.int32)


def sum_in_order(x: np.ndarray) -> float:
    """Left-to-right double sum (np.sum uses pairwise summation)."""
    acc = 0.0
    for v in x.tolist():
        acc += v
    return acc


class _HostMesh:
    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        try:
            _lib.host().mswm_mesh_free(self.handle)
        except Exception:
            pass

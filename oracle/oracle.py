"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes drivers for
  * ``oracle/_ref/libmswm_ref.so`` -- the unmodified reference (proj/src/*.cpp)
    behind ``oracle/ref_shim.cpp``;
  * ``oracle/_build/libmswm_oracle.so`` -- our plain-C restatement
    (``oracle/mswm_oracle.c``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module.  The product (``paper_2106_07154_b200``) never
does.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2106_07154_b200 import _lib
from paper_2106_07154_b200.mesh import Mesh

HERE = Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libmswm_ref.so"          # the pure reference (no product link)
DROPIN_LIB = HERE / "_ref" / "libmswm_dropin.so"    # + mswm::CudaEvaluator (tests only)
ORACLE_LIB = HERE / "_build" / "libmswm_oracle.so"

vp = C.c_void_p
i32p, i64p, f64p, u8p = _lib.i32p, _lib.i64p, _lib.f64p, _lib.u8p
ERRLEN = 512

STATUS_NAMES = {0: "ok", 1: "config", 2: "usage", 3: "topology", 4: "dry_vertex", 5: "cuda",
                6: "nccl", 7: "nomem"}


class OracleError(RuntimeError):
    def __init__(self, status, msg, vertex=-1):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.vertex = vertex


_ref = None
_dropin = None
_orc = None


def ref_available() -> bool:
    return REF_LIB.exists()


def dropin() -> C.CDLL:
    """libmswm_dropin.so: the C++ drop-in over the product's C ABI (tests only;
    loading it maps libmswm_cuda.so)."""
    global _dropin
    if _dropin is None:
        ref()
        if not DROPIN_LIB.exists():
            raise RuntimeError(f"{DROPIN_LIB} not built (make -C oracle ref)")
        lib = C.CDLL(str(DROPIN_LIB))
        lib.ref_cuda_eval_create.restype = vp
        lib.ref_cuda_eval_create.argtypes = [vp, vp, f64p, f64p, C.c_double, C.c_int, C.c_char_p,
                                             C.c_int]
        lib.ref_cuda_stepper_create.restype = vp
        lib.ref_cuda_stepper_create.argtypes = [vp, vp, f64p, f64p, C.c_double, C.c_int, C.c_int,
                                                C.c_char_p, C.c_int]
        lib.ref_cuda_stepper_free.restype = None
        lib.ref_cuda_stepper_free.argtypes = [vp]
        lib.ref_cuda_stepper_run.restype = C.c_int
        lib.ref_cuda_stepper_run.argtypes = [vp, C.c_int, f64p, f64p, f64p, C.c_double, C.c_int,
                                             C.c_int64, C.c_int, C.c_char_p, C.c_int,
                                             C.POINTER(C.c_int)]
        lib.ref_cuda_stepper_ledger.restype = None
        lib.ref_cuda_stepper_ledger.argtypes = [vp, i64p, i64p]
        _dropin = lib
    return _dropin


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            raise RuntimeError(f"{REF_LIB} not built (make -C oracle ref)")
        lib = C.CDLL(str(REF_LIB))
        E = [C.c_char_p, C.c_int]
        sig = {
            "ref_mesh_icosahedral": (vp, [C.c_int, C.c_double] + E),
            "ref_mesh_icosphere": (vp, [C.c_int, C.c_int, C.c_double] + E),
            "ref_mesh_from_desc": (vp, [C.POINTER(_lib.MeshDesc), f64p, f64p, f64p, f64p]),
            "ref_mesh_free": (None, [vp]),
            "ref_mesh_sizes": (None, [vp, i64p]),
            "ref_mesh_desc": (None, [vp, C.POINTER(_lib.MeshDesc)]),
            "ref_mesh_geometry": (None, [vp] + [C.POINTER(f64p)] * 4),
            "ref_mesh_rederive": (C.c_int, [vp] + E),
            "ref_mesh_validate": (C.c_int, [vp] + E),
            "ref_total_mass": (C.c_double, [vp, f64p]),
            "ref_total_energy": (C.c_double, [vp, f64p, f64p, f64p, C.c_double]),
            "ref_courant": (C.c_int, [vp, vp, f64p, C.c_double, C.c_int, f64p, C.c_char_p,
                                      C.c_int]),
            "ref_regions_make": (vp, [vp, u8p, C.c_int] + E + [C.POINTER(C.c_int)]),
            "ref_regions_free": (None, [vp]),
            "ref_regions_labels": (None, [vp, u8p, u8p, u8p]),
            "ref_regions_group": (C.c_int64, [vp, C.c_int, i32p]),
            "ref_regions_validate": (C.c_int, [vp, vp]),
            "ref_regions_validate_labels": (C.c_int, [vp, vp, u8p, u8p, u8p, C.c_char_p, C.c_int]),
            "ref_eval_create": (vp, [vp, vp, f64p, f64p, C.c_double, C.c_int, C.c_uint64, C.c_int] + E),
            "ref_eval_free": (None, [vp]),
            "ref_eval": (C.c_int, [vp, f64p, f64p, C.c_uint, f64p, f64p] + E
                         + [C.POINTER(C.c_int)]),
            "ref_closure": (C.c_int, [vp, f64p, f64p, C.c_uint, C.c_int, i32p, i64p] + E),
            "ref_stepper_create": (vp, [vp]),
            "ref_stepper_free": (None, [vp]),
            "ref_step": (C.c_int, [vp, C.c_int, f64p, f64p, f64p, C.c_double, C.c_int,
                                   C.c_int64] + E + [C.POINTER(C.c_int), f64p]),
            "ref_ledger": (None, [vp, i64p, i64p, i64p]),
            "ref_lts_coeffs": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, f64p] + E),
            "ref_init_tc5": (C.c_int, [vp, f64p, f64p, f64p, f64p] + E),
            "ref_convergence_study": (C.c_int, [vp, vp, C.c_int, C.c_int, f64p, C.c_int,
                                                C.c_double, f64p] + E),
            "ref_partition": (C.c_int, [vp, vp, C.c_int, C.c_uint64, i32p] + E),
            "ref_block_plan": (vp, [vp, vp, i32p, C.c_int] + E),
            "ref_block_plan_free": (None, [vp]),
            "ref_block_plan_list": (C.c_int64, [vp, C.c_int, C.c_int, i32p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _ref = lib
    return _ref


def _err():
    return C.create_string_buffer(ERRLEN)


def _check(rc, buf, vertex=-1):
    if rc != 0:
        raise OracleError(rc, buf.value.decode(errors="replace"), vertex)


def _p(a, t):
    return a.ctypes.data_as(t)


# --------------------------------------------------------------------------
# reference meshes

class RefMesh:
    """A reference VoronoiMesh held by the shim."""

    def __init__(self, handle):
        if not handle:
            raise RuntimeError("reference mesh construction failed")
        self.handle = handle

    def __del__(self):
        if getattr(self, "handle", None):
            ref().ref_mesh_free(self.handle)
            self.handle = None

    @classmethod
    def icosahedral(cls, level, radius=6371220.0):
        buf = _err()
        h = ref().ref_mesh_icosahedral(level, radius, buf, ERRLEN)
        if not h:
            raise OracleError(1, buf.value.decode())
        return cls(h)

    @classmethod
    def icosphere(cls, level, lloyd, radius=6371220.0):
        buf = _err()
        h = ref().ref_mesh_icosphere(level, lloyd, radius, buf, ERRLEN)
        if not h:
            raise OracleError(1, buf.value.decode())
        return cls(h)

    @classmethod
    def from_mesh(cls, mesh: Mesh):
        d = mesh.desc()
        geo = [mesh.cell_xyz, mesh.vertex_xyz, mesh.edge_xyz, mesh.kite_area]
        ptrs = [(_p(np.ascontiguousarray(g), f64p) if g is not None else None) for g in geo]
        obj = cls(ref().ref_mesh_from_desc(C.byref(d), *ptrs))
        obj._keep = mesh
        return obj

    def as_mesh(self) -> Mesh:
        sizes = np.zeros(5, np.int64)
        ref().ref_mesh_sizes(self.handle, _p(sizes, i64p))
        d = _lib.MeshDesc()
        ref().ref_mesh_desc(self.handle, C.byref(d))
        geo = [f64p() for _ in range(4)]
        ref().ref_mesh_geometry(self.handle, *[C.byref(g) for g in geo])
        if not geo[3]:
            geo[3] = None
        return Mesh.from_desc(d, int(sizes[3]), int(sizes[4]), geo, owner=self)

    def rederive(self):
        buf = _err()
        _check(ref().ref_mesh_rederive(self.handle, buf, ERRLEN), buf)

    def validate(self):
        buf = _err()
        _check(ref().ref_mesh_validate(self.handle, buf, ERRLEN), buf)

    def total_mass(self, h):
        h = np.ascontiguousarray(h, np.float64)
        return ref().ref_total_mass(self.handle, _p(h, f64p))

    def total_energy(self, h, u, b, gravity):
        """harness.cpp:107-123 (the reference itself)."""
        return ref().ref_total_energy(self.handle, _p(np.ascontiguousarray(h, np.float64), f64p),
                                      _p(np.ascontiguousarray(u, np.float64), f64p),
                                      _p(np.ascontiguousarray(b, np.float64), f64p), gravity)

    def courant(self, regions, u, dt, M):
        """integrators.cpp:632-659 (the reference itself); regions may be None."""
        out = np.zeros(2)
        buf = _err()
        _check(ref().ref_courant(self.handle, regions.handle if regions is not None else None,
                                 _p(np.ascontiguousarray(u, np.float64), f64p), dt, M,
                                 _p(out, f64p), buf, ERRLEN), buf)
        return float(out[0]), float(out[1])


class RefRegions:
    def __init__(self, mesh: RefMesh, fine_mask, width=1):
        fm = np.ascontiguousarray(fine_mask, np.uint8)
        buf = _err()
        nw = C.c_int(0)
        self.handle = ref().ref_regions_make(mesh.handle, _p(fm, u8p), width, buf, ERRLEN,
                                             C.byref(nw))
        if not self.handle:
            raise OracleError(1, buf.value.decode())
        self.mesh = mesh
        self.n_warnings = nw.value

    def __del__(self):
        if getattr(self, "handle", None):
            ref().ref_regions_free(self.handle)
            self.handle = None

    def labels(self, nC, nE):
        cl = np.zeros(nC, np.uint8)
        cs = np.zeros(nC, np.uint8)
        el = np.zeros(nE, np.uint8)
        ref().ref_regions_labels(self.handle, _p(cl, u8p), _p(cs, u8p), _p(el, u8p))
        return cl, cs, el

    def group(self, g):
        n = ref().ref_regions_group(self.handle, g, None)
        ids = np.zeros(n, np.int32)
        ref().ref_regions_group(self.handle, g, _p(ids, i32p))
        return ids

    def groups(self):
        return [self.group(g) for g in range(11)]

    def validate(self):
        return ref().ref_regions_validate(self.mesh.handle, self.handle)

    def validate_labels(self, cell_label, cell_sub, edge_label):
        """validate_regions on these labels (lists rebuilt from them): its messages."""
        cl = np.ascontiguousarray(cell_label, np.uint8)
        cs = np.ascontiguousarray(cell_sub, np.uint8)
        el = np.ascontiguousarray(edge_label, np.uint8)
        buf = C.create_string_buffer(1 << 16)
        n = ref().ref_regions_validate_labels(self.mesh.handle, self.handle, _p(cl, u8p),
                                              _p(cs, u8p), _p(el, u8p), buf, len(buf))
        msgs = [x for x in buf.value.decode().split("\n") if x]
        assert n == len(msgs) or len(buf.value) >= len(buf) - 2
        return msgs


class RefEvaluator:
    """SerialEvaluator (nranks=0) or ThreadedEvaluator (nranks>=1)."""

    def __init__(self, mesh: RefMesh, regions: RefRegions | None, b, f, gravity, nranks=0,
                 seed=12345, replication=1):
        self.b = np.ascontiguousarray(b, np.float64)
        self.f = np.ascontiguousarray(f, np.float64)
        buf = _err()
        self.handle = ref().ref_eval_create(mesh.handle, regions.handle if regions else None,
                                            _p(self.b, f64p), _p(self.f, f64p), gravity, nranks,
                                            seed, replication, buf, ERRLEN)
        if not self.handle:
            raise OracleError(1, buf.value.decode())
        self.mesh, self.regions = mesh, regions
        self.stepper = None

    @classmethod
    def cuda(cls, mesh: RefMesh, regions: RefRegions | None, b, f, gravity, device=0):
        """The reference's evaluator slot filled with mswm::CudaEvaluator
        (oracle/drop_in_evaluator.hpp) -- the C++ drop-in over the C ABI."""
        obj = cls.__new__(cls)
        obj.b = np.ascontiguousarray(b, np.float64)
        obj.f = np.ascontiguousarray(f, np.float64)
        buf = _err()
        obj.handle = dropin().ref_cuda_eval_create(mesh.handle, regions.handle if regions else None,
                                                _p(obj.b, f64p), _p(obj.f, f64p), gravity, device,
                                                buf, ERRLEN)
        if not obj.handle:
            raise OracleError(5, buf.value.decode())
        obj.mesh, obj.regions, obj.stepper = mesh, regions, None
        return obj

    def __del__(self):
        if getattr(self, "stepper", None):
            ref().ref_stepper_free(self.stepper)
            self.stepper = None
        if getattr(self, "handle", None):
            ref().ref_eval_free(self.handle)
            self.handle = None

    def eval(self, h, u, mask, dh, du):
        buf = _err()
        dv = C.c_int(-1)
        rc = ref().ref_eval(self.handle, _p(np.ascontiguousarray(h), f64p),
                            _p(np.ascontiguousarray(u), f64p), mask, _p(dh, f64p), _p(du, f64p),
                            buf, ERRLEN, C.byref(dv))
        _check(rc, buf, dv.value)

    def closure(self, h, u, mask, kind):
        n = C.c_int64(0)
        buf = _err()
        h = np.ascontiguousarray(h)
        u = np.ascontiguousarray(u)
        _check(ref().ref_closure(self.handle, _p(h, f64p), _p(u, f64p), mask, kind, None,
                                 C.byref(n), buf, ERRLEN), buf)
        ids = np.zeros(n.value, np.int32)
        _check(ref().ref_closure(self.handle, _p(h, f64p), _p(u, f64p), mask, kind,
                                 _p(ids, i32p), C.byref(n), buf, ERRLEN), buf)
        return ids

    def step(self, scheme, h, u, time, dt, M, n_steps):
        """Stepper::step n times on copies; returns (h, u, time, seconds)."""
        if self.stepper is None:
            self.stepper = ref().ref_stepper_create(self.handle)
        h = np.array(h, np.float64, copy=True)
        u = np.array(u, np.float64, copy=True)
        t = C.c_double(time)
        secs = C.c_double(0)
        dv = C.c_int(-1)
        buf = _err()
        rc = ref().ref_step(self.stepper, scheme, _p(h, f64p), _p(u, f64p), C.byref(t), dt, M,
                            n_steps, buf, ERRLEN, C.byref(dv), C.byref(secs))
        _check(rc, buf, dv.value)
        return h, u, t.value, secs.value

    def ledger(self):
        if self.stepper is None:
            self.stepper = ref().ref_stepper_create(self.handle)
        c = np.zeros(16, np.int64)
        e = np.zeros(16, np.int64)
        s = C.c_int64(0)
        ref().ref_ledger(self.stepper, _p(c, i64p), _p(e, i64p), C.byref(s))
        return c.reshape(4, 4), e.reshape(4, 4), s.value


class CudaStepperRef:
    """mswm::CudaStepper (oracle/drop_in_evaluator.hpp), the C++
    device-resident Stepper over the C ABI, on a reference mesh / map."""

    def __init__(self, mesh: RefMesh, regions: RefRegions | None, b, f, gravity, replication=1,
                 device=0):
        self.b = np.ascontiguousarray(b, np.float64)
        self.f = np.ascontiguousarray(f, np.float64)
        buf = _err()
        self.handle = dropin().ref_cuda_stepper_create(
            mesh.handle, regions.handle if regions else None, _p(self.b, f64p), _p(self.f, f64p),
            gravity, replication, device, buf, ERRLEN)
        if not self.handle:
            raise OracleError(5, buf.value.decode())
        self.mesh, self.regions = mesh, regions

    def __del__(self):
        if getattr(self, "handle", None):
            dropin().ref_cuda_stepper_free(self.handle)
            self.handle = None

    def run(self, scheme, h, u, time, dt, M, n_steps, per_call=True):
        h = np.array(h, np.float64, copy=True)
        u = np.array(u, np.float64, copy=True)
        t = C.c_double(time)
        dv = C.c_int(-1)
        buf = _err()
        rc = dropin().ref_cuda_stepper_run(self.handle, scheme, _p(h, f64p), _p(u, f64p),
                                           C.byref(t), dt, M, n_steps, int(per_call), buf, ERRLEN,
                                           C.byref(dv))
        _check(rc, buf, dv.value)
        return h, u, t.value

    def ledger(self):
        c = np.zeros(16, np.int64)
        e = np.zeros(16, np.int64)
        dropin().ref_cuda_stepper_ledger(self.handle, _p(c, i64p), _p(e, i64p))
        return c.reshape(4, 4), e.reshape(4, 4)


def ref_init_tc5(mesh: RefMesh):
    """The reference's TC5 initial state (harness.cpp:35-72): h, u, b, f."""
    m = mesh.as_mesh()
    h, u = np.zeros(m.n_cells), np.zeros(m.n_edges)
    b, f = np.zeros(m.n_cells), np.zeros(m.n_vertices)
    buf = _err()
    _check(ref().ref_init_tc5(mesh.handle, _p(h, f64p), _p(u, f64p), _p(b, f64p), _p(f, f64p),
                              buf, ERRLEN), buf)
    return h, u, b, f


def ref_convergence_study(mesh: RefMesh, regions: RefRegions | None, scheme, M, dts, duration):
    """The reference's convergence_study on TC5 (harness.cpp:243-309)."""
    dts = np.ascontiguousarray(dts, np.float64)
    n = len(dts)
    out = np.zeros(2 * n + 4)
    buf = _err()
    _check(ref().ref_convergence_study(mesh.handle, regions.handle if regions else None,
                                       int(scheme), int(M), _p(dts, f64p), n, float(duration),
                                       _p(out, f64p), buf, ERRLEN), buf)
    return {"err_h": out[:n], "err_u": out[n:2 * n], "slope_h": out[2 * n],
            "slope_u": out[2 * n + 1], "monotone_h": bool(out[2 * n + 2]),
            "monotone_u": bool(out[2 * n + 3])}


def ref_lts_coeffs(order, stage, k, M):
    out = np.zeros(3)
    buf = _err()
    _check(ref().ref_lts_coeffs(order, stage, k, M, _p(out, f64p), buf, ERRLEN), buf)
    return out


def ref_partition(mesh: RefMesh, regions: RefRegions | None, nparts, seed=12345):
    n = mesh.as_mesh().n_cells
    labels = np.zeros(n, np.int32)
    buf = _err()
    _check(ref().ref_partition(mesh.handle, regions.handle if regions else None, nparts, seed,
                               _p(labels, i32p), buf, ERRLEN), buf)
    return labels


def ref_block_plan(mesh: RefMesh, regions: RefRegions, labels, nranks):
    labels = np.ascontiguousarray(labels, np.int32)
    buf = _err()
    h = ref().ref_block_plan(mesh.handle, regions.handle, _p(labels, i32p), nranks, buf, ERRLEN)
    if not h:
        raise OracleError(1, buf.value.decode())
    out = []
    try:
        for b in range(3 * nranks):
            lists = []
            for which in range(4):
                n = ref().ref_block_plan_list(h, b, which, None)
                ids = np.zeros(n, np.int32)
                ref().ref_block_plan_list(h, b, which, _p(ids, i32p))
                lists.append(ids)
            out.append(lists)
    finally:
        ref().ref_block_plan_free(h)
    return out


# --------------------------------------------------------------------------
# the plain-C restatement (oracle/mswm_oracle.c)

def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not ORACLE_LIB.exists():
            raise RuntimeError(f"{ORACLE_LIB} not built (make -C oracle restatement)")
        lib = C.CDLL(str(ORACLE_LIB))
        sig = {
            "orc_create": (vp, [C.POINTER(_lib.MeshDesc), f64p, f64p, C.c_double]),
            "orc_destroy": (None, [vp]),
            "orc_tendencies": (C.c_int, [vp, f64p, f64p, i32p, C.c_int64, i32p, C.c_int64, f64p,
                                         f64p]),
            "orc_last_closure": (C.c_int64, [vp, C.c_int, i32p]),
            "orc_dry_vertex": (C.c_int, [vp]),
            "orc_set_regions": (C.c_int, [vp, u8p, C.c_int, C.POINTER(C.c_int)]),
            "orc_get_labels": (None, [vp, u8p, u8p, u8p]),
            "orc_get_group": (C.c_int64, [vp, C.c_int, i32p]),
            "orc_eval": (C.c_int, [vp, f64p, f64p, C.c_uint, f64p, f64p]),
            "orc_lts_coeffs": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, f64p]),
            "orc_step": (C.c_int, [vp, C.c_int, f64p, f64p, f64p, C.c_double, C.c_int,
                                   C.c_int64]),
            "orc_ledger": (None, [vp, i64p, i64p, i64p]),
            "orc_total_mass": (C.c_double, [vp, f64p]),
            "orc_total_energy": (C.c_double, [vp, f64p, f64p]),
            "orc_courant": (C.c_int, [vp, f64p, C.c_double, C.c_int, f64p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _orc = lib
    return _orc


class Oracle:
    """CPU restatement of evaluator + regions + stepper on one mesh."""

    def __init__(self, mesh: Mesh, b, f, gravity):
        self.mesh = mesh
        self._desc = mesh.desc()
        self.b = np.ascontiguousarray(b, np.float64)
        self.f = np.ascontiguousarray(f, np.float64)
        self.handle = orc().orc_create(C.byref(self._desc), _p(self.b, f64p), _p(self.f, f64p),
                                       gravity)

    def __del__(self):
        if getattr(self, "handle", None):
            orc().orc_destroy(self.handle)
            self.handle = None

    def _rc(self, rc):
        if rc != 0:
            v = orc().orc_dry_vertex(self.handle) if rc == 4 else -1
            raise OracleError(rc, "oracle restatement", v)

    def set_regions(self, fine_mask, width=1):
        fm = np.ascontiguousarray(fine_mask, np.uint8)
        w = C.c_int(0)
        self._rc(orc().orc_set_regions(self.handle, _p(fm, u8p), width, C.byref(w)))
        return w.value

    def labels(self):
        m = self.mesh
        cl = np.zeros(m.n_cells, np.uint8)
        cs = np.zeros(m.n_cells, np.uint8)
        el = np.zeros(m.n_edges, np.uint8)
        orc().orc_get_labels(self.handle, _p(cl, u8p), _p(cs, u8p), _p(el, u8p))
        return cl, cs, el

    def group(self, g):
        n = orc().orc_get_group(self.handle, g, None)
        ids = np.zeros(n, np.int32)
        orc().orc_get_group(self.handle, g, _p(ids, i32p))
        return ids

    def groups(self):
        return [self.group(g) for g in range(11)]

    def eval(self, h, u, mask, dh, du):
        self._rc(orc().orc_eval(self.handle, _p(np.ascontiguousarray(h), f64p),
                                _p(np.ascontiguousarray(u), f64p), mask, _p(dh, f64p),
                                _p(du, f64p)))

    def tendencies(self, h, u, cells, edges, dh, du):
        cells = np.ascontiguousarray(cells, np.int32)
        edges = np.ascontiguousarray(edges, np.int32)
        self._rc(orc().orc_tendencies(self.handle, _p(np.ascontiguousarray(h), f64p),
                                      _p(np.ascontiguousarray(u), f64p), _p(cells, i32p),
                                      len(cells), _p(edges, i32p), len(edges), _p(dh, f64p),
                                      _p(du, f64p)))

    def last_closure(self, kind):
        n = orc().orc_last_closure(self.handle, kind, None)
        ids = np.zeros(n, np.int32)
        orc().orc_last_closure(self.handle, kind, _p(ids, i32p))
        return ids

    def step(self, scheme, h, u, time, dt, M, n_steps):
        h = np.array(h, np.float64, copy=True)
        u = np.array(u, np.float64, copy=True)
        t = C.c_double(time)
        self._rc(orc().orc_step(self.handle, scheme, _p(h, f64p), _p(u, f64p), C.byref(t), dt, M,
                                n_steps))
        return h, u, t.value

    def total_mass(self, h):
        return orc().orc_total_mass(self.handle, _p(np.ascontiguousarray(h, np.float64), f64p))

    def total_energy(self, h, u):
        return orc().orc_total_energy(self.handle, _p(np.ascontiguousarray(h, np.float64), f64p),
                                      _p(np.ascontiguousarray(u, np.float64), f64p))

    def courant(self, u, dt, M):
        out = np.zeros(2)
        self._rc(orc().orc_courant(self.handle, _p(np.ascontiguousarray(u, np.float64), f64p), dt,
                                   M, _p(out, f64p)))
        return float(out[0]), float(out[1])

    def ledger(self):
        c = np.zeros(16, np.int64)
        e = np.zeros(16, np.int64)
        s = C.c_int64(0)
        orc().orc_ledger(self.handle, _p(c, i64p), _p(e, i64p), C.byref(s))
        return c.reshape(4, 4), e.reshape(4, 4), s.value


def orc_lts_coeffs(order, stage, k, M):
    out = np.zeros(3)
    rc = orc().orc_lts_coeffs(order, stage, k, M, _p(out, f64p))
    if rc:
        raise OracleError(rc, "lts coeffs")
    return out

"""Host-side mirror of the reference interface for the LTS3 hot path.

Names, argument meanings and error behaviour follow the reference C++ API
(proj/include/mswm/{errors,integrators,regions,ledger}.hpp) so the parity
tests read like the reference's own tests.  Every call goes through the
C ABI of ``libmswm_cuda.so`` (include/mswm_cuda.h); there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .mesh import Mesh

# --------------------------------------------------------------------------
# errors (errors.hpp:9-49)


class Error(RuntimeError):
    pass


class ConfigError(Error):
    pass


class UsageError(Error):
    pass


class TopologyError(Error):
    pass


class DryVertexError(Error):
    """errors.hpp:45-49; ``step`` is the 1-based step of the advance() batch
    it happened in (harness.cpp:183-190), 0 for an eval call."""
    def __init__(self, msg, vertex, step=0):
        super().__init__(msg)
        self.vertex = vertex
        self.step = step


class CudaError(Error):
    pass


_STATUS = {1: ConfigError, 2: UsageError, 3: TopologyError, 5: CudaError, 6: CudaError,
           7: CudaError}


def _raise(rc: int, msg: str, vertex: int = -1, step: int = 0):
    if rc == 0:
        return
    if rc == 4:
        raise DryVertexError(msg, vertex, step)
    raise _STATUS.get(rc, Error)(msg)


# --------------------------------------------------------------------------
# GroupBit (integrators.hpp:43-61), Scheme (:26), regions enums (regions.hpp:12-21)

class GroupBit(enum.IntFlag):
    kCellsFinePlain = 1 << 0
    kCellsUF1 = 1 << 1
    kCellsUF2 = 1 << 2
    kCellsIf1 = 1 << 3
    kCellsIf2 = 1 << 4
    kCellsCoarse = 1 << 5
    kEdgesFinePlain = 1 << 6
    kEdgesUFine = 1 << 7
    kEdgesIf1 = 1 << 8
    kEdgesIf2 = 1 << 9
    kEdgesCoarse = 1 << 10


kCellsAll = 0x3F
kEdgesAll = 0x7C0
kMaskAll = 0x7FF

# the four LTS3 masks of Stepper::lts_step (integrators.cpp:452-461)
MASK_COARSE_ONLY = GroupBit.kCellsCoarse | GroupBit.kEdgesCoarse
MASK_IF_COARSE = (GroupBit.kCellsIf1 | GroupBit.kCellsIf2 | GroupBit.kCellsCoarse
                  | GroupBit.kEdgesIf1 | GroupBit.kEdgesIf2 | GroupBit.kEdgesCoarse)
MASK_STEP1 = MASK_IF_COARSE | GroupBit.kCellsUF1 | GroupBit.kCellsUF2 | GroupBit.kEdgesUFine
MASK_SUB = (GroupBit.kCellsFinePlain | GroupBit.kCellsUF1 | GroupBit.kCellsUF2
            | GroupBit.kCellsIf1 | GroupBit.kCellsIf2 | GroupBit.kEdgesFinePlain
            | GroupBit.kEdgesUFine | GroupBit.kEdgesIf1 | GroupBit.kEdgesIf2)
LTS3_MASKS = [int(MASK_STEP1), int(MASK_IF_COARSE), int(MASK_SUB), int(MASK_COARSE_ONLY)]


class Scheme(enum.IntEnum):
    SSPRK2 = 0
    SSPRK3 = 1
    RK4 = 2
    LTS2 = 3
    LTS3 = 4


def parse_scheme(name: str) -> Scheme:
    """integrators.cpp:250-258"""
    try:
        return {"ssprk2": Scheme.SSPRK2, "ssprk3": Scheme.SSPRK3, "rk4": Scheme.RK4,
                "lts2": Scheme.LTS2, "lts3": Scheme.LTS3}[name]
    except KeyError:
        raise ConfigError(f"unknown scheme '{name}' (expected ssprk2, ssprk3, rk4, lts2 or lts3)")


class CellRegion(enum.IntEnum):
    Fine = 0
    Interface1 = 1
    Interface2 = 2
    Coarse = 3


class CellSub(enum.IntEnum):
    None_ = 0
    UnderlineF1 = 1
    UnderlineF2 = 2


class EdgeRegion(enum.IntEnum):
    FineEdge = 0
    UnderlineFineEdge = 1
    Interface1Edge = 2
    Interface2Edge = 3
    CoarseEdge = 4


GROUP_NAMES = ["cells_fine_plain", "cells_uf1", "cells_uf2", "cells_if1", "cells_if2",
               "cells_coarse", "edges_fine", "edges_ufine", "edges_if1", "edges_if2",
               "edges_coarse"]

CLOSURE_FLUX, CLOSURE_QT, CLOSURE_K, CLOSURE_PV = range(4)


@dataclass
class State:
    """integrators.hpp:18-24"""
    h: np.ndarray
    u: np.ndarray
    time: float = 0.0


@dataclass
class SchemeConfig:
    """integrators.hpp:33-39"""
    scheme: Scheme = Scheme.SSPRK3
    dt: float = 0.0
    substeps: int = 1
    gravity: float = 9.80616
    replication: int = 1


@dataclass
class WorkLedger:
    """ledger.hpp:25-60 (wall-time fields are kept by the caller)."""
    cell_evals: np.ndarray
    edge_evals: np.ndarray
    steps_taken: int

    def total_cell_evals(self) -> int:
        return int(self.cell_evals.sum())

    def total_edge_evals(self) -> int:
        return int(self.edge_evals.sum())

    def total_evals(self) -> int:
        return self.total_cell_evals() + self.total_edge_evals()


@dataclass
class RegionMap:
    """regions.hpp:26-49: labels plus the 11 ascending group lists."""
    cell_label: np.ndarray
    cell_sublabel: np.ndarray
    edge_label: np.ndarray
    interface_width: int
    groups: list
    warnings: list

    def __getattr__(self, name):
        groups = self.__dict__.get("groups")
        if groups is not None and name in GROUP_NAMES:
            return groups[GROUP_NAMES.index(name)]
        if name == "cells_fine":
            return np.sort(np.concatenate(groups[0:3]))
        raise AttributeError(name)

    def group_sizes(self):
        return [len(g) for g in self.groups]


@dataclass
class RegionReport:
    """regions.hpp:74-79."""
    n_fine: int = 0
    n_if1: int = 0
    n_if2: int = 0
    n_coarse: int = 0
    n_uf1: int = 0
    n_uf2: int = 0
    violations: list = field(default_factory=list)
    counts: list = field(default_factory=list)   # offending elements per check kind
    first: list = field(default_factory=list)    # lowest offending id per check kind, -1: none

    def ok(self) -> bool:
        return not self.violations


_WARN_TEXT = {1: "no fine cell touches Interface1; underline layers are empty",
              2: "fine region is one layer thick; second underline layer is empty "
                 "(third-order interface prediction degrades)",
              4: "fine region is only two layers thick; no plain fine cells remain"}


# --------------------------------------------------------------------------

class CudaContext:
    """One mswm_cuda_ctx: a mesh resident on one B200."""

    def __init__(self, mesh: Mesh, b, f_vertex, gravity: float = 9.80616, device: int = 0,
                 order="hilbert", fine_mask=None, interface_width: int = 1):
        """order: "hilbert" (space-filling-curve device layout, default),
        "regions" (region-major: LTS groups contiguous, Hilbert inside; needs
        fine_mask), "input" (the caller's numbering) or an explicit cell
        permutation.  Results are bitwise independent of it."""
        self.lib = _lib.cuda()
        self.mesh = mesh
        self._desc = mesh.desc()
        if isinstance(order, str):
            if order not in ("hilbert", "input", "regions"):
                raise UsageError(f"unknown order '{order}'")
            if order == "regions":
                if fine_mask is None:
                    raise UsageError("order='regions' needs the fine mask")
                from .layout import region_major_order
                order = region_major_order(mesh, fine_mask, interface_width)
            else:
                order = mesh.locality_order() if order == "hilbert" else None
        self._order = None if order is None else np.ascontiguousarray(order, np.int32)
        optr = _p(self._order, _lib.i32p) if self._order is not None else None
        handle = C.c_void_p()
        rc = self.lib.mswm_cuda_create(C.byref(self._desc), device, optr, C.byref(handle))
        if rc:
            _raise(rc, self.lib.mswm_cuda_last_error(None).decode())
        self.handle = handle
        self.regions: RegionMap | None = None
        self.set_fields(b, f_vertex, gravity)

    def close(self):
        if getattr(self, "handle", None):
            self.lib.mswm_cuda_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc:
            msg = self.lib.mswm_cuda_last_error(self.handle).decode()
            v, st = -1, C.c_int64(0)
            if rc == 4:
                v = self.lib.mswm_cuda_dry_vertex(self.handle, C.byref(st))
            _raise(rc, msg, v, st.value)

    def _f64(self, a, n: int, what: str, writable: bool = False) -> np.ndarray:
        """The native side reads / writes exactly n doubles: check before the call."""
        if writable:
            if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous \
                    or not a.flags.writeable:
                raise UsageError(f"{what} must be a writable contiguous float64 array")
        else:
            a = np.ascontiguousarray(a, np.float64)
        if a.shape != (n,):
            raise UsageError(f"{what} has shape {a.shape}, expected ({n},)")
        return a

    # -- setup ---------------------------------------------------------------
    def set_fields(self, b, f_vertex, gravity: float):
        self.b = np.ascontiguousarray(b, np.float64)
        self.f = np.ascontiguousarray(f_vertex, np.float64)
        if self.b.shape != (self.mesh.n_cells,):
            raise UsageError("bottom topography field size does not match the mesh")
        if self.f.shape != (self.mesh.n_vertices,):
            raise UsageError("Coriolis field size does not match the mesh")
        self.gravity = float(gravity)
        self._check(self.lib.mswm_cuda_set_fields(self.handle, _p(self.b, _lib.f64p),
                                                  _p(self.f, _lib.f64p), self.gravity))

    def make_regions(self, fine_mask, interface_width: int = 1) -> RegionMap:
        """make_regions (regions.cpp:164-171) on the device from a host mask."""
        m = self.mesh
        fm = np.ascontiguousarray(fine_mask, np.uint8)
        if fm.shape != (m.n_cells,):
            raise UsageError("fine mask size does not match the mesh")
        cl = np.zeros(m.n_cells, np.uint8)
        cs = np.zeros(m.n_cells, np.uint8)
        el = np.zeros(m.n_edges, np.uint8)
        sizes = np.zeros(11, np.int64)
        warn = C.c_int(0)
        self._check(self.lib.mswm_cuda_set_regions(
            self.handle, _p(fm, _lib.u8p), interface_width, _p(cl, _lib.u8p), _p(cs, _lib.u8p),
            _p(el, _lib.u8p), _p(sizes, _lib.i64p), C.byref(warn)))
        groups = []
        for g in range(11):
            ids = np.zeros(int(sizes[g]), np.int32)
            self._check(self.lib.mswm_cuda_get_group(self.handle, g, _p(ids, _lib.i32p)))
            groups.append(ids)
        warnings = [_WARN_TEXT[warn.value]] if warn.value else []
        self.regions = RegionMap(cl, cs, el, interface_width, groups, warnings)
        return self.regions

    def validate_regions(self, regions: RegionMap | None = None) -> RegionReport:
        """validate_regions (regions.cpp:173-288): the label checks on the device
        (mswm_cuda_validate_labels), the list-cover checks on the group lists."""
        m = self.mesh
        r = regions if regions is not None else self.regions
        if r is None:
            raise UsageError("no region map to validate")
        rep = RegionReport()
        cl = np.ascontiguousarray(r.cell_label, np.uint8)
        if cl.shape != (m.n_cells,):
            rep.violations.append("cell label array size mismatch")
            return rep
        g = r.groups
        rep.n_fine = sum(len(x) for x in g[0:3])
        rep.n_uf1, rep.n_uf2 = len(g[1]), len(g[2])
        rep.n_if1, rep.n_if2, rep.n_coarse = len(g[3]), len(g[4]), len(g[5])

        def cover(lists, n, what):
            ids = np.concatenate([np.asarray(x, np.int64) for x in lists]) if lists else \
                np.zeros(0, np.int64)
            if ids.size and (ids.min() < 0 or ids.max() >= n):
                rep.violations.append(f"{what} id out of range in a group list")
                ids = ids[(ids >= 0) & (ids < n)]
            seen = np.bincount(ids, minlength=n)
            bad = np.flatnonzero(seen != 1)
            if bad.size:
                i = int(bad[0])
                rep.violations.append(f"{what} {i} has no region" if seen[i] == 0
                                      else f"{what} {i} is in several regions")

        cover(g[0:6], m.n_cells, "cell")
        for k, name in ((1, "1"), (2, "2")):
            ids = np.asarray(g[k], np.int64)
            bad = ids[cl[ids] != 0] if ids.size else ids
            if bad.size:
                rep.violations.append(
                    f"underline layer {name} leaves the fine region at cell {int(bad[0])}")
        cs = None if r.cell_sublabel is None else np.ascontiguousarray(r.cell_sublabel, np.uint8)
        el = None if r.edge_label is None else np.ascontiguousarray(r.edge_label, np.uint8)
        if cs is not None and cs.shape != (m.n_cells,):
            raise UsageError("cell sublabel array size mismatch")
        if el is not None and el.shape != (m.n_edges,):
            rep.violations.append("edge label array size mismatch")
            return rep
        counts = np.zeros(6, np.int64)
        first = np.zeros(6, np.int32)
        self._check(self.lib.mswm_cuda_validate_labels(
            self.handle, _p(cl, _lib.u8p), None if cs is None else _p(cs, _lib.u8p),
            None if el is None else _p(el, _lib.u8p), int(r.interface_width),
            _p(counts, _lib.i64p), _p(first, _lib.i32p)))
        rep.counts, rep.first = counts.tolist(), first.tolist()
        w = int(r.interface_width)
        text = ("cell {i} has an invalid label",
                f"Interface1 cell {{i}} is not at distance 1..{w} from fine",
                f"Interface2 cell {{i}} is not at distance {w + 1}..{2 * w} from fine",
                f"coarse cell {{i}} is too close to fine for width {w}",
                "fine cell {i} has the wrong underline sublabel",
                "edge {i} label disagrees with the fine-side-wins rule")
        for k in range(6):
            if counts[k]:
                rep.violations.append(text[k].format(i=int(first[k])))
        if el is not None:
            cover(g[6:11], m.n_edges, "edge")
        return rep

    def closure(self, mask: int, kind: int) -> np.ndarray:
        n = C.c_int64(0)
        self._check(self.lib.mswm_cuda_get_closure(self.handle, int(mask), kind, None,
                                                   C.byref(n)))
        ids = np.zeros(n.value, np.int32)
        self._check(self.lib.mswm_cuda_get_closure(self.handle, int(mask), kind,
                                                   _p(ids, _lib.i32p), C.byref(n)))
        return ids

    # -- device-resident stepping ------------------------------------------
    def upload(self, state: State):
        h = self._f64(state.h, self.mesh.n_cells, "h")
        u = self._f64(state.u, self.mesh.n_edges, "u")
        self._check(self.lib.mswm_cuda_state_upload(self.handle, _p(h, _lib.f64p),
                                                    _p(u, _lib.f64p), float(state.time)))

    def download(self, state: State | None = None) -> State:
        m = self.mesh
        if state is None:
            state = State(np.zeros(m.n_cells), np.zeros(m.n_edges), 0.0)
        self._f64(state.h, m.n_cells, "state.h", writable=True)
        self._f64(state.u, m.n_edges, "state.u", writable=True)
        t = C.c_double(0.0)
        self._check(self.lib.mswm_cuda_state_download(self.handle, _p(state.h, _lib.f64p),
                                                      _p(state.u, _lib.f64p), C.byref(t)))
        state.time = t.value
        return state

    def advance(self, scheme: Scheme, dt: float, substeps: int = 1, n_steps: int = 1,
                sync: bool = True):
        self._check(self.lib.mswm_cuda_step(self.handle, int(scheme), float(dt), int(substeps),
                                            int(n_steps), 1 if sync else 0))

    def sync(self):
        self._check(self.lib.mswm_cuda_sync(self.handle))

    def ledger(self) -> WorkLedger:
        c = np.zeros(16, np.int64)
        e = np.zeros(16, np.int64)
        s = C.c_int64(0)
        self._check(self.lib.mswm_cuda_ledger(self.handle, _p(c, _lib.i64p), _p(e, _lib.i64p),
                                              C.byref(s)))
        return WorkLedger(c.reshape(4, 4), e.reshape(4, 4), s.value)

    def reset_ledger(self):
        self._check(self.lib.mswm_cuda_ledger_reset(self.handle))

    def stream_ptr(self) -> int:
        return self.lib.mswm_cuda_stream(self.handle) or 0

    def set_profiling(self, on):
        """True/1: time every evaluation of the captured step; 2: only the first
        evaluation covering half the mesh (cheaper inside timed steps)."""
        self._check(self.lib.mswm_cuda_set_profiling(self.handle, int(on)))

    def eval_profile(self, cap: int = 4096):
        ms = (C.c_float * cap)()
        nc = np.zeros(cap, np.int64)
        ne = np.zeros(cap, np.int64)
        n = C.c_int(0)
        self._check(self.lib.mswm_cuda_eval_profile(self.handle, ms, _p(nc, _lib.i64p),
                                                    _p(ne, _lib.i64p), cap, C.byref(n)))
        k = min(n.value, cap)
        return np.array(ms[:k], np.float64), nc[:k], ne[:k]

    def layout_info(self) -> dict:
        kp, ident = C.c_int(0), C.c_int(0)
        self._check(self.lib.mswm_cuda_layout_info(self.handle, C.byref(kp), C.byref(ident)))
        return {"kernel_path": {0: "explicit"}[kp.value],
                "input_order": bool(ident.value)}

    def stencil_info(self) -> dict:
        """16-bit stencil offsets in use, and the edges that need the int32 table."""
        o, n = C.c_int(0), C.c_int64(0)
        self._check(self.lib.mswm_cuda_stencil_info(self.handle, C.byref(o), C.byref(n)))
        return {"offsets16": bool(o.value), "n_wide": n.value}

    def index_info(self) -> dict:
        """16-bit index records of kernels A, B, C in use, and the vertices /
        cells / edges whose warps read the int32 tables instead."""
        p = C.c_int(0)
        n = [C.c_int64(0) for _ in range(3)]
        self._check(self.lib.mswm_cuda_index_info(self.handle, C.byref(p), *[C.byref(x) for x in n]))
        return {"packed16": bool(p.value & 1), "cell_records": bool(p.value & 2),
                "n_wide_vertices": n[0].value, "n_wide_cells": n[1].value,
                "n_wide_edges": n[2].value}

    def kernels_per_step(self) -> int:
        n = C.c_int64(0)
        self._check(self.lib.mswm_cuda_kernels_per_step(self.handle, C.byref(n)))
        return n.value

    def partition(self, sweep_order, n_parts: int):
        """Device partition (partition.cpp:219-231, 338-353): (rank of every
        cell, owner rank of every edge) -- each region class cut into n_parts
        near-equal runs of ``sweep_order``.  Needs make_regions first."""
        m = self.mesh
        o = np.ascontiguousarray(sweep_order, np.int32)
        if o.shape != (m.n_cells,):
            raise UsageError(f"sweep_order must have shape ({m.n_cells},)")
        roc = np.zeros(m.n_cells, np.int32)
        own = np.zeros(m.n_edges, np.int32)
        self._check(self.lib.mswm_cuda_partition(self.handle, _p(o, _lib.i32p), int(n_parts),
                                                 _p(roc, _lib.i32p), _p(own, _lib.i32p)))
        return roc, own

    def halo_reach(self, rank_of_cell, n_ranks: int):
        """Device halo plan of a partition (partition.cpp:355-392): uint64 bit
        sets of the ranks whose local mesh holds each cell / edge / vertex."""
        m = self.mesh
        r = np.ascontiguousarray(rank_of_cell, np.int32)
        if r.shape != (m.n_cells,):
            raise UsageError(f"rank_of_cell must have shape ({m.n_cells},)")
        cr = np.zeros(m.n_cells, np.uint64)
        er = np.zeros(m.n_edges, np.uint64)
        vr = np.zeros(m.n_vertices, np.uint64)
        self._check(self.lib.mswm_cuda_halo_reach(self.handle, _p(r, _lib.i32p), int(n_ranks),
                                                  _p(cr, _lib.u64p), _p(er, _lib.u64p),
                                                  _p(vr, _lib.u64p)))
        return cr, er, vr

    def set_replication(self, replication: int) -> None:
        """Cost replication (SchemeConfig::replication): the tendency
        arithmetic repeated per evaluation (operators.cpp:60), results
        unchanged, ledger counts scaled."""
        self._check(self.lib.mswm_cuda_set_replication(self.handle, int(replication)))

    def concurrent_coarse(self) -> int:
        """1: the last captured LTS3 step ran its coarse stage concurrently
        with the substeps; 0: in sequence; -1: no LTS3 step captured yet."""
        v = C.c_int(0)
        self._check(self.lib.mswm_cuda_schedule_info(self.handle, C.byref(v)))
        return v.value

    def total_mass(self) -> float:
        out = C.c_double(0.0)
        self._check(self.lib.mswm_cuda_total_mass(self.handle, C.byref(out)))
        return out.value

    def diagnostics(self, exact: bool = True) -> tuple[float, float]:
        """(total_mass, total_energy) of the device state (harness.cpp:99-123);
        exact: the reference's sequential summation order, else a
        deterministic device tree sum."""
        m, e = C.c_double(0.0), C.c_double(0.0)
        self._check(self.lib.mswm_cuda_diagnostics(self.handle, int(exact), C.byref(m),
                                                   C.byref(e)))
        return m.value, e.value

    def total_energy(self, exact: bool = True) -> float:
        return self.diagnostics(exact)[1]

    def courant(self, dt: float, substeps: int = 1) -> tuple[float, float]:
        """courant_numbers (integrators.cpp:632-659): (fine, coarse)."""
        f, c = C.c_double(0.0), C.c_double(0.0)
        self._check(self.lib.mswm_cuda_courant(self.handle, float(dt), int(substeps), C.byref(f),
                                               C.byref(c)))
        return f.value, c.value


def _p(a, t):
    return a.ctypes.data_as(t)


class CudaEvaluator:
    """TendencyEvaluator (integrators.hpp:68-73) on the GPU.

    ``eval(h, u, mask, dh, du)`` writes dh/du only on the masked groups and
    leaves every other entry untouched; only ``kMaskAll`` is legal without a
    region map.
    """

    def __init__(self, ctx: CudaContext):
        self.ctx = ctx

    def eval(self, h, u, mask: int, dh: np.ndarray, du: np.ndarray):
        c = self.ctx
        m = c.mesh
        c._f64(dh, m.n_cells, "dh", writable=True)
        c._f64(du, m.n_edges, "du", writable=True)
        h = c._f64(h, m.n_cells, "h")
        u = c._f64(u, m.n_edges, "u")
        c._check(c.lib.mswm_cuda_eval(c.handle, _p(h, _lib.f64p), _p(u, _lib.f64p), int(mask),
                                      _p(dh, _lib.f64p), _p(du, _lib.f64p)))


class CudaStepper:
    """Stepper (integrators.hpp:136-160) with device-resident state.

    Each call uploads the State, advances on the device and downloads it --
    the drop-in form.  Long runs should call ``ctx.upload`` once,
    ``ctx.advance(..., n_steps)`` and ``ctx.download`` at the end.
    """

    def __init__(self, ctx: CudaContext):
        self.ctx = ctx

    def _run(self, state: State, scheme: Scheme, dt: float, M: int):
        self.ctx.upload(state)
        self.ctx.advance(scheme, dt, M, 1)
        self.ctx.download(state)

    def ssprk_step(self, order: int, state: State, dt: float):
        if order not in (2, 3):
            raise UsageError("ssprk_step: order must be 2 or 3")
        self._run(state, Scheme.SSPRK2 if order == 2 else Scheme.SSPRK3, dt, 1)

    def rk4_step(self, state: State, dt: float):
        self._run(state, Scheme.RK4, dt, 1)

    def lts_step(self, order: int, state: State, dt: float, substeps: int):
        if order not in (2, 3):
            raise UsageError("lts_step: order must be 2 or 3")
        self._run(state, Scheme.LTS2 if order == 2 else Scheme.LTS3, dt, substeps)

    def step(self, state: State, cfg: SchemeConfig):
        self._run(state, cfg.scheme, cfg.dt, cfg.substeps)

"""Multi-rank LTS3 on B200s: rank contexts, halo plans, transports.

One rank = one GPU = one ``mswm_cuda_ctx`` holding the rank's piece of the
mesh (``partition.LocalMesh``: owned cells/edges + two-hop halo, the
reference's block plan, partition.cpp:307-403).  Region labels come from the
global ``RegionMap`` (bit-exact with make_regions), outputs are the owned
elements only, and halo copies of the stage arrays are refreshed before every
evaluation.  Transports:

* NCCL point-to-point (one process per GPU, ``torch.distributed`` for the
  rendezvous): ``RankContext.init_nccl``;
* an in-process group of rank contexts on one device (``CudaGroup``), used to
  test the exchange path on a single GPU without kernels that wait on each
  other.

Per-rank results are bitwise identical to the single-GPU path (and to the
reference): every owned element's arithmetic reads exactly the values the
single-GPU evaluation reads.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .api import CudaContext, Error, State, _p, _raise
from .mesh import Mesh
from .partition import LocalMesh, build_local_meshes, partition_cells


def swap_needs(rank: int, n_ranks: int, needs: dict) -> dict:
    """Setup-time metadata swap over torch.distributed: given this rank's
    {peer: positions it needs from peer}, return {peer: positions peer needs
    from this rank}."""
    import torch.distributed as dist
    allv = [None] * n_ranks
    dist.all_gather_object(allv, {int(q): np.asarray(v, np.int32) for q, v in needs.items()})
    return {int(q): allv[int(q)].get(rank, np.zeros(0, np.int32)) for q in needs}


def publish_store(store_dir, wl, device: int = 0, n_ranks: int | None = None) -> dict:
    """Rank 0 of a multi-GPU job: on one global context (closed again) the
    device region labels of the global mesh and, for ``n_ranks``, the
    partition's halo plan (halo_reach bit sets); then the whole workload,
    labels, locality order and plan written as a binary store (store.py)
    that every rank memory-maps.  Returns the extra arrays written."""
    from . import store
    g = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, device=device)
    rm = g.make_regions(wl.fine_mask, wl.width)
    extra = {"cell_label": np.asarray(rm.cell_label, np.uint8),
             "cell_sub": np.asarray(rm.cell_sublabel, np.uint8),
             "edge_label": np.asarray(rm.edge_label, np.uint8),
             "order": np.asarray(wl.mesh.locality_order(), np.int32)}
    if n_ranks:
        # partition and halo plan on the device (partition.cpp:219-231,
        # 338-353, 355-392)
        roc, own = g.partition(extra["order"], n_ranks)
        cr, er, vr = g.halo_reach(roc, n_ranks)
        extra.update({"rank_of_cell": roc, "edge_owner": own, "cell_reach": cr,
                      "edge_reach": er, "vertex_reach": vr})
    g.close()
    del g
    store.save_workload(store_dir, wl, extra, digest=False)
    return extra


def layout_from_store(store_dir, rank: int, n_ranks: int):
    """(workload, DistributedLayout for ``rank`` alone) from a published
    store: the global tables are shared read-only maps, only this rank's
    local mesh and halo plan are materialised."""
    from . import store
    wl, extra = store.load_workload(store_dir, mmap=True)
    reach = part = None
    if "cell_reach" in extra and int(np.max(extra["rank_of_cell"])) == n_ranks - 1:
        reach = (extra["cell_reach"], extra["edge_reach"], extra["vertex_reach"])
        if "edge_owner" in extra:
            part = (np.asarray(extra["rank_of_cell"]), np.asarray(extra["edge_owner"]))
    lay = DistributedLayout(wl.mesh, extra["cell_label"], extra["cell_sub"], extra["edge_label"],
                            n_ranks, order=np.asarray(extra["order"]), only=rank, reach=reach,
                            partition=part)
    return wl, lay


class DistributedLayout:
    """Partition + local meshes of a global mesh with given region labels."""

    def __init__(self, mesh: Mesh, cell_label, cell_sub, edge_label, n_ranks: int,
                 order: np.ndarray | None = None, only: int | None = None, ctx=None,
                 reach=None, partition=None):
        """``partition``: precomputed (rank_of_cell, edge_owner), e.g. the
        device partition published by rank 0; else partition_cells on the
        host."""
        self.mesh = mesh
        self.n_ranks = n_ranks
        self.cell_label = np.asarray(cell_label, np.uint8)
        self.cell_sub = np.asarray(cell_sub, np.uint8)
        self.edge_label = np.asarray(edge_label, np.uint8)
        self.order = mesh.locality_order() if order is None else np.asarray(order)
        own = None
        if partition is not None:
            self.rank_of_cell, own = partition
        else:
            self.rank_of_cell = partition_cells(self.order, self.cell_label, n_ranks)
        self.locals: list[LocalMesh] = build_local_meshes(mesh, self.cell_label, self.cell_sub,
                                                          self.edge_label, self.rank_of_cell,
                                                          n_ranks, only=only, ctx=ctx,
                                                          reach=reach, own_edges=own)
        hr = np.empty(mesh.n_cells, np.int64)
        hr[self.order] = np.arange(mesh.n_cells)
        self.hilbert_rank = hr

    def local_order(self, r: int) -> np.ndarray:
        """Device layout of rank r: local cells along the global curve."""
        lm = self.locals[r]
        o = np.argsort(self.hilbert_rank[lm.cells], kind="stable").astype(np.int32)
        return np.concatenate([o, [lm.n_cells - 1]]).astype(np.int32)


class RankContext:
    """A CudaContext on one rank's local mesh."""

    def __init__(self, layout: DistributedLayout, rank: int, b, f, gravity: float,
                 interface_width: int = 1, device: int = 0):
        lm = layout.locals[rank]
        self.layout, self.rank, self.lm = layout, rank, lm
        self.local_mesh = lm.as_mesh()
        self.ctx = CudaContext(self.local_mesh, lm.gather_cells(np.asarray(b, np.float64)),
                               lm.gather_vertices(np.asarray(f, np.float64)), gravity, device,
                               order=layout.local_order(rank))
        cl = np.concatenate([layout.cell_label[lm.cells], [3]]).astype(np.uint8)
        cs = np.concatenate([layout.cell_sub[lm.cells], [0]]).astype(np.uint8)
        el = np.concatenate([layout.edge_label[lm.edges], [4]]).astype(np.uint8)
        self._labels = (cl, cs, el, lm.cell_owned, lm.edge_owned)
        lib = self.ctx.lib
        self.ctx._check(lib.mswm_cuda_set_labels(
            self.ctx.handle, _p(cl, _lib.u8p), _p(cs, _lib.u8p), _p(el, _lib.u8p),
            _p(lm.cell_owned, _lib.u8p), _p(lm.edge_owned, _lib.u8p), interface_width))
        peers = sorted(set(lm.send_cells) | set(lm.recv_cells))
        counts, ids = [], []
        for q in peers:
            parts = [lm.send_cells.get(q, np.zeros(0, np.int32)),
                     lm.send_edges.get(q, np.zeros(0, np.int32)),
                     lm.recv_cells.get(q, np.zeros(0, np.int32)),
                     lm.recv_edges.get(q, np.zeros(0, np.int32))]
            counts.extend(len(x) for x in parts)
            ids.extend(parts)
        self._peers = np.asarray(peers, np.int32)
        self._counts = np.asarray(counts, np.int64)
        self._ids = np.concatenate(ids).astype(np.int32) if ids else np.zeros(1, np.int32)
        self.ctx._check(lib.mswm_cuda_set_halo(
            self.ctx.handle, rank, layout.n_ranks, len(peers), _p(self._peers, _lib.i32p),
            _p(self._counts, _lib.i64p), _p(self._ids, _lib.i32p)))

    # -- halo restriction per mask --------------------------
    def halo_needs(self, mask: int) -> dict[int, np.ndarray]:
        """Positions within each peer's receive list that the evaluation with
        `mask` reads: {peer rank: positions}."""
        lib = self.ctx.lib
        counts = np.zeros(max(len(self._peers), 1), np.int64)
        self.ctx._check(lib.mswm_cuda_halo_needs(self.ctx.handle, mask, _p(counts, _lib.i64p), None))
        pos = np.zeros(max(int(counts.sum()), 1), np.int32)
        self.ctx._check(lib.mswm_cuda_halo_needs(self.ctx.handle, mask, _p(counts, _lib.i64p),
                                                 _p(pos, _lib.i32p)))
        out, at = {}, 0
        for j, q in enumerate(self._peers):
            out[int(q)] = pos[at:at + counts[j]].copy()
            at += counts[j]
        return out

    def set_halo_mask(self, mask: int, send: dict[int, np.ndarray], recv: dict[int, np.ndarray]):
        """Install the restriction: send[q] = positions in my send list to q
        (q's needs from me), recv[q] = my needs from q."""
        empty = np.zeros(0, np.int32)
        sc = np.array([len(send.get(int(q), empty)) for q in self._peers] or [0], np.int64)
        rc = np.array([len(recv.get(int(q), empty)) for q in self._peers] or [0], np.int64)
        sp = np.concatenate([send.get(int(q), empty) for q in self._peers] + [np.zeros(1, np.int32)])
        rp = np.concatenate([recv.get(int(q), empty) for q in self._peers] + [np.zeros(1, np.int32)])
        sp, rp = sp.astype(np.int32), rp.astype(np.int32)
        self.ctx._check(self.ctx.lib.mswm_cuda_set_halo_mask(
            self.ctx.handle, mask, _p(sc, _lib.i64p), _p(sp, _lib.i32p), _p(rc, _lib.i64p),
            _p(rp, _lib.i32p)))

    def restrict_halos(self, masks, exchange=None):
        """Per-mask halo restriction for this rank.  `exchange(needs)` maps this
        rank's {peer: positions} to {peer: that peer's positions for me}; by
        default torch.distributed all_gather_object (setup time only)."""
        if exchange is None:
            def exchange(needs):
                return swap_needs(self.rank, self.layout.n_ranks, needs)
        for m in masks:
            needs = self.halo_needs(int(m))
            self.set_halo_mask(int(m), exchange(needs), needs)

    # -- NCCL transport ------------------------------------------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_char * 128)()
        rc = _lib.cuda().mswm_cuda_nccl_unique_id(C.cast(buf, C.c_void_p))
        if rc:
            _raise(rc, _lib.cuda().mswm_cuda_last_error(None).decode())
        return bytes(buf)

    def init_nccl(self, unique_id: bytes):
        buf = (C.c_char * 128).from_buffer_copy(unique_id)
        self.ctx._check(self.ctx.lib.mswm_cuda_comm_init(
            self.ctx.handle, C.cast(buf, C.c_void_p), self.rank, self.layout.n_ranks))

    # -- peer-store transport ---------------------------------------------------
    def peer_export(self) -> tuple[bytes, np.ndarray]:
        """This rank's arena as a CUDA IPC handle plus the table of where each
        neighbour's values land in it (after restrict_halos: the arena follows
        the halo plans)."""
        n = C.c_int64(0)
        self.ctx._check(self.ctx.lib.mswm_cuda_peer_export(self.ctx.handle, None, None, 0, C.byref(n)))
        rows = np.zeros((max(n.value, 1), 5), np.int64)
        buf = (C.c_char * 64)()
        self.ctx._check(self.ctx.lib.mswm_cuda_peer_export(
            self.ctx.handle, C.cast(buf, C.c_void_p), _p(rows, _lib.i64p), rows.shape[0], C.byref(n)))
        return bytes(buf), rows[:n.value]

    def peer_import(self, peer_rank: int, handle: bytes, rows: np.ndarray):
        buf = (C.c_char * 64).from_buffer_copy(handle)
        rows = np.ascontiguousarray(rows, np.int64)
        self.ctx._check(self.ctx.lib.mswm_cuda_peer_import(
            self.ctx.handle, int(peer_rank), C.cast(buf, C.c_void_p), _p(rows, _lib.i64p),
            rows.shape[0]))

    def init_peer(self):
        """Halo exchanges as stores into the neighbours' buffers (CUDA IPC over
        NVLink peer access) with device flags instead of NCCL send/recv: the
        handles and tables travel once over torch.distributed."""
        import torch.distributed as dist
        allv = [None] * self.layout.n_ranks
        dist.all_gather_object(allv, self.peer_export())
        for q in self._peers:
            self.peer_import(int(q), *allv[int(q)])
        self.ctx._check(self.ctx.lib.mswm_cuda_peer_enable(self.ctx.handle, 1))

    def peer_exchange(self, phase: int):
        """One full-halo exchange of the state in two host-ordered halves (0:
        pack + store + signal, 1: wait + unpack) -- the cross-process test of
        the mapping; stepping runs them back to back inside the step graph."""
        self.ctx._check(self.ctx.lib.mswm_cuda_peer_exchange(self.ctx.handle, int(phase)))

    # -- state ---------------------------------------------------------------
    def upload(self, h_global, u_global, time: float = 0.0):
        lm = self.lm
        self.ctx.upload(State(lm.gather_cells(np.asarray(h_global, np.float64)),
                              lm.gather_edges(np.asarray(u_global, np.float64)), time))

    def download_owned(self, h_global: np.ndarray, u_global: np.ndarray) -> float:
        """Write this rank's owned values into the global arrays."""
        st = self.ctx.download()
        lm = self.lm
        h_global[lm.cells[:lm.n_owned_cells]] = st.h[:lm.n_owned_cells]
        u_global[lm.edges[:lm.n_owned_edges]] = st.u[:lm.n_owned_edges]
        return st.time


class CudaGroup:
    """All ranks of a layout as contexts on one device, stepped in lockstep."""

    def __init__(self, ranks: list[RankContext]):
        self.ranks = ranks
        lib = _lib.cuda()
        arr = (C.c_void_p * len(ranks))(*[r.ctx.handle.value for r in ranks])
        h = C.c_void_p()
        rc = lib.mswm_cuda_group_create(arr, len(ranks), C.byref(h))
        if rc:
            _raise(rc, lib.mswm_cuda_last_error(None).decode())
        self.handle = h
        self.lib = lib

    def restrict_halos(self, masks):
        """Per-mask halo restriction of every member (in-process peers)."""
        for m in masks:
            needs = [rc.halo_needs(int(m)) for rc in self.ranks]
            for r, rc in enumerate(self.ranks):
                send = {q: needs[q].get(r, np.zeros(0, np.int32)) for q in needs[r]}
                rc.set_halo_mask(int(m), send, needs[r])

    def use_nccl_loopback(self):
        """Halo copies as NCCL send/recv to self over a one-rank communicator
        (the NCCL transport's code path on one GPU)."""
        rc = self.lib.mswm_cuda_group_nccl_loopback(self.handle)
        if rc:
            _raise(rc, self.lib.mswm_cuda_group_last_error(self.handle).decode())

    def use_peer_stores(self, on: bool = True):
        """Halo exchanges as stores into the neighbours' buffers plus device
        flags (the peer-store transport with in-process pointers)."""
        rc = self.lib.mswm_cuda_group_peer(self.handle, int(on))
        if rc:
            _raise(rc, self.lib.mswm_cuda_group_last_error(self.handle).decode())

    def advance(self, scheme, dt: float, substeps: int = 1, n_steps: int = 1):
        rc = self.lib.mswm_cuda_group_step(self.handle, int(scheme), float(dt), int(substeps),
                                           int(n_steps))
        if rc:
            _raise(rc, self.lib.mswm_cuda_group_last_error(self.handle).decode())

    def close(self):
        if getattr(self, "handle", None):
            self.lib.mswm_cuda_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

"""Domain decomposition for the multi-GPU LTS3 path.

Restates the reference's rank/block layout for one process per GPU:

* ``partition_cells`` -- per-class balanced split (partition.cpp:219-231): each
  class (fine incl. underline, coarse, interface) is cut into N near-equal
  consecutive runs, so every rank holds 1/N of the fine work (weighted M x by
  the substeps) *and* 1/N of the coarse work and no rank idles in a phase
  (PAPER.md:482-483).  The sweep order is the Hilbert curve instead of the
  reference's BFS sweep; the boundary-refinement pass is not used.
* ``edge_owner`` -- edge ownership rule of make_block_plan (partition.cpp:338-353):
  the first cell of ``edge_cells`` whose class equals the edge's class.
* ``LocalMesh`` -- owned cells plus the cells within two hops (the reference's
  halo, partition.cpp:355-392), every ring edge and ring vertex of those cells,
  renumbered locally; references that leave the local set point to one dummy
  cell/edge/vertex whose values are never read by an owned output.  The halo
  plan lists, per peer, which local halo elements that peer owns (receive) and
  which owned elements the peer needs (send), both in ascending global id so
  both sides agree on the order.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import Mesh

# class of a cell: 0 fine (incl. underline), 1 coarse, 2 interface (partition.cpp:16-25)
def cell_class(cell_label: np.ndarray) -> np.ndarray:
    cl = np.asarray(cell_label)
    return np.where(cl == 0, 0, np.where(cl == 3, 1, 2)).astype(np.int8)


def edge_class(edge_label: np.ndarray) -> np.ndarray:
    """partition.cpp:27-37: fine/underline-fine edges 0, coarse 1, interfaces 2."""
    el = np.asarray(edge_label)
    return np.where(el <= 1, 0, np.where(el == 4, 1, 2)).astype(np.int8)


def partition_cells(order: np.ndarray, cell_label: np.ndarray, n_parts: int) -> np.ndarray:
    """rank of every cell: position pos of t in its class's run along `order`
    goes to part pos*N/t (partition.cpp:219-231)."""
    n = len(order)
    if n_parts < 1 or n_parts > n:
        raise ValueError("n_parts out of range")
    cls = cell_class(cell_label)[order]
    rank = np.zeros(n, np.int32)
    for k in range(3):
        sel = np.nonzero(cls == k)[0]
        t = len(sel)
        if t == 0:
            continue
        pos = np.arange(t, dtype=np.int64)
        rank[order[sel]] = (pos * n_parts // t).astype(np.int32)
    return rank


def partition_device(ctx, order: np.ndarray, n_parts: int):
    """(rank_of_cell, edge_owner) computed on the device by a CudaContext on
    the global mesh with its region map (mswm_cuda_partition): the same rules
    as partition_cells and edge_owner, run as a class-keyed order-preserving
    compaction of the sweep plus one pass over the edges."""
    return ctx.partition(order, n_parts)


def edge_owner(mesh: Mesh, cell_label: np.ndarray, edge_label: np.ndarray,
               rank_of_cell: np.ndarray) -> np.ndarray:
    """Rank owning each edge (partition.cpp:338-353)."""
    ec = mesh.edge_cells
    ccls = cell_class(cell_label)
    ecls = edge_class(edge_label)
    first = ccls[ec[:, 0]] == ecls
    second = ccls[ec[:, 1]] == ecls
    if not np.all(first | second):
        bad = int(np.nonzero(~(first | second))[0][0])
        raise ValueError(f"edge {bad} has no adjacent cell of its own region class")
    owner_cell = np.where(first, ec[:, 0], ec[:, 1])
    return rank_of_cell[owner_cell].astype(np.int32)


def ring_neighbours(mesh: Mesh):
    co = mesh.cell_offset
    deg = np.diff(co)
    rows = np.repeat(np.arange(mesh.n_cells), deg)
    return rows, mesh.cell_cells, mesh.cell_edges, mesh.cell_vertices


@dataclass
class LocalMesh:
    """One rank's piece of the mesh in local numbering (plus one dummy of each)."""
    rank: int
    n_ranks: int
    cells: np.ndarray          # global ids of local cells (owned first, ascending within)
    edges: np.ndarray
    vertices: np.ndarray
    n_owned_cells: int
    n_owned_edges: int
    tables: dict               # mswm_mesh_desc tables, local ids
    cell_owned: np.ndarray     # uint8 per local cell (dummy excluded -> 0)
    edge_owned: np.ndarray
    send_cells: dict = field(default_factory=dict)   # peer -> local ids (ascending global)
    recv_cells: dict = field(default_factory=dict)
    send_edges: dict = field(default_factory=dict)
    recv_edges: dict = field(default_factory=dict)

    @property
    def n_cells(self):
        return len(self.cells) + 1

    @property
    def n_edges(self):
        return len(self.edges) + 1

    @property
    def n_vertices(self):
        return len(self.vertices) + 1

    def as_mesh(self) -> Mesh:
        m = Mesh(self.n_cells, self.n_edges, self.n_vertices, self.tables, None, None, None, None,
                 False)
        return m

    def gather_cells(self, x: np.ndarray) -> np.ndarray:
        """Local view of a global cell field (dummy value 1.0)."""
        return np.concatenate([x[self.cells], [1.0]])

    def gather_edges(self, x: np.ndarray) -> np.ndarray:
        return np.concatenate([x[self.edges], [0.0]])

    def gather_vertices(self, x: np.ndarray) -> np.ndarray:
        return np.concatenate([x[self.vertices], [0.0]])


def halo_reach(mesh: Mesh, rank_of_cell: np.ndarray, n_ranks: int, ctx=None):
    """Local-mesh membership of every rank at once (make_block_plan's 2-hop
    halo, partition.cpp:355-392): uint64 bit sets per cell / edge / vertex of
    the ranks whose local mesh (owned cells + cells within two hops, their
    ring edges and ring vertices) holds it.  ``ctx`` (a CudaContext on the
    mesh): computed on the device (mswm_cuda_halo_reach); else vectorised
    on the host.  Two OR passes over the ring neighbours replace one BFS per
    rank."""
    if not 1 <= n_ranks <= 64:
        raise ValueError("n_ranks must lie in [1, 64]")
    if ctx is not None:
        return ctx.halo_reach(rank_of_cell, n_ranks)
    co = np.asarray(mesh.cell_offset, np.int64)
    nbr = np.asarray(mesh.cell_cells)
    r = np.left_shift(np.uint64(1), np.asarray(rank_of_cell, np.uint64))
    for _ in range(2):
        r = r | np.bitwise_or.reduceat(r[nbr], co[:-1])
    ec = np.asarray(mesh.edge_cells)
    vc = np.asarray(mesh.vertex_cells)
    return r, r[ec[:, 0]] | r[ec[:, 1]], r[vc[:, 0]] | r[vc[:, 1]] | r[vc[:, 2]]


def _has(bits: np.ndarray, q: int) -> np.ndarray:
    return (bits >> np.uint64(q)) & np.uint64(1) == np.uint64(1)


def build_local_meshes(mesh: Mesh, cell_label, cell_sub, edge_label, rank_of_cell: np.ndarray,
                       n_ranks: int, only: int | None = None, ctx=None, reach=None,
                       own_edges: np.ndarray | None = None) -> list:
    """Local meshes and halo plans.  With ``only`` = r, the tables are built
    for rank r alone (the others are None) -- what one process of a
    multi-GPU run needs.  The membership bit sets come from the device when
    ``ctx`` (a CudaContext on ``mesh``) is given (halo_reach), or precomputed
    as ``reach``."""
    own_e = (edge_owner(mesh, cell_label, edge_label, rank_of_cell) if own_edges is None
             else np.asarray(own_edges))
    co = mesh.cell_offset
    cr, er, vr = reach if reach is not None else halo_reach(mesh, rank_of_cell, n_ranks, ctx)

    def sets_of(r):
        owned_c = rank_of_cell == r
        owned_e = own_e == r
        e_mask = _has(er, r)
        if np.any(owned_e & ~e_mask):
            raise AssertionError("an owned edge is not a ring edge of a local cell")
        return owned_c, _has(cr, r), owned_e, e_mask

    build = range(n_ranks) if only is None else [only]
    out = [None] * n_ranks
    for r in build:
        owned_c, lc_mask, owned_e, e_mask = sets_of(r)
        # cells: owned first, then halo, each ascending
        cells = np.concatenate([np.nonzero(owned_c)[0], np.nonzero(lc_mask & ~owned_c)[0]])
        v_mask = _has(vr, r)
        edges = np.concatenate([np.nonzero(owned_e)[0], np.nonzero(e_mask & ~owned_e)[0]])
        verts = np.nonzero(v_mask)[0]
        nC, nE, nV = len(cells) + 1, len(edges) + 1, len(verts) + 1
        dC, dE, dV = nC - 1, nE - 1, nV - 1
        gc = np.full(mesh.n_cells, dC, np.int32)
        gc[cells] = np.arange(len(cells), dtype=np.int32)
        ge = np.full(mesh.n_edges, dE, np.int32)
        ge[edges] = np.arange(len(edges), dtype=np.int32)
        gv = np.full(mesh.n_vertices, dV, np.int32)
        gv[verts] = np.arange(len(verts), dtype=np.int32)
        deg = np.diff(co)[cells]
        # local CSR rings (dummy cell: a triangle of dummies)
        offs = np.zeros(nC + 1, np.int32)
        offs[1:len(cells) + 1] = np.cumsum(deg)
        offs[nC] = offs[nC - 1] + 3
        take = csr_take(co, cells)
        ring_e = np.concatenate([ge[mesh.cell_edges[take]], [dE] * 3]).astype(np.int32)
        ring_v = np.concatenate([gv[mesh.cell_vertices[take]], [dV] * 3]).astype(np.int32)
        ring_c = np.concatenate([gc[mesh.cell_cells[take]], [dC] * 3]).astype(np.int32)
        eoff_g = mesh.edge_edge_offset
        slen = np.diff(eoff_g)[edges]
        eoff = np.zeros(nE + 1, np.int32)
        eoff[1:len(edges) + 1] = np.cumsum(slen)
        eoff[nE] = eoff[nE - 1]
        stake = csr_take(eoff_g, edges)
        t = {
            "cell_offset": offs,
            "cell_edges": ring_e,
            "cell_vertices": ring_v,
            "cell_cells": ring_c,
            "edge_cells": np.concatenate([gc[mesh.edge_cells[edges]], [[dC, dC]]]).astype(np.int32),
            "edge_vertices": np.concatenate([gv[mesh.edge_vertices[edges]], [[dV, dV]]]).astype(np.int32),
            "vertex_cells": np.concatenate([gc[mesh.vertex_cells[verts]], [[dC] * 3]]).astype(np.int32),
            "vertex_edges": np.concatenate([ge[mesh.vertex_edges[verts]], [[dE] * 3]]).astype(np.int32),
            "edge_edge_offset": eoff,
            "edge_edges": ge[mesh.edge_edges[stake]].astype(np.int32),
            "edge_cell_sign": np.concatenate([mesh.edge_cell_sign[edges], [[-1, 1]]]).astype(np.int8),
            "edge_vertex_sign": np.concatenate([mesh.edge_vertex_sign[edges], [[-1, 1]]]).astype(np.int8),
            "edge_len": np.concatenate([mesh.edge_len[edges], [1.0]]),
            "edge_dual_len": np.concatenate([mesh.edge_dual_len[edges], [1.0]]),
            "cell_area": np.concatenate([mesh.cell_area[cells], [1.0]]),
            "vertex_area": np.concatenate([mesh.vertex_area[verts], [1.0]]),
            "vertex_kite": np.concatenate([mesh.vertex_kite[verts], [[1.0, 1.0, 1.0]]]),
            "edge_weight": mesh.edge_weight[stake].astype(np.float64),
        }
        t = {k: np.ascontiguousarray(v) for k, v in t.items()}
        cell_owned = np.zeros(nC, np.uint8)
        cell_owned[:int(owned_c.sum())] = 1
        edge_owned = np.zeros(nE, np.uint8)
        edge_owned[:int(owned_e.sum())] = 1
        lm = LocalMesh(r, n_ranks, cells.astype(np.int64), edges.astype(np.int64),
                       verts.astype(np.int64), int(owned_c.sum()), int(owned_e.sum()), t,
                       cell_owned, edge_owned)
        # halo plan: receive from each peer the halo elements it owns; send to
        # each peer the owned elements inside its local set.  Ascending global
        # id on both sides.
        for p in range(n_ranks):
            if p == r:
                continue
            p_owned_c, p_lc = rank_of_cell == p, _has(cr, p)
            p_owned_e, p_e = own_e == p, _has(er, p)
            rc_ = np.nonzero(lc_mask & p_owned_c)[0]
            re_ = np.nonzero(e_mask & p_owned_e)[0]
            sc_ = np.nonzero(owned_c & p_lc)[0]
            se_ = np.nonzero(owned_e & p_e)[0]
            if len(rc_) or len(re_):
                lm.recv_cells[p] = gc[rc_]
                lm.recv_edges[p] = ge[re_]
            if len(sc_) or len(se_):
                lm.send_cells[p] = gc[sc_]
                lm.send_edges[p] = ge[se_]
        out[r] = lm
    return out


def csr_take(off: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """Indices into a CSR value array for the given rows, row after row."""
    off = np.asarray(off, np.int64)
    lens = off[rows + 1] - off[rows]
    if len(rows) == 0 or lens.sum() == 0:
        return np.zeros(0, np.int64)
    starts = np.repeat(off[rows] - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens)
    return starts + np.arange(int(lens.sum()), dtype=np.int64)


def _local_ids(local_globals: np.ndarray, wanted: np.ndarray) -> np.ndarray:
    idx = np.argsort(local_globals, kind="stable")
    pos = np.searchsorted(local_globals[idx], wanted)
    ids = idx[pos]
    assert np.array_equal(local_globals[ids], wanted)
    return ids.astype(np.int32)

"""Multi-rank host logic on CPU: partition rules, local meshes, halo plans,
and a world_size-2 gloo run of the halo exchange + per-rank evaluation
against the single-process oracle (test_partition.cpp:180-410 analogues)."""
import os

import numpy as np
import pytest

from helpers import bits_equal
from oracle.oracle import Oracle
from paper_2106_07154_b200 import workloads as W
from paper_2106_07154_b200.api import LTS3_MASKS, kMaskAll
from paper_2106_07154_b200.dist import DistributedLayout
from paper_2106_07154_b200.partition import cell_class, edge_class, edge_owner


def _labels(wl):
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, wl.width)
    return o, o.labels()


@pytest.fixture(scope="module")
def sphere():
    wl = W.small_sphere(5, seed=21, cap_deg=25.0)
    o, (cl, cs, el) = _labels(wl)
    return wl, o, cl, cs, el


@pytest.mark.parametrize("n_ranks", [1, 2, 3, 8])
def test_partition_balance_and_ownership(sphere, n_ranks):
    wl, o, cl, cs, el = sphere
    lay = DistributedLayout(wl.mesh, cl, cs, el, n_ranks)
    cls = cell_class(cl)
    # per-class balance within one cell (test_partition.cpp:180-210)
    for k in range(3):
        counts = np.bincount(lay.rank_of_cell[cls == k], minlength=n_ranks)
        assert counts.max() - counts.min() <= 1
    # every cell and edge owned exactly once
    owned_c = np.concatenate([lm.cells[:lm.n_owned_cells] for lm in lay.locals])
    owned_e = np.concatenate([lm.edges[:lm.n_owned_edges] for lm in lay.locals])
    assert np.array_equal(np.sort(owned_c), np.arange(wl.mesh.n_cells))
    assert np.array_equal(np.sort(owned_e), np.arange(wl.mesh.n_edges))
    # edge owner = first adjacent cell of the edge's class (partition.cpp:338-353)
    own = edge_owner(wl.mesh, cl, el, lay.rank_of_cell)
    ec = wl.mesh.edge_cells
    ecls = edge_class(el)
    for e in range(0, wl.mesh.n_edges, 37):
        c = ec[e][0] if cls[ec[e][0]] == ecls[e] else ec[e][1]
        assert own[e] == lay.rank_of_cell[c]


def test_local_cells_equal_reference_block_plan_halos(ref_lib, sphere):
    """Owned + halo cells of a rank = the union over its three blocks of the
    reference's make_block_plan owned + 2-hop halo (partition.cpp:355-392)."""
    wl, o, cl, cs, el = sphere
    n = 3
    lay = DistributedLayout(wl.mesh, cl, cs, el, n)
    rm = ref_lib.RefMesh.from_mesh(wl.mesh)
    rr = ref_lib.RefRegions(rm, wl.fine_mask, 1)
    plan = ref_lib.ref_block_plan(rm, rr, lay.rank_of_cell, n)
    for r in range(n):
        cells = set()
        edges_owned = set()
        for b in range(3 * r, 3 * r + 3):
            owned_c, owned_e, halo_c, halo_e = plan[b]
            cells |= set(owned_c.tolist()) | set(halo_c.tolist())
            edges_owned |= set(owned_e.tolist())
        lm = lay.locals[r]
        assert set(lm.cells.tolist()) == cells
        assert set(lm.edges[:lm.n_owned_edges].tolist()) == edges_owned


@pytest.mark.parametrize("n_ranks", [2, 4])
def test_local_evaluation_bitwise_equals_global(sphere, n_ranks):
    """Each rank's oracle evaluation on its local mesh (owned outputs only,
    halo values from the global state) equals the global evaluation."""
    wl, o, cl, cs, el = sphere
    lay = DistributedLayout(wl.mesh, cl, cs, el, n_ranks)
    for mask in LTS3_MASKS + [kMaskAll]:
        dh_g = np.full(wl.mesh.n_cells, np.nan)
        du_g = np.full(wl.mesh.n_edges, np.nan)
        o.eval(wl.h, wl.u, mask, dh_g, du_g)
        for lm in lay.locals:
            lo = Oracle(lm.as_mesh(), lm.gather_cells(wl.b), lm.gather_vertices(wl.f), wl.gravity)
            lcl = np.concatenate([cl[lm.cells], [3]])
            lcs = np.concatenate([cs[lm.cells], [0]])
            lel = np.concatenate([el[lm.edges], [4]])
            cells = [i for i in range(lm.n_owned_cells)
                     if mask & (1 << (int(lcs[i]) if lcl[i] == 0 else int(lcl[i]) + 2))]
            edges = [e for e in range(lm.n_owned_edges) if mask & (1 << (6 + int(lel[e])))]
            dh = np.full(lm.n_cells, np.nan)
            du = np.full(lm.n_edges, np.nan)
            lo.tendencies(lm.gather_cells(wl.h), lm.gather_edges(wl.u), cells, edges, dh, du)
            assert bits_equal(dh[cells], dh_g[lm.cells[cells]])
            assert bits_equal(du[edges], du_g[lm.edges[edges]])


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = W.small_sphere(4, seed=5, cap_deg=30.0)
        o, (cl, cs, el) = _labels(wl)
        lay = DistributedLayout(wl.mesh, cl, cs, el, world)
        lm = lay.locals[rank]
        rng = np.random.default_rng(1)
        field_c = rng.normal(size=wl.mesh.n_cells)
        field_e = rng.normal(size=wl.mesh.n_edges)
        # local arrays: owned values only, halo poisoned with NaN
        hc = np.full(lm.n_cells, np.nan)
        ue = np.full(lm.n_edges, np.nan)
        hc[:lm.n_owned_cells] = field_c[lm.cells[:lm.n_owned_cells]]
        ue[:lm.n_owned_edges] = field_e[lm.edges[:lm.n_owned_edges]]
        # halo exchange through gloo with the plan the device path uses
        reqs, bufs = [], {}
        for p in sorted(set(lm.send_cells) | set(lm.recv_cells)):
            sbuf = torch.from_numpy(np.concatenate([hc[lm.send_cells[p]], ue[lm.send_edges[p]]]))
            rbuf = torch.empty(len(lm.recv_cells[p]) + len(lm.recv_edges[p]), dtype=torch.float64)
            bufs[p] = rbuf
            reqs.append(dist.isend(sbuf, p))
            reqs.append(dist.irecv(rbuf, p))
        for r in reqs:
            r.wait()
        for p, rbuf in bufs.items():
            v = rbuf.numpy()
            nc = len(lm.recv_cells[p])
            hc[lm.recv_cells[p]] = v[:nc]
            ue[lm.recv_edges[p]] = v[nc:]
        ok_halo = bits_equal(hc[:-1], field_c[lm.cells]) and bits_equal(ue[:-1], field_e[lm.edges])
        # per-rank evaluation on the exchanged state vs the global oracle
        dh_g = np.zeros(wl.mesh.n_cells)
        du_g = np.zeros(wl.mesh.n_edges)
        h = 1000.0 + field_c
        u = field_e
        o.eval(h, u, kMaskAll, dh_g, du_g)
        lo = Oracle(lm.as_mesh(), lm.gather_cells(wl.b), lm.gather_vertices(wl.f), wl.gravity)
        hl = 1000.0 + hc
        hl[-1] = 1.0
        ul = ue.copy()
        ul[-1] = 0.0
        dh = np.zeros(lm.n_cells)
        du = np.zeros(lm.n_edges)
        cells = np.arange(lm.n_owned_cells)
        edges = np.arange(lm.n_owned_edges)
        lo.tendencies(hl, ul, cells, edges, dh, du)
        ok_eval = bits_equal(dh[cells], dh_g[lm.cells[cells]]) and \
            bits_equal(du[edges], du_g[lm.edges[edges]])
        q.put((rank, bool(ok_halo), bool(ok_eval)))
    finally:
        dist.destroy_process_group()


def _read_sets(lm, lo):
    """h-read cells and u-read edges of the oracle's last local evaluation
    (operators.cpp:61-86 over its closure lists): the per-mask halo
    restriction keeps exactly the halo entries in these sets."""
    m = lm.as_mesh()
    flux, _, kcells, verts = (lo.last_closure(k) for k in range(4))
    cells = np.zeros(m.n_cells, bool)
    edges = np.zeros(m.n_edges, bool)
    cells[m.vertex_cells[verts].ravel()] = True
    edges[m.vertex_edges[verts].ravel()] = True
    for i in kcells:
        edges[m.cell_edges[m.cell_offset[i]:m.cell_offset[i + 1]]] = True
    edges[flux] = True
    cells[m.edge_cells[flux].ravel()] = True
    return cells, edges


def _gloo_restricted_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2106_07154_b200.api import MASK_SUB
    from paper_2106_07154_b200.dist import swap_needs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = W.small_sphere(4, seed=5, cap_deg=30.0)
        o, (cl, cs, el) = _labels(wl)
        groups = o.groups()
        lay = DistributedLayout(wl.mesh, cl, cs, el, world)
        lm = lay.locals[rank]
        rng = np.random.default_rng(2)
        h = 1000.0 + rng.normal(size=wl.mesh.n_cells)
        u = rng.normal(size=wl.mesh.n_edges)
        results = []
        for mask in (kMaskAll, int(MASK_SUB)):
            in_c = np.zeros(wl.mesh.n_cells, bool)
            in_e = np.zeros(wl.mesh.n_edges, bool)
            for g in range(6):
                if mask >> g & 1:
                    in_c[groups[g]] = True
            for g in range(5):
                if mask >> (6 + g) & 1:
                    in_e[groups[6 + g]] = True
            cells = np.flatnonzero(in_c[lm.cells[:lm.n_owned_cells]]).astype(np.int32)
            edges = np.flatnonzero(in_e[lm.edges[:lm.n_owned_edges]]).astype(np.int32)
            lo = Oracle(lm.as_mesh(), lm.gather_cells(wl.b), lm.gather_vertices(wl.f), wl.gravity)
            # closure of this rank's outputs (values irrelevant here)
            lo.tendencies(np.ones(lm.n_cells) * 1000.0, np.zeros(lm.n_edges), cells, edges,
                          np.zeros(lm.n_cells), np.zeros(lm.n_edges))
            rc_, re_ = _read_sets(lm, lo)
            peers = sorted(set(lm.send_cells) | set(lm.recv_cells))
            needs = {}
            for p in peers:
                rl = np.concatenate([rc_[lm.recv_cells[p]], re_[lm.recv_edges[p]]])
                needs[p] = np.flatnonzero(rl).astype(np.int32)
            give = swap_needs(rank, world, needs)
            # restricted exchange; everything not exchanged stays NaN
            hc = np.full(lm.n_cells, np.nan)
            ue = np.full(lm.n_edges, np.nan)
            hc[:lm.n_owned_cells] = h[lm.cells[:lm.n_owned_cells]]
            ue[:lm.n_owned_edges] = u[lm.edges[:lm.n_owned_edges]]
            reqs, bufs = [], {}
            for p in peers:
                full = np.concatenate([hc[lm.send_cells[p]], ue[lm.send_edges[p]]])
                sbuf = torch.from_numpy(np.ascontiguousarray(full[give[p]]))
                rbuf = torch.empty(len(needs[p]), dtype=torch.float64)
                bufs[p] = rbuf
                reqs.append(dist.isend(sbuf, p))
                reqs.append(dist.irecv(rbuf, p))
            for r in reqs:
                r.wait()
            for p, rbuf in bufs.items():
                nc = len(lm.recv_cells[p])
                pos = needs[p]
                v = rbuf.numpy()
                hc[lm.recv_cells[p][pos[pos < nc]]] = v[pos < nc]
                ue[lm.recv_edges[p][pos[pos >= nc] - nc]] = v[pos >= nc]
            hc[-1] = 1.0
            ue[-1] = 0.0
            dh = np.zeros(lm.n_cells)
            du = np.zeros(lm.n_edges)
            lo.tendencies(hc, ue, cells, edges, dh, du)
            dh_g = np.zeros(wl.mesh.n_cells)
            du_g = np.zeros(wl.mesh.n_edges)
            o.eval(h, u, mask, dh_g, du_g)
            n_needed = sum(len(v) for v in needs.values())
            n_full = sum(len(lm.recv_cells[p]) + len(lm.recv_edges[p]) for p in peers)
            results.append((bool(bits_equal(dh[cells], dh_g[lm.cells[cells]])
                                 and bits_equal(du[edges], du_g[lm.edges[edges]])),
                            n_needed, n_full))
        q.put((rank, results))
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_restricted_halos():
    """Per-mask halo restriction: each rank exchanges only
    the halo entries its masked evaluation reads (positions swapped with
    dist.swap_needs over gloo); NaN elsewhere; results stay bitwise."""
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_restricted_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    for _, results in res:
        (ok_all, n_all, full), (ok_sub, n_sub, _) = results
        assert ok_all and ok_sub
        assert n_sub < n_all <= full


def test_gloo_two_rank_halo_exchange_and_evaluation():
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] for r in res), "halo values differ from the owners' values"
    assert all(r[2] for r in res), "rank evaluation differs from the global oracle"

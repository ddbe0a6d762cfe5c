"""Multi-rank device path on one GPU: N rank contexts (local meshes, owned
outputs, halo plans) stepped in lockstep by an in-process group whose halo
exchange is device copies -- the same pack/unpack and schedule as the NCCL
transport, without kernels that wait on one another.  Results must equal the
single-context path and the oracle bitwise (acceptance.cpp:205-244 analogue:
ranks bitwise = serial)."""
import numpy as np
import pytest

from helpers import bits_equal
from oracle.oracle import Oracle
from paper_2106_07154_b200 import workloads as W
from paper_2106_07154_b200.api import LTS3_MASKS, MASK_SUB, Scheme, kMaskAll
from paper_2106_07154_b200.dist import CudaGroup, DistributedLayout, RankContext

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_ranks", [2, 3, 4])
@pytest.mark.parametrize("scheme", [Scheme.LTS3, Scheme.RK4, Scheme.LTS2])
def test_group_ranks_bitwise_equal_oracle(n_ranks, scheme):
    wl = W.small_sphere(5, seed=23, cap_deg=25.0)
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, wl.width)
    cl, cs, el = o.labels()
    dt = wl.dt if scheme in (Scheme.LTS3, Scheme.LTS2) else wl.dt / wl.M
    n = 4
    h_ref, u_ref, _ = o.step(int(scheme), wl.h, wl.u, 0.0, dt, wl.M, n)
    lay = DistributedLayout(wl.mesh, cl, cs, el, n_ranks)
    ranks = [RankContext(lay, r, wl.b, wl.f, wl.gravity) for r in range(n_ranks)]
    for rc in ranks:
        rc.upload(wl.h, wl.u)
    grp = CudaGroup(ranks)
    grp.advance(scheme, dt, wl.M, n)
    h = np.full(wl.mesh.n_cells, np.nan)
    u = np.full(wl.mesh.n_edges, np.nan)
    for rc in ranks:
        rc.download_owned(h, u)
    assert bits_equal(h, h_ref) and bits_equal(u, u_ref)
    # the per-rank ledgers add up to the serial one
    c_ref, e_ref, _ = o.ledger()
    c = sum(rc.ctx.ledger().cell_evals for rc in ranks)
    e = sum(rc.ctx.ledger().edge_evals for rc in ranks)
    assert np.array_equal(c, c_ref) and np.array_equal(e, e_ref)


def test_planar_group_c1():
    wl = W.config1(n_steps=10)
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, wl.width)
    cl, cs, el = o.labels()
    h_ref, u_ref, _ = o.step(int(Scheme.LTS3), wl.h, wl.u, 0.0, wl.dt, wl.M, wl.n_steps)
    lay = DistributedLayout(wl.mesh, cl, cs, el, 4)
    ranks = [RankContext(lay, r, wl.b, wl.f, wl.gravity) for r in range(4)]
    for rc in ranks:
        rc.upload(wl.h, wl.u)
    CudaGroup(ranks).advance(Scheme.LTS3, wl.dt, wl.M, wl.n_steps)
    h = np.full(wl.mesh.n_cells, np.nan)
    u = np.full(wl.mesh.n_edges, np.nan)
    for rc in ranks:
        rc.download_owned(h, u)
    assert bits_equal(h, h_ref) and bits_equal(u, u_ref)


@pytest.mark.parametrize("n_ranks", [2, 4])
@pytest.mark.parametrize("scheme", [Scheme.LTS3, Scheme.LTS2, Scheme.RK4])
def test_group_restricted_halos_bitwise(n_ranks, scheme):
    """Per-mask halo restriction: exchanging only the halo
    entries each evaluation reads (plus the coarse-stage refresh) keeps every
    rank bitwise equal to the oracle; the substep exchange is much smaller
    than the full halo."""
    wl = W.small_sphere(5, seed=23, cap_deg=25.0)
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, wl.width)
    cl, cs, el = o.labels()
    dt = wl.dt if scheme in (Scheme.LTS3, Scheme.LTS2) else wl.dt / wl.M
    h_ref, u_ref, _ = o.step(int(scheme), wl.h, wl.u, 0.0, dt, wl.M, 4)
    lay = DistributedLayout(wl.mesh, cl, cs, el, n_ranks)
    ranks = [RankContext(lay, r, wl.b, wl.f, wl.gravity) for r in range(n_ranks)]
    grp = CudaGroup(ranks)
    full = sum(sum(len(v) for v in rc.lm.recv_cells.values()) +
               sum(len(v) for v in rc.lm.recv_edges.values()) for rc in ranks)
    sub = sum(sum(len(v) for v in rc.halo_needs(int(MASK_SUB)).values()) for rc in ranks)
    assert 0 < sub < full / 2
    grp.restrict_halos(LTS3_MASKS + [kMaskAll])
    for rc in ranks:
        rc.upload(wl.h, wl.u)
    grp.advance(scheme, dt, wl.M, 4)
    h = np.full(wl.mesh.n_cells, np.nan)
    u = np.full(wl.mesh.n_edges, np.nan)
    for rc in ranks:
        rc.download_owned(h, u)
    assert bits_equal(h, h_ref) and bits_equal(u, u_ref)


@pytest.mark.parametrize("overlap", ["2", "1", "0"])
@pytest.mark.parametrize("fork", ["1", "0"])
@pytest.mark.parametrize("n_ranks,M", [(2, 4), (3, 2), (4, 4)])
def test_group_concurrent_coarse_step_bitwise(fork, overlap, n_ranks, M, monkeypatch):
    """The coarse stage on its own stream with its own (restricted) halo
    exchange, concurrent with the substeps and their exchanges, on every
    rank; and every other exchange on a side stream while the interior
    outputs evaluate (MSWM_OVERLAP=1: steps 1 and 2, 2: every evaluation;
    the boundary outputs after the halo lands): bitwise equal to the oracle over several coarse steps, and to
    the sequential schedule (MSWM_FORK=0, MSWM_OVERLAP=0)."""
    monkeypatch.setenv("MSWM_FORK", fork)
    monkeypatch.setenv("MSWM_OVERLAP", overlap)
    wl = W.small_sphere(6, seed=41, cap_deg=25.0, M=M)
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, wl.width)
    cl, cs, el = o.labels()
    h_ref, u_ref, _ = o.step(int(Scheme.LTS3), wl.h, wl.u, 0.0, wl.dt, M, 3)
    lay = DistributedLayout(wl.mesh, cl, cs, el, n_ranks)
    ranks = [RankContext(lay, r, wl.b, wl.f, wl.gravity) for r in range(n_ranks)]
    grp = CudaGroup(ranks)
    grp.restrict_halos(LTS3_MASKS + [kMaskAll])
    for rc in ranks:
        rc.upload(wl.h, wl.u)
    grp.advance(Scheme.LTS3, wl.dt, M, 3)
    for rc in ranks:
        assert rc.ctx.concurrent_coarse() == (1 if fork == "1" else 0)
    h = np.full(wl.mesh.n_cells, np.nan)
    u = np.full(wl.mesh.n_edges, np.nan)
    for rc in ranks:
        rc.download_owned(h, u)
    assert bits_equal(h, h_ref) and bits_equal(u, u_ref)


@pytest.mark.parametrize("scheme", [Scheme.LTS3, Scheme.RK4])
def test_group_over_nccl_loopback_bitwise(scheme):
    """The halo copies of a 3-rank group as NCCL send/recv (to self, over
    one-rank communicators: the NCCL transport's calls, buffers and graph
    capture on one GPU), with the concurrent coarse step on the second
    communicator and the interior / boundary overlap: bitwise the oracle."""
    wl = W.small_sphere(6, seed=43, cap_deg=25.0)
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, wl.width)
    cl, cs, el = o.labels()
    dt = wl.dt if scheme == Scheme.LTS3 else wl.dt / wl.M
    h_ref, u_ref, _ = o.step(int(scheme), wl.h, wl.u, 0.0, dt, wl.M, 3)
    lay = DistributedLayout(wl.mesh, cl, cs, el, 3)
    ranks = [RankContext(lay, r, wl.b, wl.f, wl.gravity) for r in range(3)]
    grp = CudaGroup(ranks)
    grp.use_nccl_loopback()
    grp.restrict_halos(LTS3_MASKS + [kMaskAll])
    for rc in ranks:
        rc.upload(wl.h, wl.u)
    grp.advance(scheme, dt, wl.M, 3)
    if scheme == Scheme.LTS3:
        assert all(rc.ctx.concurrent_coarse() == 1 for rc in ranks)
    h = np.full(wl.mesh.n_cells, np.nan)
    u = np.full(wl.mesh.n_edges, np.nan)
    for rc in ranks:
        rc.download_owned(h, u)
    assert bits_equal(h, h_ref) and bits_equal(u, u_ref)


@pytest.mark.parametrize("n_ranks", [2, 5, 8])
def test_device_halo_plan_equals_host(n_ranks):
    """The partition's halo plan computed on the device (mswm_cuda_halo_reach:
    2-hop reach bit sets of every rank at once, partition.cpp:355-392) equals
    the host computation, and so do the local meshes built from it."""
    from paper_2106_07154_b200.api import CudaContext
    from paper_2106_07154_b200.partition import halo_reach, partition_cells
    wl = W.small_sphere(6, seed=47, cap_deg=20.0)
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, wl.width)
    cl, cs, el = o.labels()
    order = wl.mesh.locality_order()
    roc = partition_cells(order, cl, n_ranks)
    ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, order="hilbert")
    dev = halo_reach(wl.mesh, roc, n_ranks, ctx)
    host = halo_reach(wl.mesh, roc, n_ranks)
    for a, b in zip(dev, host):
        assert np.array_equal(a, b)
    la = DistributedLayout(wl.mesh, cl, cs, el, n_ranks, order=order, ctx=ctx)
    lb = DistributedLayout(wl.mesh, cl, cs, el, n_ranks, order=order)
    for x, y in zip(la.locals, lb.locals):
        assert np.array_equal(x.cells, y.cells) and np.array_equal(x.edges, y.edges)
        assert all(np.array_equal(x.tables[k], y.tables[k]) for k in x.tables)
        assert {q: v.tolist() for q, v in x.send_cells.items()} == \
            {q: v.tolist() for q, v in y.send_cells.items()}


@pytest.mark.parametrize("n_ranks", [1, 3, 8])
def test_device_partition_equals_host(n_ranks):
    """The partition computed on the device (mswm_cuda_partition: class-keyed
    order-preserving compaction of the sweep, partition.cpp:219-231; edge
    ownership, :338-353) equals partition_cells / edge_owner on the host, on
    the region-major and the input numbering; bad arguments are usage errors."""
    from paper_2106_07154_b200.api import CudaContext, UsageError
    from paper_2106_07154_b200.partition import edge_owner, partition_cells, partition_device
    for wl in [W.small_sphere(6, seed=47, cap_deg=20.0), W.config1(n_steps=1)]:
        o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
        o.set_regions(wl.fine_mask, wl.width)
        cl, cs, el = o.labels()
        order = wl.mesh.locality_order()
        roc = partition_cells(order, cl, n_ranks)
        own = edge_owner(wl.mesh, cl, el, roc)
        for layout in ["regions", "input"]:
            ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, order=layout,
                              fine_mask=wl.fine_mask)
            ctx.make_regions(wl.fine_mask, wl.width)
            droc, down = partition_device(ctx, order, n_ranks)
            assert np.array_equal(droc, roc) and np.array_equal(down, own)
            # every class split evenly
            for k in range(3):
                sel = np.isin(cl, [0] if k == 0 else ([3] if k == 1 else [1, 2]))
                cnt = np.bincount(droc[sel], minlength=n_ranks)
                assert cnt.max() - cnt.min() <= 1
        with pytest.raises(UsageError):
            ctx.partition(np.concatenate([order[:-1], order[:1]]), n_ranks)  # not a permutation
        with pytest.raises(UsageError):
            ctx.partition(order, 0)
    lay = DistributedLayout(wl.mesh, cl, cs, el, n_ranks, order=order,
                            partition=partition_device(ctx, order, n_ranks))
    ref = DistributedLayout(wl.mesh, cl, cs, el, n_ranks, order=order)
    for x, y in zip(lay.locals, ref.locals):
        assert np.array_equal(x.cells, y.cells) and np.array_equal(x.edges, y.edges)


@pytest.mark.parametrize("n_ranks,restrict", [(2, True), (3, False), (4, True)])
@pytest.mark.parametrize("scheme", [Scheme.LTS3, Scheme.RK4, Scheme.LTS2])
def test_group_over_peer_stores_bitwise(scheme, n_ranks, restrict):
    """The peer-store transport inside a group (k_push stores into the
    neighbours' double-buffered regions and raises their flags, k_wait_unpack
    consumes them; both channels, graph replays over several steps so both
    buffer halves and the sequence counters cycle): bitwise the oracle."""
    wl = W.small_sphere(6, seed=47, cap_deg=25.0)
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, wl.width)
    cl, cs, el = o.labels()
    dt = wl.dt if scheme in (Scheme.LTS3, Scheme.LTS2) else wl.dt / wl.M
    h_ref, u_ref, _ = o.step(int(scheme), wl.h, wl.u, 0.0, dt, wl.M, 5)
    lay = DistributedLayout(wl.mesh, cl, cs, el, n_ranks)
    ranks = [RankContext(lay, r, wl.b, wl.f, wl.gravity) for r in range(n_ranks)]
    grp = CudaGroup(ranks)
    if restrict:
        grp.restrict_halos(LTS3_MASKS + [kMaskAll])
    grp.use_peer_stores()
    for rc in ranks:
        rc.upload(wl.h, wl.u)
    grp.advance(scheme, dt, wl.M, 2)
    grp.advance(scheme, dt, wl.M, 3)
    if scheme == Scheme.LTS3 and restrict:
        assert all(rc.ctx.concurrent_coarse() == 1 for rc in ranks)
    h = np.full(wl.mesh.n_cells, np.nan)
    u = np.full(wl.mesh.n_edges, np.nan)
    for rc in ranks:
        rc.download_owned(h, u)
    assert bits_equal(h, h_ref) and bits_equal(u, u_ref)
    # back to device copies: the same group keeps stepping (graphs recaptured)
    grp.use_peer_stores(False)
    h2_ref, u2_ref, _ = o.step(int(scheme), h_ref, u_ref, 0.0, dt, wl.M, 1)
    grp.advance(scheme, dt, wl.M, 1)
    for rc in ranks:
        rc.download_owned(h, u)
    assert bits_equal(h, h2_ref) and bits_equal(u, u2_ref)


def test_peer_stores_across_processes():
    """Two processes on one GPU: each rank maps the other's arena through CUDA
    IPC (handles and tables over gloo), stores its owned values into it and
    raises the flag; after a host barrier each unpacks what the other stored
    (no kernel ever waits on another process)."""
    import os
    import socket
    import subprocess
    import sys
    from pathlib import Path
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    root = Path(__file__).resolve().parents[1]
    cmd = ["timeout", "600", sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(root / "tests" / "peer_ipc_worker.py")]
    env = dict(os.environ, PYTHONPATH=f"{root}:{root / 'tests'}")
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=root)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "PEER_IPC_OK rank 0" in out.stdout and "PEER_IPC_OK rank 1" in out.stdout


def test_peer_stores_silent_neighbour_is_an_error(monkeypatch):
    """A neighbour that never raises its flag ends the bounded wait with an
    error naming it (no device hang); once it has pushed, the same wait
    passes and delivers its values."""
    from paper_2106_07154_b200.api import CudaError, State
    monkeypatch.setenv("MSWM_PEER_TIMEOUT_MS", "200")
    wl = W.small_sphere(4, seed=3, cap_deg=25.0)
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, wl.width)
    lay = DistributedLayout(wl.mesh, *o.labels(), 2)
    ranks = [RankContext(lay, r, wl.b, wl.f, wl.gravity) for r in range(2)]
    grp = CudaGroup(ranks)
    grp.use_peer_stores()
    for rc in ranks:
        lm = rc.lm
        hp, up = lm.gather_cells(wl.h), lm.gather_edges(wl.u)
        hp[lm.n_owned_cells:-1] = np.nan
        up[lm.n_owned_edges:-1] = np.nan
        rc.ctx.upload(State(hp, up, 0.0))
    ranks[0].peer_exchange(0)
    with pytest.raises(CudaError, match="rank 1 did not signal"):
        ranks[0].peer_exchange(1)
    ranks[1].peer_exchange(0)
    ranks[0].peer_exchange(1)
    ranks[1].peer_exchange(1)
    for rc in ranks:
        st = rc.ctx.download()
        assert bits_equal(st.h, rc.lm.gather_cells(wl.h)) and bits_equal(st.u, rc.lm.gather_edges(wl.u))


def test_peer_stores_wait_then_push(monkeypatch):
    """The wait really waits: rank 0's wait + unpack is enqueued first and polls
    its flag while rank 1's push is launched afterwards on rank 1's own stream
    (one block each on an idle device; the poll is bounded, so a failure to
    overlap is an error, never a hang); the values stored during the poll are
    the ones unpacked."""
    from paper_2106_07154_b200.api import State
    monkeypatch.setenv("MSWM_PEER_TIMEOUT_MS", "5000")
    wl = W.small_sphere(4, seed=9, cap_deg=25.0)
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, wl.width)
    lay = DistributedLayout(wl.mesh, *o.labels(), 2)
    ranks = [RankContext(lay, r, wl.b, wl.f, wl.gravity) for r in range(2)]
    grp = CudaGroup(ranks)
    grp.use_peer_stores()
    for rnd in range(4):
        scale = 1.0 + rnd
        for rc in ranks:
            lm = rc.lm
            hp, up = lm.gather_cells(wl.h) * scale, lm.gather_edges(wl.u) * scale
            hp[lm.n_owned_cells:-1] = np.nan
            up[lm.n_owned_edges:-1] = np.nan
            rc.ctx.upload(State(hp, up, 0.0))
        ranks[0].peer_exchange(0)      # rank 0's values and flag are out
        ranks[0].peer_exchange(2)      # enqueued: polls for rank 1's flag
        ranks[1].peer_exchange(0)      # arrives while rank 0 polls
        ranks[0].ctx.sync()            # raises if the wait ran out of budget
        ranks[1].peer_exchange(1)
        for rc in ranks:
            st = rc.ctx.download()
            assert bits_equal(st.h, rc.lm.gather_cells(wl.h) * scale)
            assert bits_equal(st.u, rc.lm.gather_edges(wl.u) * scale)


@pytest.mark.parametrize("scheme,n_ranks", [(Scheme.LTS3, 3), (Scheme.RK4, 2), (Scheme.LTS2, 4),
                                            (Scheme.LTS3, 4)])
def test_peer_stores_asynchronous_ranks_bitwise(scheme, n_ranks, monkeypatch):
    """Every rank steps by itself -- its own stream, its own step graph, launched
    without waiting for the others, as one process per GPU would -- and only
    the peer-store flags order the halo exchanges (both channels, double
    buffering, sequence counters across graph replays).  Small meshes on an
    idle device, so the ranks' kernels are co-resident; the polls are bounded,
    so a protocol error would be an error, not a hang.  Bitwise the oracle."""
    monkeypatch.setenv("MSWM_PEER_TIMEOUT_MS", "20000")
    wl = W.small_sphere(5, seed=53, cap_deg=25.0)
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, wl.width)
    dt = wl.dt if scheme in (Scheme.LTS3, Scheme.LTS2) else wl.dt / wl.M
    h_ref, u_ref, _ = o.step(int(scheme), wl.h, wl.u, 0.0, dt, wl.M, 5)
    lay = DistributedLayout(wl.mesh, *o.labels(), n_ranks)
    ranks = [RankContext(lay, r, wl.b, wl.f, wl.gravity) for r in range(n_ranks)]
    grp = CudaGroup(ranks)                       # only to wire the arenas in-process
    grp.restrict_halos(LTS3_MASKS + [kMaskAll])
    grp.use_peer_stores()
    for rc in ranks:
        rc.upload(wl.h, wl.u)
        # plans and the step graph first: building them frees device memory, which
        # on this one shared device would wait for the other ranks' polling kernels
        rc.ctx.advance(scheme, dt, wl.M, 0)
    for n in (2, 3):
        for rc in ranks:                         # no rank waits for another on the host
            rc.ctx.advance(scheme, dt, wl.M, n, sync=False)
        for rc in ranks:
            rc.ctx.sync()
    if scheme == Scheme.LTS3:
        assert all(rc.ctx.concurrent_coarse() == 1 for rc in ranks)
    h = np.full(wl.mesh.n_cells, np.nan)
    u = np.full(wl.mesh.n_edges, np.nan)
    for rc in ranks:
        rc.download_owned(h, u)
    assert bits_equal(h, h_ref) and bits_equal(u, u_ref)

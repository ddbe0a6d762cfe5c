"""Binary workload store (store.py) and the rank-local multi-GPU setup built
on it (dist.layout_from_store): CPU tests, world_size-2 gloo."""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

from helpers import bits_equal
from oracle.oracle import Oracle
from paper_2106_07154_b200 import store
from paper_2106_07154_b200 import workloads as W
from paper_2106_07154_b200.dist import DistributedLayout, layout_from_store


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _labels(wl):
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, wl.width)
    return o.labels()


@pytest.mark.parametrize("which", ["c1", "sphere"])
def test_store_round_trip(tmp_path, which):
    wl = W.config1(n_steps=3) if which == "c1" else W.small_sphere(4, seed=3)
    extra = {"order": wl.mesh.locality_order(), "tag": np.arange(5, dtype=np.int64)}
    store.save_workload(tmp_path / "s", wl, extra)
    for mmap in (True, False):
        wl2, ex2 = store.load_workload(tmp_path / "s", mmap=mmap, verify=True)
        assert wl2.mesh.digest() == wl.mesh.digest()
        for n in ("h", "u", "b", "f"):
            assert bits_equal(getattr(wl2, n), getattr(wl, n))
        assert np.array_equal(wl2.fine_mask, wl.fine_mask)
        assert (wl2.dt, wl2.M, wl2.gravity, wl2.width, wl2.name) == \
            (wl.dt, wl.M, wl.gravity, wl.width, wl.name)
        assert np.array_equal(ex2["order"], extra["order"]) and np.array_equal(ex2["tag"], extra["tag"])
        d = wl2.mesh.desc()  # memory-mapped tables pass the boundary's checks
        assert d.n_cells == wl.mesh.n_cells
    # the oracle reads the mapped tables exactly like the in-memory ones
    wl2, _ = store.load_workload(tmp_path / "s")
    o1 = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o2 = Oracle(wl2.mesh, np.array(wl2.b), np.array(wl2.f), wl2.gravity)
    dh1, du1 = np.zeros(wl.mesh.n_cells), np.zeros(wl.mesh.n_edges)
    dh2, du2 = np.zeros(wl.mesh.n_cells), np.zeros(wl.mesh.n_edges)
    o1.eval(wl.h, wl.u, 0x7FF, dh1, du1)
    o2.eval(np.array(wl2.h), np.array(wl2.u), 0x7FF, dh2, du2)
    assert bits_equal(dh1, dh2) and bits_equal(du1, du2)


def test_store_rejects_damage(tmp_path):
    wl = W.config1(n_steps=1)
    store.save_workload(tmp_path / "s", wl)
    np.save(tmp_path / "s" / "mesh" / "edge_len.npy", np.zeros(3))
    with pytest.raises(ValueError):
        store.load_workload(tmp_path / "s")


def _shard_worker(rank, world, port, root, q, with_reach=False):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if rank == 0:
            # what dist.publish_store does, with the oracle's labels standing
            # in for the device labelling (no GPU here)
            wl = W.small_sphere(5, seed=21, cap_deg=25.0)
            cl, cs, el = _labels(wl)
            extra = {"cell_label": cl, "cell_sub": cs, "edge_label": el,
                     "order": wl.mesh.locality_order()}
            if with_reach:  # what publish_store adds from the device
                from paper_2106_07154_b200.partition import halo_reach, partition_cells
                roc = partition_cells(extra["order"], cl, world)
                cr, er, vr = halo_reach(wl.mesh, roc, world)
                extra.update({"rank_of_cell": roc, "cell_reach": cr, "edge_reach": er,
                              "vertex_reach": vr})
            store.save_workload(root, wl, extra)
        dist.barrier()
        wl, lay = layout_from_store(root, rank, world)
        lm = lay.locals[rank]
        others_unbuilt = all(lay.locals[r] is None for r in range(world) if r != rank)
        q.put((rank, others_unbuilt, lm.cells.tobytes(), lm.edges.tobytes(),
               {k: v.tobytes() for k, v in lm.tables.items()},
               {p: v.tobytes() for p, v in lm.send_cells.items()},
               {p: v.tobytes() for p, v in lm.recv_edges.items()}))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("with_reach", [False, True])
def test_rank_local_setup_from_store_gloo(tmp_path, with_reach):
    """world_size 2: rank 0 publishes the store, each rank builds only its
    own local mesh + halo plan from the shared maps; both equal the
    single-process DistributedLayout."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    root = str(tmp_path / "store")
    ps = [ctx.Process(target=_shard_worker, args=(r, world, port, root, q, with_reach))
          for r in range(world)]
    for p in ps:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    wl = W.small_sphere(5, seed=21, cap_deg=25.0)
    cl, cs, el = _labels(wl)
    ref = DistributedLayout(wl.mesh, cl, cs, el, world)
    for rank, others_unbuilt, cells, edges, tables, send_c, recv_e in got:
        assert others_unbuilt
        lm = ref.locals[rank]
        assert cells == lm.cells.tobytes() and edges == lm.edges.tobytes()
        assert tables == {k: v.tobytes() for k, v in lm.tables.items()}
        assert send_c == {p: v.tobytes() for p, v in lm.send_cells.items()}
        assert recv_e == {p: v.tobytes() for p, v in lm.recv_edges.items()}

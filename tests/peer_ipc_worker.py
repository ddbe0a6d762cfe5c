"""Worker of test_peer_stores_across_processes (2 processes, one GPU, gloo)."""
import os
import sys

import numpy as np
import torch.distributed as dist

from paper_2106_07154_b200 import workloads as W
from paper_2106_07154_b200.api import LTS3_MASKS, State, kMaskAll
from paper_2106_07154_b200.dist import DistributedLayout, RankContext
from oracle.oracle import Oracle


def main():
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    wl = W.small_sphere(5, seed=29, cap_deg=25.0)
    o = Oracle(wl.mesh, wl.b, wl.f, wl.gravity)
    o.set_regions(wl.fine_mask, wl.width)
    cl, cs, el = o.labels()
    lay = DistributedLayout(wl.mesh, cl, cs, el, ws)
    rc = RankContext(lay, rank, wl.b, wl.f, wl.gravity, device=0)
    rc.restrict_halos(LTS3_MASKS + [kMaskAll])   # several halos share the arena
    rc.init_peer()
    lm = rc.lm
    h = lm.gather_cells(wl.h)
    u = lm.gather_edges(wl.u)
    for rnd in range(3):                          # both buffer halves, rising sequence numbers
        hh, uu = h * (rnd + 1.0), u * (rnd + 1.0)
        hp, up = hh.copy(), uu.copy()
        hp[lm.n_owned_cells:-1] = np.nan          # halo copies poisoned (the last entry is the dummy)
        up[lm.n_owned_edges:-1] = np.nan
        rc.ctx.upload(State(hp, up, 0.0))
        rc.peer_exchange(0)                       # pack + store into the neighbour + signal
        dist.barrier()                            # host order: every store has landed
        rc.peer_exchange(1)                       # flags are up: no waiting on the device
        st = rc.ctx.download()
        assert np.array_equal(st.h.view(np.int64), hh.view(np.int64)), (rank, rnd)
        assert np.array_equal(st.u.view(np.int64), uu.view(np.int64)), (rank, rnd)
        dist.barrier()
    print(f"PEER_IPC_OK rank {rank}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python
"""Per-rank compute time of an N-way partition, measured on ONE B200.

    MSWM_HALO_DRYRUN=1 python scripts/rank_timing.py c4 8 [steps]

Partitions the workload exactly as the multi-GPU bench does (per-class
balanced Hilbert runs, 2-hop halos, per-mask restricted exchanges), creates
every rank's context on this one device, and times each rank stepping ALONE
(LTS3 coarse steps, CUDA events on its stream) with the halo transfers
skipped (MSWM_HALO_DRYRUN=1: pack and unpack kernels still run, the
NCCL send/recv is left out).  No kernels wait on other ranks.  Prints one
JSON line: single-context ms/step, per-rank ms/step, and the bytes each
exchange of each rank moves -- the inputs of the latency model in DESIGN.md
section 7 (results of the dry-run steps are not used).
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_07154_b200 import workloads as W  # noqa: E402
from paper_2106_07154_b200.api import (LTS3_MASKS, CudaContext, Scheme, State,  # noqa: E402
                                       kMaskAll)
from paper_2106_07154_b200.dist import DistributedLayout, RankContext  # noqa: E402


def time_steps(ctx, wl, steps):
    stream = torch.cuda.ExternalStream(ctx.stream_ptr())
    ctx.advance(Scheme.LTS3, wl.dt, wl.M, 3)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.advance(Scheme.LTS3, wl.dt, wl.M, steps, sync=False)
    e1.record(stream)
    torch.cuda.synchronize()
    ctx.sync()
    return e0.elapsed_time(e1) / steps


def main():
    if os.environ.get("MSWM_HALO_DRYRUN") != "1":
        raise SystemExit("set MSWM_HALO_DRYRUN=1 (timing aid: transfers skipped)")
    cfg, n = sys.argv[1], int(sys.argv[2])
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    t0 = time.time()
    wl = W.CONFIGS[cfg]()
    g = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, order="regions", fine_mask=wl.fine_mask,
                    interface_width=wl.width)
    rm = g.make_regions(wl.fine_mask, wl.width)
    g.upload(State(wl.h, wl.u, 0.0))
    t_single = time_steps(g, wl, steps)
    g.set_profiling(1)
    g.advance(Scheme.LTS3, wl.dt, wl.M, 2)
    ms1, nc1, ne1 = g.eval_profile()
    single_evals = {"ms": [round(float(x), 4) for x in ms1], "cells": [int(x) for x in nc1],
                    "edges": [int(x) for x in ne1]}
    g.close()
    del g
    lay = DistributedLayout(wl.mesh, rm.cell_label, rm.cell_sublabel, rm.edge_label, n)
    ranks = [RankContext(lay, r, wl.b, wl.f, wl.gravity, wl.width) for r in range(n)]
    masks = LTS3_MASKS + [kMaskAll]
    needs = {m: [rc.halo_needs(int(m)) for rc in ranks] for m in masks}
    for m in masks:
        for r, rc in enumerate(ranks):
            send = {q: needs[m][q].get(r, np.zeros(0, np.int32)) for q in needs[m][r]}
            rc.set_halo_mask(int(m), send, needs[m][r])
    per_rank, fork, evals = [], [], []
    for rc in ranks:
        rc.upload(wl.h, wl.u)
        per_rank.append(time_steps(rc.ctx, wl, steps))
        fork.append(rc.ctx.concurrent_coarse())
        # per-evaluation device times of one profiled step (events around
        # every evaluation: step 1, step 2, the 3M substeps, the coarse step)
        rc.ctx.set_profiling(1)
        rc.ctx.advance(Scheme.LTS3, wl.dt, wl.M, 2)
        ms, nc, ne = rc.ctx.eval_profile()
        evals.append({"ms": [round(float(x), 4) for x in ms], "cells": [int(x) for x in nc],
                      "edges": [int(x) for x in ne]})
        rc.ctx.set_profiling(0)
    # bytes received per exchange (8 B per value) per rank and mask, and peers
    xbytes = {hex(int(m)): [int(8 * sum(len(v) for v in needs[m][r].values())) for r in range(n)]
              for m in masks}
    xpeers = {hex(int(m)): [int(sum(1 for v in needs[m][r].values() if len(v))) for r in range(n)]
              for m in masks}
    print(json.dumps({
        "config": cfg, "n_ranks": n, "M": wl.M, "steps": steps, "single_ms_per_step": t_single,
        "single_evals": single_evals, "rank_ms_per_step": per_rank, "max_rank_ms": max(per_rank),
        "ideal_ms": t_single / n, "compute_efficiency": t_single / (n * max(per_rank)),
        "concurrent_coarse": fork, "evals_per_rank": evals, "owned_cells": [rc.lm.n_owned_cells for rc in ranks],
        "local_cells": [rc.lm.n_cells for rc in ranks],
        "recv_bytes_per_exchange": xbytes, "peers_per_exchange": xpeers,
        "setup_s": time.time() - t0}))


if __name__ == "__main__":
    main()

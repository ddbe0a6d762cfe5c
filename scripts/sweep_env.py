#!/usr/bin/env python
"""A/B sweep of create-time knobs (MSWM_* env) on one workload.

    python scripts/sweep_env.py c4 "MSWM_FLOW=0" "MSWM_FLOW_SLAB=16 MSWM_FLOW_LAG=500" ...

Builds the workload once, then per setting: a fresh context (env is read at
create), 3 warm-up coarse steps, 10 timed steps (CUDA events on the
library stream); prints ms/step and the largest evaluation's device time.
Development tool: bench.py is the reported measurement.
"""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_07154_b200 import workloads as W  # noqa: E402
from paper_2106_07154_b200.api import CudaContext, Scheme, State  # noqa: E402


def main():
    cfg = sys.argv[1]
    t0 = time.time()
    wl = W.CONFIGS[cfg]()
    print(f"{cfg}: {wl.mesh.n_cells} cells, built in {time.time() - t0:.1f}s", flush=True)
    steps = int(os.environ.get("SWEEP_STEPS", "10"))
    for setting in sys.argv[2:]:
        saved = dict(os.environ)
        for kv in setting.split():
            k, v = kv.split("=", 1)
            os.environ[k] = v
        try:
            ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, order="regions",
                              fine_mask=wl.fine_mask, interface_width=wl.width)
            ctx.make_regions(wl.fine_mask, wl.width)
            ctx.upload(State(wl.h, wl.u, 0.0))
            prof = int(os.environ.get("SWEEP_PROF", "1"))
            ctx.set_profiling(prof)
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
            ms = e0.elapsed_time(e1) / steps
            evms, evnc, evne = ctx.eval_profile() if prof else ([0.0] * 3, [0], [0])
            k = int(np.argmax(evne))
            print(f"{setting:40s} ms/step {ms:8.3f}  big-eval ms {evms[k]:.3f}  "
                  f"evals {' '.join(f'{x:.3f}' for x in evms[:16])}  kernels {ctx.kernels_per_step()}",
                  flush=True)
            ctx.close()
            del ctx
        except Exception as ex:  # keep sweeping
            print(f"{setting:40s} FAILED {ex!r}", flush=True)
        os.environ.clear()
        os.environ.update(saved)


if __name__ == "__main__":
    main()

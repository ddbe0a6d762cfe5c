#!/usr/bin/env python
"""LTS3 TRiSK shallow-water benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One "step" is one LTS3 coarse step (Stepper::lts_step(3, ...),
proj/src/integrators.cpp:412-575) over the whole synthetic mesh.  `value`
is whole-job edge-tendency evaluations per second (the WorkLedger unit,
proj/include/mswm/ledger.hpp:25-60) with the state resident in HBM; `e2e`
is the same metric through the drop-in C-ABI call a reference user makes
(upload h,u from pinned host memory, one coarse step, download h,u).  The
dominant kernel's roofline is one tendency evaluation (kernels A+B+C with
the fused stage update) timed with CUDA events inside the timed steps.
Under torchrun the mesh is partitioned across the ranks (strong scaling):
per-class balanced Hilbert partition, two-hop halos, NCCL point-to-point
halo exchange before every evaluation.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "LTS3 edge-tendency evals/s"
UNIT = "edge-evals/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def _rss_gb() -> float:
    try:
        with open("/proc/self/status") as fh:
            for line in fh:
                if line.startswith("VmRSS:"):
                    return int(line.split()[1]) / 2**20
    except OSError:
        pass
    return float("nan")


def start_rss_monitor(period: float = 10.0) -> None:
    """MSWM_BENCH_RSS=1: log this process's resident set every `period` s
    (host-memory diagnosis of the largest configurations)."""
    if os.environ.get("MSWM_BENCH_RSS") != "1":
        return

    def run():
        while True:
            log(f"[rss] {time.strftime('%H:%M:%S')} {_rss_gb():.1f} GB")
            time.sleep(period)

    threading.Thread(target=run, daemon=True).start()


# ---------------------------------------------------------------------------
# distributed plumbing

def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        if torch.cuda.is_available():
            # more ranks than GPUs only for the dry-run check (MSWM_HALO_DRYRUN=1)
            local %= torch.cuda.device_count()
        backend = os.environ.get("MSWM_DIST_BACKEND",
                                 "nccl" if torch.cuda.is_available() else "gloo")
        if backend == "nccl":
            torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_sum(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def allreduce_max(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# workload + algorithmic bytes

def make_workload(name: str, level: int | None = None):
    from paper_2106_07154_b200 import workloads as W
    if level is not None and name in W.SPHERE_LEVEL:
        return W.CONFIGS[name](level=level)
    return W.CONFIGS[name]()


def bytes_per_eval(mesh):
    """B_E per edge evaluation and B_C per cell evaluation:
    B_E = 32 + 8 + 8 + 4 + 4 + 12*S + 64*(nV/nE), B_C = 36 + 4*deg."""
    S = mesh.n_stencil / mesh.n_edges
    deg = mesh.n_ring / mesh.n_cells
    BE = 32 + 8 + 8 + 4 + 4 + 12 * S + 64 * (mesh.n_vertices / mesh.n_edges)
    BC = 36 + 4 * deg
    return BE, BC


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md clocks line)

class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baselines (oracle/_ref = the unmodified reference)

class RefRunner:
    """The reference's own LTS3 path (oracle/_ref = unmodified proj/src):
    Stepper::lts_step(3) with SerialEvaluator (nranks=0) or ThreadedEvaluator
    over partition_multiconstraint + make_block_plan (nranks ranks).
    ``rm``: a reference VoronoiMesh already built (the reference arm's own
    builder); default: the workload's tables loaded into one."""

    def __init__(self, wl, nranks: int, rm=None):
        from oracle.oracle import RefEvaluator, RefMesh, RefRegions
        self.wl = wl
        self.rm = RefMesh.from_mesh(wl.mesh) if rm is None else rm
        self.rr = RefRegions(self.rm, wl.fine_mask, wl.width)
        self.ev = RefEvaluator(self.rm, self.rr, wl.b, wl.f, wl.gravity, nranks=nranks)
        self.h, self.u, self.t = wl.h, wl.u, 0.0

    def steps(self, n: int, scheme: int = 4, dt: float | None = None):
        """Run n steps (LTS3 coarse steps by default); returns (edge evals/s,
        s/step, edge evals/step)."""
        _, e0, s0 = self.ev.ledger()
        dt = self.wl.dt if dt is None else dt
        self.h, self.u, self.t, secs = self.ev.step(scheme, self.h, self.u, self.t, dt,
                                                    self.wl.M, n)
        _, e1, s1 = self.ev.ledger()
        per = int(e1.sum() - e0.sum()) // max(s1 - s0, 1)
        return per * n / secs, secs / n, per


def host_info() -> dict:
    """CPU model, logical CPUs and RAM of this box."""
    model, mem = None, None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemTotal:"):
                    mem = round(int(line.split()[1]) / 2**20, 1)
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "threads_available": cpu_threads(),
            "ram_gb": mem}


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _mem_available() -> float:
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024.0
    except OSError:
        pass
    return float("inf")


def ref_ranks(wl, threads: int):
    """Rank count for the reference's ThreadedEvaluator that fits host RAM:
    it allocates full-size h/u buffers plus scratch per block, 3 blocks per
    rank (rank_pool.cpp:93-95), ~36 B per (cell + edge) per block (SURVEY.md
    §8(d)).  Returns (ranks, note); ranks 0 = SerialEvaluator, None = does
    not fit at all."""
    per_block = 36.0 * (wl.mesh.n_cells + wl.mesh.n_edges)
    avail = 0.5 * _mem_available()
    fit = int(avail // (3 * per_block))
    if threads > 1 and fit >= 2:
        r = min(threads, fit)
        return r, ("" if r == threads else
                   f"; {r} of {threads} threads: more ranks would exceed host RAM")
    if 3 * per_block <= avail:
        return 0, "; SerialEvaluator: ranks would exceed host RAM"
    return None, "reference needs more host RAM than this box has"


def loaded_repo_libraries() -> list:
    """Shared objects of this repo mapped into the process (/proc/self/maps)."""
    out = set()
    try:
        with open("/proc/self/maps") as fh:
            for line in fh:
                path = line.split()[-1]
                if path.endswith(".so") and str(ROOT) in path:
                    out.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(out)


def reference_workload(name: str, level: int | None = None):
    """The workload with its mesh built by the REFERENCE's own generator
    (build_voronoi_mesh(subdivide_icosahedron(L)), proj/src/mesh_build.cpp:
    185-366, via oracle/_ref) for the spherical configurations, so the
    reference arm maps no product library; its tables equal ours bitwise
    (tests/test_reference_arm.py).  The planar configurations have no
    reference generator (it is sphere-only): their tables come from our
    planar builder, the table adapter SURVEY.md §8(c) names."""
    from paper_2106_07154_b200 import workloads as W
    if name not in W.SPHERE_LEVEL:
        return W.CONFIGS[name](), None, "planar tables from the repo's builder (the reference has no planar generator)"
    from oracle.oracle import RefMesh
    level = level or W.SPHERE_LEVEL[name]
    t0 = time.time()
    rm = RefMesh.icosahedral(level, W.EARTH_RADIUS)
    mesh = rm.as_mesh()
    note = f"reference build_voronoi_mesh(subdivide_icosahedron({level})) in {time.time() - t0:.0f} s"
    return W.CONFIGS[name](mesh=mesh, level=level), rm, note


def run_reference_arm(args, ws, rank):
    """--impl reference: the reference's own CPU LTS3 path on this box's host
    cores, same config / metric / step count as the GPU arm.  Only oracle/_ref
    (the unmodified reference + its C shim) is loaded."""
    if rank != 0:
        return
    from oracle.oracle import ref_available
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    wl, rm, mesh_note = reference_workload(args.config, args.level)
    log(f"reference arm: {mesh_note}")
    threads = cpu_threads()
    # ThreadedEvaluator on every host thread (the reference's parallel path)
    # as far as host RAM allows
    best, note = ref_ranks(wl, threads)
    if best is None:
        print(json.dumps({"impl": "reference", "unavailable": f"{args.config}: {note}"}))
        return
    cores = max(1, best)
    runner = RefRunner(wl, best, rm)
    for _ in range(args.warmup):
        _, sps0, _ = runner.steps(1)
        log(f"reference {cores} threads: {sps0:.3f} s/step (warm-up)")
        if sps0 * args.steps > 1800:  # keep the arm's wall time bounded (C5)
            break
    n = args.steps if sps0 * args.steps <= 1800 else max(1, int(1800 / sps0))
    rate, sps, per = runner.steps(n)
    del runner
    # SerialEvaluator on one core: one coarse step
    serial = None
    if not args.no_serial and ref_ranks(wl, 1)[0] is not None:
        sr = RefRunner(wl, 0, rm)
        srate, ssps, _ = sr.steps(1)
        serial = {"edge_evals_per_s": srate, "s_per_step": ssps, "cores": 1,
                  "sample": "1 LTS3 coarse step, SerialEvaluator"}
        del sr
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": ws,
        "steps": n, "warmup": args.warmup, "ms_per_step": sps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(wl, args.config, ws),
        "coarse_steps_per_s": 1.0 / sps,
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{n} LTS3 coarse steps of {args.config} after {args.warmup} "
                                   f"warm-up, reference "
                                   f"{'SerialEvaluator' if best == 0 else f'ThreadedEvaluator {best} ranks'}"
                                   f"{note}; mesh: {mesh_note}",
                         "serial_1core": serial, "host": host_info()},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "repo_libraries_loaded": loaded_repo_libraries(),
    }
    print(json.dumps(line), flush=True)


def workload_config(wl, name, ws):
    m = wl.mesh
    return {"workload": f"{name.upper()} {wl.meta.get('mesh', '')}, LTS3 M={wl.M}, "
                        f"interface width {wl.width}",
            "n_cells": m.n_cells, "n_edges": m.n_edges, "n_vertices": m.n_vertices,
            "M": wl.M, "dt": wl.dt, "fine_cells": int(wl.fine_mask.sum()),
            "parallelism": (f"{ws} GPUs: class-balanced Hilbert partition, 2-hop halos, "
                            "NCCL p2p halo exchange before every evaluation") if ws > 1 else "1 GPU",
            "l2": "inputs larger than L2 (mesh tables + state > 126 MB)" if m.n_edges > 400000
            else "working set L2-resident (correctness config)"}


# ---------------------------------------------------------------------------

def run_ours(args, ws, rank, local):
    import torch
    # MSWM_HALO_DRYRUN=1 (checks of the multi-rank bench path on one GPU:
    # ranks step independently, halo transfers skipped, results invalid)
    dry_run = os.environ.get("MSWM_HALO_DRYRUN") == "1"
    from paper_2106_07154_b200.api import CudaContext, Scheme, State

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    t0 = time.time()
    setup = {}
    rc = None
    if ws == 1:
        wl = make_workload(args.config, args.level)
        setup["workload_s"] = time.time() - t0
        log(f"[rank {rank}] workload {args.config}: {wl.mesh.n_cells} cells, {wl.mesh.n_edges} edges, "
            f"built in {time.time() - t0:.1f}s")
        t1 = time.time()
        ctx = CudaContext(wl.mesh, wl.b, wl.f, wl.gravity, device=local, order=args.order,
                          fine_mask=wl.fine_mask, interface_width=wl.width)
        setup["context_s"] = time.time() - t1
        t1 = time.time()
        rm = ctx.make_regions(wl.fine_mask, wl.width)
        setup["regions_s"] = time.time() - t1
        log(f"[rank {rank}] groups {rm.group_sizes()} (host rss {_rss_gb():.1f} GB)")
        ctx.upload(State(wl.h, wl.u, 0.0))
        io_mesh = wl.mesh
    else:
        # partitioned (strong scaling).  Rank 0 alone builds the global mesh,
        # labels it on its device and publishes it as a binary store in
        # /dev/shm; every rank memory-maps the store (one page-cache copy per
        # node) and materialises only its own local mesh + halo plan.
        import torch.distributed as dist
        from paper_2106_07154_b200.dist import RankContext, layout_from_store, publish_store
        store_dir = Path(os.environ.get("MSWM_STORE_DIR", "/dev/shm")) / \
            f"mswm_bench_{args.config}_{os.environ.get('MASTER_PORT', '0')}"
        if rank == 0:
            wl0 = make_workload(args.config, args.level)
            log(f"[rank 0] workload {args.config}: {wl0.mesh.n_cells} cells, built in "
                f"{time.time() - t0:.1f}s")
            setup["workload_s"] = time.time() - t0
            t1 = time.time()
            publish_store(store_dir, wl0, device=local, n_ranks=ws)
            setup["publish_s"] = time.time() - t1
            del wl0
        barrier(ws)
        t1 = time.time()
        wl, lay = layout_from_store(store_dir, rank, ws)
        rc = RankContext(lay, rank, wl.b, wl.f, wl.gravity, wl.width, device=local)
        # MSWM_TRANSPORT=nccl (default): ncclSend / ncclRecv inside the step graph;
        # =peer: stores into the neighbours' IPC-mapped buffers + device flags
        transport = os.environ.get("MSWM_TRANSPORT", "nccl")
        if not dry_run and transport == "nccl":
            uid = [RankContext.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            rc.init_nccl(uid[0])
        # exchange only what each evaluation reads (setup-time position swap)
        from paper_2106_07154_b200.api import LTS3_MASKS, kMaskAll
        rc.restrict_halos(LTS3_MASKS + [kMaskAll])
        if not dry_run and transport == "peer":
            rc.init_peer()
        rc.upload(wl.h, wl.u)
        barrier(ws)
        if rank == 0:
            import shutil
            shutil.rmtree(store_dir, ignore_errors=True)
        ctx = rc.ctx
        io_mesh = rc.local_mesh
        setup["rank_local_s"] = time.time() - t1
        log(f"[rank {rank}] local mesh {rc.lm.n_cells} cells ({rc.lm.n_owned_cells} owned), "
            f"{len(lay.locals[rank].send_cells)} peers, set up in {time.time() - t1:.1f}s "
            f"(host rss {_rss_gb():.1f} GB)")
    ctx.set_profiling(2)  # events around the dominant (first full-mesh) evaluation only
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=local)

    # warm-up (also captures the step graph)
    t1 = time.time()
    ctx.advance(Scheme.LTS3, wl.dt, wl.M, max(args.warmup, 1))
    setup["plans_capture_warmup_s"] = time.time() - t1
    setup["total_s"] = time.time() - t0
    ctx.reset_ledger()

    clocks = Clocks(local)
    clocks.start()
    barrier(ws)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.advance(Scheme.LTS3, wl.dt, wl.M, args.steps, sync=False)
    e1.record(stream)
    torch.cuda.synchronize()
    ctx.sync()
    barrier(ws)
    ck = clocks.stop()
    ms_local = e0.elapsed_time(e1)
    ms = allreduce_max(ms_local, ws)
    lg = ctx.ledger()
    edge_per_step = allreduce_sum(lg.total_edge_evals(), ws) / args.steps
    cell_per_step = allreduce_sum(lg.total_cell_evals(), ws) / args.steps
    ms_step = ms / args.steps
    value = edge_per_step / (ms_step / 1e3)

    # roofline of the dominant kernel: the largest tendency evaluation of the
    # last timed step, timed by the events captured around it
    BE, BC = bytes_per_eval(wl.mesh)
    evms, evnc, evne = ctx.eval_profile()
    k = int(np.argmax(evne))
    alg = BE * evne[k] + BC * evnc[k]
    # the events sit inside the step graph, so they hold the last replay's
    # times: the timed region's last step, then the same graph replayed step by
    # step (events read after each) -- the kernel's average over these launches
    ev_samples = [float(evms[k])]
    for _ in range(max(args.steps - 1, 0)):
        ctx.advance(Scheme.LTS3, wl.dt, wl.M, 1)
        ev_samples.append(float(ctx.eval_profile()[0][k]))
    ctx.reset_ledger()
    ev_mean = float(np.mean(ev_samples))
    hbm, peak_kind = peaks()
    achieved = alg / (ev_mean / 1e3) / 1e9
    step_alg = BE * edge_per_step + BC * cell_per_step
    traffic = None
    tf = ROOT / "profiles" / f"traffic_{args.config}.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get("dram_bytes_per_launch")

    # e2e through the drop-in C ABI with pinned host buffers (the rank's
    # local arrays when partitioned)
    st0 = ctx.download()
    h_pin = torch.from_numpy(np.array(st0.h)).pin_memory()
    u_pin = torch.from_numpy(np.array(st0.u)).pin_memory()
    st = State(h_pin.numpy(), u_pin.numpy(), 0.0)
    ctx.set_profiling(False)
    ctx.upload(st)
    ctx.advance(Scheme.LTS3, wl.dt, wl.M, 1)  # graph for the unprofiled path
    ctx.download(st)
    n_e2e = max(3, min(args.steps, 20))
    barrier(ws)
    t = time.perf_counter()
    for _ in range(n_e2e):
        ctx.upload(st)
        ctx.advance(Scheme.LTS3, wl.dt, wl.M, 1)
        ctx.download(st)
    e2e_s = allreduce_max(time.perf_counter() - t, ws)
    e2e_value = edge_per_step * n_e2e / e2e_s
    io_bytes = int(allreduce_sum(8 * (io_mesh.n_cells + io_mesh.n_edges), ws))

    launches = ctx.kernels_per_step() * args.steps

    # the per-stage drop-in (mswm::CudaEvaluator under the reference's own
    # Stepper, one C-ABI eval() per stage): the 3M+3 eval calls of one LTS3
    # coarse step with pageable host arrays, as the reference issues them
    # (integrators.cpp:483-563); the reference's host-side stage combines
    # are not part of this number
    dropin = None
    if ws == 1:
        from paper_2106_07154_b200.api import (MASK_COARSE_ONLY, MASK_IF_COARSE, MASK_STEP1,
                                               MASK_SUB, CudaEvaluator)
        ev = CudaEvaluator(ctx)
        hh, uu = np.array(st0.h), np.array(st0.u)
        dh, du = np.zeros_like(hh), np.zeros_like(uu)
        seq = [MASK_STEP1, MASK_IF_COARSE] + [MASK_SUB] * (3 * wl.M) + [MASK_COARSE_ONLY]
        for m in dict.fromkeys(seq):  # first call per mask builds its plan / read set
            ev.eval(hh, uu, int(m), dh, du)
        n_di = 2
        t = time.perf_counter()
        for _ in range(n_di):
            for m in seq:
                ev.eval(hh, uu, int(m), dh, du)
        di_s = (time.perf_counter() - t) / n_di
        dropin = {"value": edge_per_step / di_s, "unit": UNIT, "ms_per_coarse_step": di_s * 1e3,
                  "eval_calls_per_step": len(seq),
                  "d2h_bytes_per_step": int(8 * (edge_per_step + cell_per_step)),
                  "note": "C-ABI eval() per stage with host arrays (inputs: the masked read set "
                          "only; outputs: the masked entries only); excludes the reference "
                          "Stepper's own host-side stage combines"}

    # the comparison strategy (north_star): global RK4 at the fine step dt/M,
    # M steps per coarse interval, timed the same way
    rk4 = None
    if not args.no_rk4:
        ctx.reset_ledger()
        ctx.advance(Scheme.RK4, wl.dt / wl.M, 1, wl.M)  # warm-up + graph
        ctx.reset_ledger()
        n_iv = max(1, min(args.steps, 20))
        barrier(ws)
        torch.cuda.synchronize()
        r0 = torch.cuda.Event(enable_timing=True)
        r1 = torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        ctx.advance(Scheme.RK4, wl.dt / wl.M, 1, wl.M * n_iv, sync=False)
        r1.record(stream)
        torch.cuda.synchronize()
        ctx.sync()
        rk_ms = allreduce_max(r0.elapsed_time(r1), ws) / n_iv
        rk_edges = allreduce_sum(ctx.ledger().total_edge_evals(), ws) / n_iv
        rk4 = {"scheme": "RK4 at dt/M", "ms_per_coarse_interval": rk_ms,
               "edge_evals_per_s": rk_edges / (rk_ms / 1e3),
               "edge_evals_per_coarse_interval": rk_edges,
               "lts3_speedup_vs_rk4": rk_ms / ms_step, "intervals": n_iv}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        from oracle.oracle import ref_available
        # bounded sample: 1 warm-up + cpu_steps timed coarse steps with the
        # reference's ThreadedEvaluator on every host thread (as far as host
        # RAM allows)
        threads, note = ref_ranks(wl, cpu_threads()) if ref_available() else (None, "")
        if ref_available() and threads is None:
            cpu = {"unavailable": f"{args.config}: {note}"}
        elif ref_available():
            del ctx
            runner = RefRunner(wl, threads)
            runner.steps(1)
            rate, sps, _ = runner.steps(args.cpu_steps)
            cpu = {"value": rate, "unit": UNIT, "cores": max(threads, 1), "kind": "reference",
                   "host": host_info(),
                   "sample": f"{args.cpu_steps} LTS3 coarse step(s) of {args.config} after 1 "
                             f"warm-up, reference "
                             f"{'SerialEvaluator' if threads == 0 else f'ThreadedEvaluator {threads} ranks'}"
                             f" ({sps:.3f} s/step){note}"}
            if not args.no_rk4:
                rrate, rsps, _ = runner.steps(1, scheme=2, dt=wl.dt / wl.M)
                cpu["rk4_fine_dt"] = {"edge_evals_per_s": rrate, "s_per_step": rsps,
                                      "s_per_coarse_interval": rsps * wl.M,
                                      "sample": "1 RK4 step at dt/M, same evaluator"}
            del runner

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(wl, args.config, ws),
            "coarse_steps_per_s": 1e3 / ms_step,
            "step_algorithmic_GBps": step_alg / (ms_step / 1e3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "peak_kind": peak_kind,
                         "kernel": "tendency evaluation (A: PV+K, B: F,q~, C: dh/du + fused "
                                   f"stage update), out {int(evnc[k])} cells / {int(evne[k])} edges",
                         "algorithmic_bytes": alg, "ms": ev_mean,
                         "ms_samples": len(ev_samples), "ms_min": float(np.min(ev_samples)),
                         "ms_max": float(np.max(ev_samples)),
                         "ms_in_timed_region": ev_samples[0],
                         "ms_note": "CUDA events around the evaluation's three launches inside "
                                    "the step graph: the timed region's last step, then the same "
                                    "graph replayed step by step",
                         "share_of_step": float(evms.sum() / ms_step)},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": io_bytes,
                    "d2h_bytes_per_step": io_bytes, "steps": n_e2e},
            "e2e_dropin_eval": dropin,
            "cpu_baseline": cpu,
            "rk4_fine_dt": rk4,
            "gpu_launches": int(launches),
            "setup": {k: round(v, 2) for k, v in setup.items()},
            "clocks": ck,
        }
        if ws > 1:
            line["transport"] = os.environ.get("MSWM_TRANSPORT", "nccl")
        if dry_run and ws > 1:
            line["dry_run"] = "MSWM_HALO_DRYRUN=1: halo transfers skipped -- a check of the path, not a measurement"
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--level", type=int, default=None,
                    help="icosahedral level override of c4/c5 (tests; default: the config's)")
    ap.add_argument("--cpu-steps", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-rk4", action="store_true")
    ap.add_argument("--no-serial", action="store_true",
                    help="reference arm: skip the 1-core SerialEvaluator leg")
    ap.add_argument("--order", default="regions", choices=["regions", "hilbert", "input"],
                    help="device layout (results are bitwise independent of it)")
    args = ap.parse_args()
    start_rss_monitor()
    if args.warmup < 3:
        log("note: warmup < 3 violates the timing rules; using 3")
        args.warmup = 3
    ws, rank, local = dist_init()
    if args.impl == "reference":
        run_reference_arm(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

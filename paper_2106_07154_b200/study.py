"""Time-step convergence study on the device (proj/src/harness.cpp:243-309).

``convergence_study`` runs the scheme at every dt of a ladder from the same
initial state for the same duration, all on the GPU through one
``CudaContext``, and compares each final state with an RK4 reference run at
min(dts)/20 (the reference's choice), fitting log(err) ~ log(dt) by least
squares.  ``l2_error`` is harness.cpp:74-97 with the reference's sequential
summation order, so errors and slopes are bitwise the reference's when the
device states are (and they are: every scheme is bitwise the reference).

The reference drives it with the TC5 mountain initial state
(``init_tc5``, harness.cpp:35-72); here the caller passes the initial state,
so any workload can be studied (the tests pass the reference's TC5 state).
"""
from __future__ import annotations

import math

import numpy as np

from .api import ConfigError, CudaContext, Scheme, State, UsageError


def _seq_sum(x: np.ndarray) -> float:
    """Left-to-right sum (np.cumsum accumulates in order; np.sum is pairwise)."""
    return float(np.cumsum(x)[-1]) if len(x) else 0.0


def l2_error(mesh, a: State, ref: State, weighted: bool = False) -> dict:
    """harness.cpp:74-97: plain (default) or area / length weighted l2 and
    the max norm of a - ref."""
    if len(a.h) != mesh.n_cells or len(ref.h) != mesh.n_cells or \
            len(a.u) != mesh.n_edges or len(ref.u) != mesh.n_edges:
        raise UsageError("error norm: states do not match the mesh")
    dh = np.asarray(a.h, np.float64) - np.asarray(ref.h, np.float64)
    du = np.asarray(a.u, np.float64) - np.asarray(ref.u, np.float64)
    if weighted:
        th = np.asarray(mesh.cell_area) * dh * dh
        tu = np.asarray(mesh.edge_len) * np.asarray(mesh.edge_dual_len) * du * du
    else:
        th, tu = dh * dh, du * du
    return {"l2_h": math.sqrt(_seq_sum(th)), "l2_u": math.sqrt(_seq_sum(tu)),
            "linf_h": float(np.max(np.abs(dh), initial=0.0)),
            "linf_u": float(np.max(np.abs(du), initial=0.0))}


def run(ctx: CudaContext, state0: State, scheme: Scheme, dt: float, substeps: int,
        duration: float) -> State:
    """run_simulation's stepping loop (harness.cpp:125-196) on the device:
    duration / dt steps (a whole number, else ConfigError) from state0."""
    if not (dt > 0.0):
        raise ConfigError("time step must be positive")
    if duration < 0.0:
        raise ConfigError("duration must be non-negative")
    steps_real = duration / dt
    n = int(round(steps_real))
    if abs(steps_real - n) > 1e-6:
        raise ConfigError("duration must be a whole number of steps")
    ctx.upload(State(np.asarray(state0.h, np.float64), np.asarray(state0.u, np.float64), 0.0))
    if n:
        ctx.advance(scheme, dt, substeps, n)
    return ctx.download()


def _fit(dts, errs) -> float:
    n = len(errs)
    xs = [math.log(d) for d in dts]
    ys = [math.log(max(e, 1e-300)) for e in errs]
    sx = sy = 0.0
    for i in range(n):
        sx += xs[i]
        sy += ys[i]
    mx, my = sx / n, sy / n
    num = den = 0.0
    for i in range(n):
        num += (xs[i] - mx) * (ys[i] - my)
        den += (xs[i] - mx) * (xs[i] - mx)
    return num / den if den > 0.0 else 0.0


def convergence_study(ctx: CudaContext, state0: State, scheme: Scheme, substeps: int,
                      dts, duration: float) -> dict:
    """harness.cpp:243-309 on the device: err_h / err_u (plain l2 at the
    final time vs RK4 at min(dts)/20), least-squares slopes of log(err)
    against log(dt), and monotonicity flags."""
    dts = [float(d) for d in dts]
    if not dts:
        raise UsageError("convergence study: empty dt list")
    if any(not (d > 0.0) for d in dts):
        raise UsageError("convergence study: dt must be positive")
    if not (duration > 0.0):
        raise UsageError("convergence study: duration must be positive")
    ref = run(ctx, state0, Scheme.RK4, min(dts) / 20.0, 1, duration)
    err_h, err_u = [], []
    for dt in dts:
        st = run(ctx, state0, scheme, dt, substeps, duration)
        rep = l2_error(ctx.mesh, st, ref)
        err_h.append(rep["l2_h"])
        err_u.append(rep["l2_u"])
    order = sorted(range(len(dts)), key=lambda i: -dts[i])
    mono_h = all(err_h[order[j]] <= err_h[order[j - 1]] for j in range(1, len(order)))
    mono_u = all(err_u[order[j]] <= err_u[order[j - 1]] for j in range(1, len(order)))
    return {"dts": dts, "err_h": err_h, "err_u": err_u, "slope_h": _fit(dts, err_h),
            "slope_u": _fit(dts, err_u), "monotone_h": mono_h, "monotone_u": mono_u}

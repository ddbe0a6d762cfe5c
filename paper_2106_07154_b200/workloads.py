"""Seeded synthetic workloads C1..C5 of BASELINE.json ``configs``.

The reference ships no generator for these configurations (its only
initialiser is the TC5 mountain, proj/src/harness.cpp:35-72), so the fields
below are ours; both the CUDA path and the CPU oracle are fed the *same*
arrays, so parity does not depend on these choices.  Documented choices:

* "2 interface layers" = the paper's Interface1 + Interface2 bands with
  ``interface_width = 1``.
* Coarse dt = 0.5 * min(d_e) / sqrt(g * H_max) (C1's rule, applied to all).
* Planar fine predicates use minimum-image distance; spherical ones the
  great-circle angle (arc_angle, geometry.hpp:33-35, evaluated on the host).
* "Geostrophic" velocities come from a vertex streamfunction
  psi = g*eta/f0: u_e = -(psi(+t end) - psi(-t end)) / l_e, which is
  discretely non-divergent on the TRiSK grid (f0 = 1e-4 on the beta-plane,
  whose f jumps across the periodic y-seam; 2 Omega on the sphere).
* "Spherical-harmonic perturbation of degree <= 32" is realised as a sum of
  random 3-D plane waves cos(k.x + phi) with |k| <= 32 restricted to the
  sphere (band-limited to leading order), scaled to the stated rms.
* C5 says "same field generator as config 3"; read 0-based that is C4's
  spherical generator, which is what is used.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .mesh import Mesh

GRAVITY = 9.81
OMEGA = 7.292e-5          # harness.hpp:27
EARTH_RADIUS = 6371220.0  # harness.hpp:28


@dataclass
class Workload:
    name: str
    mesh: Mesh
    h: np.ndarray
    u: np.ndarray
    b: np.ndarray
    f: np.ndarray
    fine_mask: np.ndarray
    gravity: float
    dt: float
    M: int
    n_steps: int
    width: int = 1
    meta: dict = field(default_factory=dict)


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def coarse_dt(mesh: Mesh, depth: float, gravity: float = GRAVITY) -> float:
    return 0.5 * float(np.min(mesh.edge_dual_len)) / math.sqrt(gravity * depth)


def _velocity_from_streamfunction(mesh: Mesh, psi_v: np.ndarray) -> np.ndarray:
    ev = mesh.edge_vertices
    sg = mesh.edge_vertex_sign.astype(np.float64)
    return -(sg[:, 0] * psi_v[ev[:, 0]] + sg[:, 1] * psi_v[ev[:, 1]]) / mesh.edge_len


def _planar_modes(rng, kmax: int, n_modes: int):
    ks = []
    while len(ks) < n_modes:
        kx, ky = rng.integers(-kmax, kmax + 1, size=2)
        if 0 < kx * kx + ky * ky <= kmax * kmax:
            ks.append((int(kx), int(ky)))
    phases = rng.uniform(0.0, 2.0 * math.pi, size=n_modes)
    amps = rng.uniform(0.5, 1.0, size=n_modes)
    return np.array(ks, np.float64), phases, amps


def _planar_field(mesh: Mesh, xy: np.ndarray, modes, target_rms: float, ref_xy=None):
    ks, ph, am = modes
    ref = xy if ref_xy is None else ref_xy

    def raw(p):
        arg = (2.0 * math.pi) * (np.outer(p[:, 0], ks[:, 0]) / mesh.width
                                 + np.outer(p[:, 1], ks[:, 1]) / mesh.height) + ph
        return np.cos(arg) @ am

    scale = target_rms / float(np.sqrt(np.mean(raw(ref) ** 2)))
    return raw(xy) * scale


def _planar_dist(mesh: Mesh, xy: np.ndarray, c) -> np.ndarray:
    d = mesh.min_image(xy[:, :2] - np.asarray(c)[None, :2])
    return np.hypot(d[:, 0], d[:, 1])


def config1(seed: int = 1, n_steps: int = 100) -> Workload:
    """BASELINE configs[0]: planar 64x64, dc 10 km, Gaussian bump, f-plane."""
    mesh = Mesh.planar_hex(64, 64, 10e3)
    rng = _rng(seed)
    H = 1000.0
    c = np.array([rng.uniform(0, mesh.width), rng.uniform(0, mesh.height)])
    r = _planar_dist(mesh, mesh.cell_xyz, c)
    h = H + 10.0 * np.exp(-(r * r) / (2.0 * 50e3 * 50e3))
    u = rng.normal(0.0, 1e-3, size=mesh.n_edges)
    b = np.zeros(mesh.n_cells)
    f = np.full(mesh.n_vertices, 1e-4)
    fine = (r < 0.2 * mesh.width).astype(np.uint8)
    return Workload("C1", mesh, h, u, b, f, fine, GRAVITY, coarse_dt(mesh, H), 4, n_steps,
                    meta={"mesh": "planar_hex 64x64 dc=10km", "center": c.tolist()})


def config2(seed: int = 2, n_steps: int = 1000, nx: int = 512) -> Workload:
    """BASELINE configs[1]: planar 512x512, dc 2 km, random bathymetry."""
    mesh = Mesh.planar_hex(nx, nx, 2e3)
    rng = _rng(seed)
    b = np.zeros(mesh.n_cells)
    for _ in range(16):
        c = np.array([rng.uniform(0, mesh.width), rng.uniform(0, mesh.height)])
        A = rng.uniform(0.0, 300.0)
        s = rng.uniform(5e3, 40e3)
        r = _planar_dist(mesh, mesh.cell_xyz, c)
        b += A * np.exp(-(r * r) / (2.0 * s * s))
    eta = _planar_field(mesh, mesh.cell_xyz, _planar_modes(rng, 8, 24), 1.0)
    h = 1000.0 - b + eta
    u = np.zeros(mesh.n_edges)
    f = np.full(mesh.n_vertices, 1e-4)
    c = np.array([rng.uniform(0, mesh.width), rng.uniform(0, mesh.height)])
    fine = (_planar_dist(mesh, mesh.cell_xyz, c) < 0.15 * mesh.width).astype(np.uint8)
    return Workload("C2", mesh, h, u, b, f, fine, GRAVITY, coarse_dt(mesh, 1000.0 + 1.0), 4,
                    n_steps, meta={"mesh": f"planar_hex {nx}x{nx} dc=2km"})


def config3(seed: int = 3, n_steps: int = 100, nx: int = 2048) -> Workload:
    """BASELINE configs[2]: planar 2048x2048, dc 1 km, beta-plane, 4 fine circles."""
    mesh = Mesh.planar_hex(nx, nx, 1e3)
    rng = _rng(seed)
    H = 1000.0
    f = 1e-4 + 2e-11 * mesh.vertex_xyz[:, 1]
    modes = _planar_modes(rng, 32, 64)
    eta_c = _planar_field(mesh, mesh.cell_xyz, modes, 2.0)
    eta_v = _planar_field(mesh, mesh.vertex_xyz, modes, 2.0, ref_xy=mesh.cell_xyz)
    h = H + eta_c
    # balance with f0: psi = g*eta/f would jump across the y-seam of the
    # periodic beta-plane (f is discontinuous there)
    u = _velocity_from_streamfunction(mesh, GRAVITY * eta_v / 1e-4)
    b = np.zeros(mesh.n_cells)
    centers, radii = [], []
    while len(centers) < 4:
        c = np.array([rng.uniform(0, mesh.width), rng.uniform(0, mesh.height)])
        r = rng.uniform(0.05, 0.1) * mesh.width
        ok = True
        for c2, r2 in zip(centers, radii):
            d = mesh.min_image((c - c2)[None, :])[0]
            ok &= math.hypot(d[0], d[1]) > r + r2 + 8 * 1e3
        if ok:
            centers.append(c)
            radii.append(r)
    fine = np.zeros(mesh.n_cells, np.uint8)
    for c, r in zip(centers, radii):
        fine |= (_planar_dist(mesh, mesh.cell_xyz, c) < r).astype(np.uint8)
    return Workload("C3", mesh, h, u, b, f, fine, GRAVITY, coarse_dt(mesh, H + 4.0), 8, n_steps,
                    meta={"mesh": f"planar_hex {nx}x{nx} dc=1km beta-plane"})


def _sphere_waves(rng, kmax: float, n_waves: int):
    k = rng.normal(size=(n_waves, 3))
    k /= np.linalg.norm(k, axis=1, keepdims=True)
    k *= rng.uniform(1.0, kmax, size=(n_waves, 1))
    return k, rng.uniform(0, 2 * math.pi, n_waves), rng.uniform(0.5, 1.0, n_waves)


def _sphere_field(xyz: np.ndarray, waves, chunk: int = 1 << 20) -> np.ndarray:
    k, ph, am = waves
    out = np.empty(len(xyz))
    for s in range(0, len(xyz), chunk):
        out[s:s + chunk] = np.cos(xyz[s:s + chunk] @ k.T + ph) @ am
    return out


def _random_unit(rng) -> np.ndarray:
    v = rng.normal(size=3)
    return v / np.linalg.norm(v)


def _cap_mask(mesh: Mesh, centers, radius_rad: float) -> np.ndarray:
    fine = np.zeros(mesh.n_cells, np.uint8)
    x = mesh.cell_xyz
    for c in centers:
        ang = np.arctan2(np.linalg.norm(np.cross(x, c[None, :]), axis=1), x @ c)
        fine |= (ang < radius_rad).astype(np.uint8)
    return fine


def _spherical(name: str, level: int, seed: int, caps: int, cap_deg: float, M: int,
               n_steps: int, mesh: Mesh | None = None) -> Workload:
    """``mesh``: the icosahedral level-``level`` mesh from another builder
    (the reference arm passes the reference's own build_voronoi_mesh, whose
    tables equal ours bitwise); default: ours."""
    if mesh is None:
        mesh = Mesh.icosahedral(level, EARTH_RADIUS)
    rng = _rng(seed)
    H = 4000.0
    waves = _sphere_waves(rng, 32.0, 64)
    raw_c = _sphere_field(mesh.cell_xyz, waves)
    scale = 5.0 / float(np.sqrt(np.mean(raw_c * raw_c)))
    h = H + scale * raw_c
    f = 2.0 * OMEGA * mesh.vertex_xyz[:, 2]  # harness.cpp:68-69
    psi = (GRAVITY / (2.0 * OMEGA)) * scale * _sphere_field(mesh.vertex_xyz, waves)
    u = _velocity_from_streamfunction(mesh, psi)
    b = np.zeros(mesh.n_cells)
    centers = []
    while len(centers) < caps:
        c = _random_unit(rng)
        if all(math.degrees(math.acos(np.clip(c @ c2, -1, 1))) > 2 * cap_deg + 2 for c2 in centers):
            centers.append(c)
    fine = _cap_mask(mesh, centers, math.radians(cap_deg))
    return Workload(name, mesh, h, u, b, f, fine, GRAVITY, coarse_dt(mesh, H + 25.0), M, n_steps,
                    meta={"mesh": f"icosahedral L{level}", "caps": caps, "cap_deg": cap_deg})


def config4(seed: int = 4, n_steps: int = 100, level: int = 10, mesh: Mesh | None = None) -> Workload:
    """BASELINE configs[3]: icosahedral L10, 20 degree cap, M=4."""
    return _spherical("C4", level, seed, 1, 20.0, 4, n_steps, mesh)


def config5(seed: int = 5, n_steps: int = 20, level: int = 11, mesh: Mesh | None = None) -> Workload:
    """BASELINE configs[4]: icosahedral L11, three 10 degree caps, M=8."""
    return _spherical("C5", level, seed, 3, 10.0, 8, n_steps, mesh)


# icosahedral level of the spherical configurations (reference-built meshes)
SPHERE_LEVEL = {"c4": 10, "c5": 11}


CONFIGS = {"c1": config1, "c2": config2, "c3": config3, "c4": config4, "c5": config5}


def small_sphere(level: int = 4, seed: int = 11, cap_deg: float = 30.0, M: int = 4) -> Workload:
    """A C4-shaped workload on a small icosahedral mesh (parity tests)."""
    return _spherical(f"sphere-L{level}", level, seed, 1, cap_deg, M, 10)

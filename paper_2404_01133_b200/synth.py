"""Synthetic city scenes of the reference's shape, for tests and benchmarks.

Follows the distributions of citysplat.synthetic.generate_synthetic_city
(synthetic.py:96-203): 30% ground sheet (xy scale U(0.35, 0.7), z scale
U(0.03, 0.08), opacity U(0.45, 0.9)); the rest on the walls and roofs of
box buildings proportional to surface area (thin axis U(0.08, 0.18), planar
axes U(0.35, 0.9), opacity U(0.75, 0.98), yaw-aligned quaternions); degree-3
SH N(0, 0.05) around a per-building albedo; position jitter N(0, 0.05).
Cameras: two orbit rings (0.12 and 0.30 x extent) plus a top-down grid at
0.35 / 0.55 x extent, fx = 0.85 W (synthetic.py:206-244).

This is an input generator, not a port: it draws its own random stream
(numpy on the host, or torch on the GPU for 23M-Gaussian scenes), so scenes
are not bit-identical to the reference's; parity is always checked against
the oracle on the *same* arrays.  Every value is rounded to float32
(SURVEY.md Appendix B.4), so device float32 storage is exact.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Tuple

import numpy as np

from .core import CameraView

__all__ = ["CityArrays", "generate_city", "generate_city_torch", "look_at", "city_cameras",
           "orbit_cameras"]

SH_C0 = 0.28209479177387814


@dataclass
class CityArrays:
    positions: np.ndarray
    opacities: np.ndarray
    scales: np.ndarray
    rotations: np.ndarray
    sh: np.ndarray

    @property
    def count(self) -> int:
        return int(self.positions.shape[0])


def look_at(eye, target, width: int, height: int, fx: float, fy=None, up=(0.0, 0.0, 1.0)) -> CameraView:
    """Camera at `eye` looking at `target`, x right / y down / z forward."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    n = np.linalg.norm(fwd)
    if n == 0:
        raise ValueError("eye and target coincide")
    fwd = fwd / n
    up = np.asarray(up, dtype=np.float64)
    if abs(fwd @ up) / np.linalg.norm(up) > 0.999:
        up = np.array([0.0, 1.0, 0.0])
    right = np.cross(fwd, up)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])
    return CameraView(width=width, height=height, fx=fx, fy=fx if fy is None else fy,
                      cx=width / 2.0, cy=height / 2.0, rotation_w2c=R, translation_w2c=-R @ eye)


def _alloc(weights, total):
    raw = np.asarray(weights, dtype=np.float64)
    raw = raw / raw.sum() * total
    base = np.floor(raw).astype(np.int64)
    rem = total - int(base.sum())
    base[np.argsort(base - raw)[:rem]] += 1
    return base


def _buildings(rng, n_buildings, half):
    centers = rng.uniform(-0.85 * half, 0.85 * half, (n_buildings, 2))
    w = rng.uniform(3.0, 12.0, n_buildings)
    d = rng.uniform(3.0, 12.0, n_buildings)
    h = rng.uniform(5.0, 40.0, n_buildings)
    yaw = rng.uniform(0.0, 2.0 * math.pi, n_buildings)
    albedo = rng.uniform(0.2, 0.9, (n_buildings, 3))
    return centers, w, d, h, yaw, albedo


def generate_city(seed: int = 0, extent: float = 100.0, n_buildings: int = 40,
                  n_gaussians: int = 50_000) -> CityArrays:
    """Host (numpy) generator; float32-exact float64 arrays, sh (K, 3, 16)."""
    rng = np.random.default_rng(seed)
    half = extent / 2.0
    centers, bw, bd, bh, yaw, albedo = _buildings(rng, n_buildings, half)
    n_ground = int(round(0.3 * n_gaussians))
    area = 2.0 * bh * (bw + bd) + bw * bd
    per_b = _alloc(area, n_gaussians - n_ground)
    P, S, Q, O, A = [], [], [], [], []
    P.append(np.column_stack([rng.uniform(-half, half, n_ground), rng.uniform(-half, half, n_ground),
                              np.zeros(n_ground)]))
    S.append(np.column_stack([rng.uniform(0.35, 0.7, (n_ground, 2)), rng.uniform(0.03, 0.08, n_ground)]))
    Q.append(np.tile([1.0, 0.0, 0.0, 0.0], (n_ground, 1)))
    O.append(rng.uniform(0.45, 0.9, n_ground))
    A.append(np.tile([0.36, 0.42, 0.33], (n_ground, 1)))
    # all building faces at once: face f of building b gets a share of per_b[b]
    face_area = np.stack([bd * bh, bd * bh, bw * bh, bw * bh, bw * bd], axis=1)
    counts = np.stack([_alloc(face_area[b], per_b[b]) if per_b[b] else np.zeros(5, np.int64)
                       for b in range(n_buildings)])
    bid = np.repeat(np.arange(n_buildings), counts.sum(axis=1))
    face = np.concatenate([np.repeat(np.arange(5), counts[b]) for b in range(n_buildings)])
    nb = bid.size
    u = rng.uniform(-0.5, 0.5, nb)
    v = rng.uniform(0.0, 1.0, nb)
    thin = rng.uniform(0.08, 0.18, nb)
    t1 = rng.uniform(0.35, 0.9, nb)
    t2 = rng.uniform(0.35, 0.9, nb)
    w_, d_, h_ = bw[bid], bd[bid], bh[bid]
    loc = np.zeros((nb, 3))
    sc = np.zeros((nb, 3))
    sign = np.where(face % 2 == 0, -1.0, 1.0)
    wx = face < 2
    wy = (face >= 2) & (face < 4)
    rf = face == 4
    loc[wx] = np.column_stack([sign[wx] * w_[wx] / 2, u[wx] * d_[wx], v[wx] * h_[wx]])
    sc[wx] = np.column_stack([thin[wx], t1[wx], t2[wx]])
    loc[wy] = np.column_stack([u[wy] * w_[wy], sign[wy] * d_[wy] / 2, v[wy] * h_[wy]])
    sc[wy] = np.column_stack([t1[wy], thin[wy], t2[wy]])
    loc[rf] = np.column_stack([u[rf] * w_[rf], (v[rf] - 0.5) * d_[rf], h_[rf]])
    sc[rf] = np.column_stack([t1[rf], t2[rf], thin[rf]])
    cy, sy = np.cos(yaw[bid]), np.sin(yaw[bid])
    world = np.column_stack([centers[bid, 0] + cy * loc[:, 0] - sy * loc[:, 1],
                             centers[bid, 1] + sy * loc[:, 0] + cy * loc[:, 1], loc[:, 2]])
    P.append(world)
    S.append(sc)
    Q.append(np.column_stack([np.cos(yaw[bid] / 2), np.zeros(nb), np.zeros(nb), np.sin(yaw[bid] / 2)]))
    O.append(rng.uniform(0.75, 0.98, nb))
    A.append(albedo[bid])
    pos = np.concatenate(P)
    pos = pos + rng.normal(0.0, 0.05, pos.shape)
    alb = np.concatenate(A)
    k = pos.shape[0]
    sh = rng.normal(0.0, 0.05, (k, 3, 16))
    sh[:, :, 0] = (alb + rng.normal(0.0, 0.03, (k, 3)) - 0.5) / SH_C0
    q = np.concatenate(Q)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)
    return CityArrays(f32(pos), f32(np.concatenate(O)), f32(np.concatenate(S)), f32(q), f32(sh))


def generate_city_torch(seed: int, extent: float, n_buildings: int, n_gaussians: int, device="cuda"):
    """Same distributions, generated on the GPU (for 23M-Gaussian scenes).
    Returns float32 torch tensors (positions, opacities, scales, rotations, sh)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    rng = np.random.default_rng(seed)
    half = extent / 2.0
    centers, bw, bd, bh, yaw, albedo = _buildings(rng, n_buildings, half)
    n_ground = int(round(0.3 * n_gaussians))
    area = 2.0 * bh * (bw + bd) + bw * bd
    per_b = _alloc(area, n_gaussians - n_ground)
    face_area = np.stack([bd * bh, bd * bh, bw * bh, bw * bh, bw * bd], axis=1)
    counts = np.stack([_alloc(face_area[b], per_b[b]) if per_b[b] else np.zeros(5, np.int64)
                       for b in range(n_buildings)])
    dev = torch.device(device)
    U = lambda n, a, b: torch.rand(n, generator=g, device=dev, dtype=torch.float64) * (b - a) + a
    k = n_gaussians
    pos = torch.empty((k, 3), dtype=torch.float64, device=dev)
    sc = torch.empty((k, 3), dtype=torch.float64, device=dev)
    quat = torch.zeros((k, 4), dtype=torch.float64, device=dev)
    opac = torch.empty(k, dtype=torch.float64, device=dev)
    alb = torch.empty((k, 3), dtype=torch.float64, device=dev)
    ng = n_ground
    pos[:ng, 0] = U(ng, -half, half)
    pos[:ng, 1] = U(ng, -half, half)
    pos[:ng, 2] = 0.0
    sc[:ng, 0] = U(ng, 0.35, 0.7)
    sc[:ng, 1] = U(ng, 0.35, 0.7)
    sc[:ng, 2] = U(ng, 0.03, 0.08)
    quat[:ng, 0] = 1.0
    opac[:ng] = U(ng, 0.45, 0.9)
    alb[:ng] = torch.tensor([0.36, 0.42, 0.33], dtype=torch.float64, device=dev)
    bid = torch.from_numpy(np.repeat(np.arange(n_buildings), counts.sum(axis=1))).to(dev)
    face = torch.from_numpy(np.concatenate([np.repeat(np.arange(5), counts[b])
                                            for b in range(n_buildings)])).to(dev)
    nb = bid.numel()
    u, v = U(nb, -0.5, 0.5), U(nb, 0.0, 1.0)
    thin, t1, t2 = U(nb, 0.08, 0.18), U(nb, 0.35, 0.9), U(nb, 0.35, 0.9)
    T = lambda a: torch.from_numpy(np.asarray(a, dtype=np.float64)).to(dev)
    w_, d_, h_ = T(bw)[bid], T(bd)[bid], T(bh)[bid]
    sign = torch.where(face % 2 == 0, -1.0, 1.0).double()
    wx, wy, rf = face < 2, (face >= 2) & (face < 4), face == 4
    lx = torch.where(wx, sign * w_ / 2, u * w_)
    ly = torch.where(wx, u * d_, torch.where(wy, sign * d_ / 2, (v - 0.5) * d_))
    lz = torch.where(rf, h_, v * h_)
    s0 = torch.where(wx, thin, t1)
    s1 = torch.where(wx, t1, torch.where(wy, thin, t2))
    s2 = torch.where(rf, thin, t2)
    yb = T(yaw)[bid]
    cb = T(centers)[bid]
    cy, sy = torch.cos(yb), torch.sin(yb)
    pos[ng:, 0] = cb[:, 0] + cy * lx - sy * ly
    pos[ng:, 1] = cb[:, 1] + sy * lx + cy * ly
    pos[ng:, 2] = lz
    sc[ng:, 0], sc[ng:, 1], sc[ng:, 2] = s0, s1, s2
    quat[ng:, 0] = torch.cos(yb / 2)
    quat[ng:, 3] = torch.sin(yb / 2)
    opac[ng:] = U(nb, 0.75, 0.98)
    alb[ng:] = T(albedo)[bid]
    pos += torch.randn((k, 3), generator=g, device=dev, dtype=torch.float64) * 0.05
    quat = quat / quat.norm(dim=1, keepdim=True)
    sh = torch.randn((k, 3, 16), generator=g, device=dev, dtype=torch.float32) * 0.05
    sh[:, :, 0] = ((alb + torch.randn((k, 3), generator=g, device=dev, dtype=torch.float64) * 0.03
                    - 0.5) / SH_C0).float()
    return pos.float(), opac.float(), sc.float(), quat.float(), sh


def city_cameras(n_cameras: int, extent: float, width: int, height: int, seed: int = 0) -> List[CameraView]:
    """Orbit rings + top-down grid of the reference's camera set (synthetic.py:206-244)."""
    rng = np.random.default_rng(seed + 1)
    fx = 0.85 * width
    half = extent / 2.0
    cams = []
    n_orbit = n_cameras // 2
    n_low = n_orbit // 2
    for count, alt, radius in ((n_low, 0.12 * extent, 0.62 * half),
                               (n_orbit - n_low, 0.30 * extent, 0.85 * half)):
        for i in range(count):
            a = 2.0 * math.pi * i / max(count, 1) + rng.normal(0.0, 0.02)
            r = radius * (1.0 + rng.normal(0.0, 0.02))
            eye = [r * math.cos(a), r * math.sin(a), alt * (1.0 + rng.normal(0.0, 0.03))]
            cams.append(look_at(eye, rng.normal([0.0, 0.0, 4.0], [2.0, 2.0, 1.0]), width, height, fx))
    n_grid = n_cameras - n_orbit
    side = max(1, math.ceil(math.sqrt(n_grid)))
    lattice = np.linspace(-0.55 * half, 0.55 * half, side)
    made = 0
    for gy in lattice:
        for gx in lattice:
            if made >= n_grid:
                break
            alt = (0.35 if made % 2 == 0 else 0.55) * extent
            eye = np.array([gx, gy, alt]) + rng.normal(0.0, 0.5, 3)
            tgt = [0.6 * eye[0] + rng.normal(0.0, 1.0), 0.6 * eye[1] + rng.normal(0.0, 1.0), 0.0]
            cams.append(look_at(eye, tgt, width, height, fx))
            made += 1
    return cams


def orbit_cameras(center, radius: float, altitude: float, n: int, width: int, height: int,
                  fx_scale: float = 0.8) -> List[CameraView]:
    """cmd_bench's sweep (cli.py:203-218): orbit at `radius`, `altitude` above
    the centre, looking at the centre, fx = 0.8 W."""
    center = np.asarray(center, dtype=np.float64)
    cams = []
    for i in range(n):
        a = 2.0 * math.pi * i / n
        eye = center + np.array([radius * math.cos(a), radius * math.sin(a), altitude])
        cams.append(look_at(eye, center, width, height, fx_scale * width))
    return cams

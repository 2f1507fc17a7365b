"""Offline LoD generation on the GPU.

Builds the per-block detail levels of a partitioned scene the way
citysplat.lod.build_lod does (lod.py:211-248):

* ``significance_scores`` (lod.py:54-101): training-view hit count x opacity x
  percentile-clamped volume^0.1 -- a view hits a Gaussian whose centre is in
  front of the near plane, projects inside the image and whose support radius
  (from the largest eigenvalue of cov2d + 0.3) is at least half a pixel;
* a stable descending ranking (ties -> lower index, lod.py:114-116);
* level L keeps the top ceil(rate_L K - 1e-9 K) globally (lod.py:104-111) and
  splits them by block in ascending index order, SH truncated per level;
* MAD-clipped world bounds per block from the full membership (lod.py:130-147).

Membership comes from the CUDA contraction/binning kernel (cs_block_of_points).
This is the offline scene build feeding the benchmark, not the timed path; it
runs as float64 torch ops on the device.
"""

from __future__ import annotations

import ctypes
import math
from typing import Sequence

import numpy as np
import torch

from . import _lib, device
from ._lib import check

VOLUME_EXPONENT = 0.1     # lod.py:43
VOLUME_PERCENTILE = 90.0  # lod.py:44
MIN_FOOTPRINT_RADIUS = 0.5  # lod.py:45


def central_third(positions: torch.Tensor):
    """ContractionMap.central_third (partition.py:84-97) -> (p_min, p_max)."""
    p = positions.double()
    lo = p.min(dim=0).values.cpu().numpy()
    hi = p.max(dim=0).values.cpu().numpy()
    center = 0.5 * (lo + hi)
    sixth = np.maximum((hi - lo) / 6.0, 1e-6)
    z0, z1 = float(lo[2]), float(hi[2])
    if z1 <= z0:
        z1 = z0 + 1e-6
    return (np.array([center[0] - sixth[0], center[1] - sixth[1], z0]),
            np.array([center[0] + sixth[0], center[1] + sixth[1], z1]))


def block_membership(positions: torch.Tensor, p_min, p_max, dims) -> torch.Tensor:
    """grid_partition membership (partition.py:208-231) via the CUDA kernel."""
    dims = tuple(int(d) for d in dims) + ((1,) if len(dims) == 2 else ())
    pos = positions.contiguous()
    f32 = 1 if pos.dtype == torch.float32 else 0
    if not f32:
        pos = pos.double().contiguous()
    out = torch.empty(pos.shape[0], dtype=torch.int32, device=pos.device)
    pmin = np.ascontiguousarray(p_min, dtype=np.float64)
    pmax = np.ascontiguousarray(p_max, dtype=np.float64)
    check(_lib.load().cs_block_of_points(device.context(pos.device.index), pos.shape[0], pos.data_ptr(),
                                         f32, pmin.ctypes.data, pmax.ctypes.data, dims[0], dims[1],
                                         dims[2], out.data_ptr(), device.stream_handle(pos.device)))
    return out


def _rotmats(q: torch.Tensor) -> torch.Tensor:
    w, x, y, z = q.unbind(1)
    r = torch.stack([
        1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
        2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
        2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], dim=1)
    return r.view(-1, 3, 3)


def significance_scores(positions, opacities, scales, rotations, cameras, near=0.2,
                        alpha_floor=1.0 / 255.0, chunk=1 << 22) -> torch.Tensor:
    k = positions.shape[0]
    dev = positions.device
    hits = torch.zeros(k, dtype=torch.float64, device=dev)
    ss = math.sqrt(2.0 * math.log(1.0 / alpha_floor))
    for s in range(0, k, chunk):
        e = min(k, s + chunk)
        p = positions[s:e].double()
        r = _rotmats(rotations[s:e].double())
        sc2 = scales[s:e].double() ** 2
        sigma = torch.einsum("kij,kj,klj->kil", r, sc2, r)
        for cam in cameras:
            R = torch.from_numpy(np.asarray(cam.rotation_w2c, dtype=np.float64)).to(dev)
            T = torch.from_numpy(np.asarray(cam.translation_w2c, dtype=np.float64)).to(dev)
            t = p @ R.T + T
            z = t[:, 2]
            front = z > near
            zs = torch.where(front, z, torch.ones_like(z))
            u = cam.fx * t[:, 0] / zs + cam.cx
            v = cam.fy * t[:, 1] / zs + cam.cy
            on = front & (u >= 0) & (u <= cam.width) & (v >= 0) & (v <= cam.height)
            V = torch.einsum("ij,kjl,ml->kim", R, sigma, R)
            J = torch.zeros((e - s, 2, 3), dtype=torch.float64, device=dev)
            J[:, 0, 0] = cam.fx / zs
            J[:, 0, 2] = -cam.fx * t[:, 0] / (zs * zs)
            J[:, 1, 1] = cam.fy / zs
            J[:, 1, 2] = -cam.fy * t[:, 1] / (zs * zs)
            cov = J @ V @ J.transpose(1, 2)
            a = cov[:, 0, 0] + 0.3
            b = cov[:, 0, 1]
            c = cov[:, 1, 1] + 0.3
            mid = 0.5 * (a + c)
            lam = mid + torch.sqrt(torch.clamp(mid * mid - (a * c - b * b), min=0.0))
            radius = ss * torch.sqrt(lam)
            hits[s:e] += (on & (radius >= MIN_FOOTPRINT_RADIUS)).double()
    volume = scales.double().prod(dim=1)
    cap = float(np.percentile(volume.cpu().numpy(), VOLUME_PERCENTILE))
    return hits * opacities.double() * torch.clamp(volume, max=cap) ** VOLUME_EXPONENT


def keep_count(rate: float, k: int) -> int:
    if not 0.0 < rate <= 1.0:
        raise ValueError("compression rate must be in (0, 1]")
    if k == 0:
        return 0
    return min(k, max(1, math.ceil(rate * k - 1e-9 * k)))


def _median(x: torch.Tensor) -> torch.Tensor:
    """np.median along dim 0 (mean of the two middle values for even n)."""
    n = x.shape[0]
    s = torch.sort(x, dim=0).values
    if n % 2:
        return s[n // 2]
    return 0.5 * (s[n // 2 - 1] + s[n // 2])


def mad_bounds(p: torch.Tensor, n_mad: float):
    p = p.double()
    lo = p.min(dim=0).values
    hi = p.max(dim=0).values
    med = _median(p)
    mad = _median((p - med).abs())
    if math.isfinite(n_mad):
        ok = mad > 0
        lo = torch.where(ok, torch.maximum(lo, med - n_mad * mad), lo)
        hi = torch.where(ok, torch.minimum(hi, med + n_mad * mad), hi)
    return lo.cpu().numpy(), hi.cpu().numpy()


def build_lod_device(positions, opacities, scales, rotations, sh, membership: torch.Tensor,
                     n_blocks: int, cameras: Sequence, distance_intervals=((0.0, 200.0), (200.0, 400.0),
                                                                           (400.0, math.inf)),
                     compression_rates=(0.5, 0.34, 0.25), lod_sh_degrees=(3, 2, 1), n_mad=4.0,
                     scores=None) -> device.DeviceLodScene:
    """build_lod (lod.py:211-248) into a DeviceLodScene; rates/degrees finest-first."""
    k = positions.shape[0]
    dev = positions.device
    if scores is None:
        scores = significance_scores(positions, opacities, scales, rotations, cameras)
    order = torch.sort(-scores, stable=True).indices
    rates = tuple(reversed(compression_rates))
    degrees = tuple(reversed(lod_sh_degrees))
    mem = membership.long()
    level_clouds = []
    counts = np.zeros((len(rates), n_blocks), dtype=np.int64)
    for L, (rate, deg) in enumerate(zip(rates, degrees)):
        keep = keep_count(rate, k)
        mask = torch.zeros(k, dtype=torch.bool, device=dev)
        mask[order[:keep]] = True
        idx = torch.nonzero(mask).squeeze(1)            # ascending original index
        blk = mem[idx]
        perm = torch.sort(blk, stable=True).indices     # group by block, keep index order
        rows = idx[perm]
        counts[L] = torch.bincount(blk, minlength=n_blocks).cpu().numpy()
        C = (deg + 1) ** 2
        level_clouds.append(device.DeviceCloud.from_torch(
            positions[rows], opacities[rows], scales[rows], rotations[rows], sh[rows][:, :, :C]))
    bmin = np.zeros((n_blocks, 3))
    bmax = np.zeros((n_blocks, 3))
    for j in range(n_blocks):
        m = torch.nonzero(mem == j).squeeze(1)
        if m.numel():
            bmin[j], bmax[j] = mad_bounds(positions[m], n_mad)
    return device.DeviceLodScene.from_device_levels(level_clouds, counts, bmin, bmax,
                                                    distance_intervals, degrees, dev.index)

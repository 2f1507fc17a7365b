"""LoD generation on the GPU, hand-written kernels.

Builds the per-block detail levels of a partitioned scene the way
citysplat.lod.build_lod does (lod.py:211-248), entirely through libcsgpu:

* ``significance_scores`` (lod.py:54-101) -> ``cs_significance`` (K15 hit
  counts in the projection's float64 op order, volume percentile, scores);
* ``priority``  (lod.py:114-116)          -> ``cs_priority`` (stable 64-bit
  radix sort of the complemented score bits: descending, ties -> lower index);
* level rows    (lod.py:222-234)          -> ``cs_lod_rows`` (level L keeps the
  top ceil(rate_L K - 1e-9 K), grouped by block, ascending index);
* ``mad_bounds`` (lod.py:130-147)         -> ``cs_mad_bounds`` (per-block
  medians / MADs from stable sorts, clipping as the reference);
* ``cloud.take(rows).with_sh_degree(d)``  -> ``cs_gather_cloud``.

Membership comes from the contraction/binning kernel (cs_block_of_points).
Host-facing mirrors with the reference signatures live in ``lod.py``.
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


def _cams(cameras):
    views = [c if hasattr(c, "rotation_w2c") else c.view for c in cameras]
    arr = (_lib.CsCamera * max(len(views), 1))()
    for i, v in enumerate(views):
        arr[i] = device.camera_struct(v)
    return arr, len(views)


def significance_scores(cloud: "device.DeviceCloud", cameras: Sequence, settings=None,
                        return_hits: bool = False):
    """lod.significance_scores (lod.py:54-101) of a DeviceCloud -> float64 device tensor."""
    from .render import RenderSettings
    settings = settings or RenderSettings()
    k = cloud.count
    dev = cloud.device
    scores = torch.empty(k, dtype=torch.float64, device=dev)
    hits = torch.empty(k, dtype=torch.int32, device=dev)
    arr, n = _cams(cameras)
    desc = cloud.desc()
    cset = device.settings_struct(settings)
    check(_lib.load().cs_significance(device.context(dev.index), ctypes.byref(desc),
                                      ctypes.cast(arr, ctypes.c_void_p), n, ctypes.byref(cset),
                                      scores.data_ptr(), hits.data_ptr(), device.stream_handle(dev)),
          "cs_significance")
    return (scores, hits) if return_hits else scores


def priority(scores: torch.Tensor) -> torch.Tensor:
    """lod._priority (lod.py:114-116): int32 indices, descending score, ties -> lower index."""
    scores = scores.to(torch.float64).contiguous()
    order = torch.empty(scores.shape[0], dtype=torch.int32, device=scores.device)
    check(_lib.load().cs_priority(device.context(scores.device.index), scores.shape[0],
                                  scores.data_ptr(), order.data_ptr(),
                                  device.stream_handle(scores.device)), "cs_priority")
    return order


def keep_count(rate: float, k: int) -> int:
    """lod._keep_count (lod.py:104-111)."""
    if not 0.0 < rate <= 1.0:
        raise ValueError("compression rate must be in (0, 1]")
    if k == 0:
        return 0
    return min(k, max(1, math.ceil(rate * k - 1e-9 * k)))


def level_rows(order: torch.Tensor, membership: torch.Tensor, n_blocks: int, rates_coarsest_first):
    """Kept rows of every level (lod.py:222-234) -> (rows int32 device (L, K), counts (L, J))."""
    k = order.shape[0]
    n_levels = len(rates_coarsest_first)
    rows = torch.empty((n_levels, max(k, 1)), dtype=torch.int32, device=order.device)
    counts = np.zeros((n_levels, n_blocks), dtype=np.int64)
    rates = np.ascontiguousarray(rates_coarsest_first, dtype=np.float64)
    mem = membership.to(torch.int32).contiguous()
    check(_lib.load().cs_lod_rows(device.context(order.device.index), k, order.data_ptr(),
                                  mem.data_ptr(), n_blocks, rates.ctypes.data, n_levels,
                                  rows.data_ptr(), counts.ctypes.data,
                                  device.stream_handle(order.device)), "cs_lod_rows")
    return rows, counts


def block_bounds(cloud: "device.DeviceCloud", membership: torch.Tensor, n_blocks: int, n_mad: float):
    """mad_bounds (lod.py:130-147) of every block's members -> (bmin, bmax) (J, 3) float64."""
    bmin = np.zeros((n_blocks, 3))
    bmax = np.zeros((n_blocks, 3))
    mem = membership.to(torch.int32).contiguous()
    desc = cloud.desc()
    check(_lib.load().cs_mad_bounds(device.context(cloud.device.index), ctypes.byref(desc),
                                    mem.data_ptr(), n_blocks, float(n_mad), bmin.ctypes.data,
                                    bmax.ctypes.data, device.stream_handle(cloud.device)),
          "cs_mad_bounds")
    return bmin, bmax


def gather(cloud: "device.DeviceCloud", rows: torch.Tensor, sh_coeffs: int) -> "device.DeviceCloud":
    """cloud.take(rows).with_sh_degree(...) on the device (rows: int32 device)."""
    n = int(rows.shape[0])
    dev = cloud.device
    dt = cloud.pos_op.dtype
    quads = torch.empty((3, n, 4), dtype=dt, device=dev)
    stride = device.sh_stride(sh_coeffs)
    sh = torch.empty((n, stride), dtype=torch.float32, device=dev)
    out = device.DeviceCloud(quads[0], quads[1], quads[2], sh, sh_coeffs, n)
    src = cloud.desc()
    dst = out.desc()
    rows = rows.to(torch.int32).contiguous()
    check(_lib.load().cs_gather_cloud(device.context(dev.index), ctypes.byref(src), rows.data_ptr(),
                                      n, ctypes.byref(dst), device.stream_handle(dev)),
          "cs_gather_cloud")
    return out


def build_lod_cloud(full: "device.DeviceCloud", membership: torch.Tensor, n_blocks: int,
                    cameras: Sequence,
                    distance_intervals=((0.0, 200.0), (200.0, 400.0), (400.0, math.inf)),
                    compression_rates=(0.5, 0.34, 0.25), lod_sh_degrees=(3, 2, 1), n_mad=4.0,
                    scores=None, settings=None) -> device.DeviceLodScene:
    """build_lod (lod.py:211-248) of a DeviceCloud into a DeviceLodScene.

    Rates / SH degrees are finest-first as in RunConfig and reversed here."""
    if scores is None:
        scores = significance_scores(full, cameras, settings)
    order = priority(scores)
    rates = tuple(reversed(compression_rates))
    degrees = tuple(reversed(lod_sh_degrees))
    rows, counts = level_rows(order, membership, n_blocks, rates)
    level_clouds = []
    for L, deg in enumerate(degrees):
        C = min((deg + 1) ** 2, full.sh_coeffs)
        level_clouds.append(gather(full, rows[L, :int(counts[L].sum())], C))
    bmin, bmax = block_bounds(full, membership, n_blocks, n_mad)
    return device.DeviceLodScene.from_device_levels(level_clouds, counts, bmin, bmax,
                                                    distance_intervals, degrees, full.device.index)


def build_lod_device(positions, opacities, scales, rotations, sh, membership: torch.Tensor,
                     n_blocks: int, cameras: Sequence, distance_intervals=((0.0, 200.0), (200.0, 400.0),
                                                                           (400.0, math.inf)),
                     compression_rates=(0.5, 0.34, 0.25), lod_sh_degrees=(3, 2, 1), n_mad=4.0,
                     scores=None) -> device.DeviceLodScene:
    """build_lod from device tensors (K,3),(K,),(K,3),(K,4),(K,3,C)."""
    full = device.DeviceCloud.from_torch(positions, opacities, scales, rotations, sh)
    return build_lod_cloud(full, membership, n_blocks, cameras, distance_intervals,
                           compression_rates, lod_sh_degrees, n_mad, scores)

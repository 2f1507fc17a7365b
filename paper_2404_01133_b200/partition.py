"""Training-data assignment on the GPU.

Drop-in for the assignment half of citysplat.partition (partition.py:172-439),
same names, signatures, return types and exceptions:

* ``bounds_contain``  (partition.py:172-181)  host utility, as the reference;
* ``enlarge_bounds``  (partition.py:234-259)  counts on the device (cs_bounds_contain
  over ``grid.contracted``);
* ``assign_b1``       (partition.py:318-334)  the "rest" render is the full cloud
  with block j's rows excluded (``cs_source.exclude``: identical image to
  ``cloud.take(~mask)``, no copy), SSIM by ``cs_ssim``;
* ``assign_b2``       (partition.py:337-345)  camera-centre containment, contracted
  on the device;
* ``assign``          (partition.py:348-439)  full images once per pose at
  ``assignment_scale``, one masked render + SSIM per (pose, block) -- all on the
  device, the l_ssim matrix read back once; enlarged-bounds retry and
  failure bookkeeping as the reference;
* ``AssignmentMatrix`` (partition.py:262-292).

A caller-supplied ``renderer=`` (the reference's injection hook) is honoured:
it is called with host clouds exactly as the reference does, and only the SSIM
runs on the device.
"""

from __future__ import annotations

import ctypes
import math
import warnings
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np
import torch

from . import _lib, device
from ._lib import check

__all__ = ["AssignmentMatrix", "bounds_contain", "enlarge_bounds", "assign_b1", "assign_b2",
           "assign", "ENLARGE_FACTOR"]

ENLARGE_FACTOR = 1.2  # partition.py:45

_WINDOW = 11
_SIGMA = 1.5


def _ssim_window() -> np.ndarray:
    """metrics._gaussian_window (metrics.py:61-64), the reference's arithmetic."""
    g = np.exp(-((np.arange(_WINDOW) - _WINDOW // 2) ** 2) / (2.0 * _SIGMA ** 2))
    w = np.outer(g, g)
    return np.ascontiguousarray(w / w.sum(), dtype=np.float64)


_W2D = _ssim_window()


@dataclass(frozen=True)
class AssignmentMatrix:
    """partition.AssignmentMatrix (partition.py:262-292)."""

    entries: np.ndarray
    provenance: np.ndarray
    bounds_min_used: np.ndarray
    bounds_max_used: np.ndarray
    image_ids: tuple
    unassignable: tuple

    @property
    def n_poses(self) -> int:
        return self.entries.shape[0]

    @property
    def n_blocks(self) -> int:
        return self.entries.shape[1]

    def images_for_block(self, j: int) -> list:
        return [self.image_ids[i] for i in np.nonzero(self.entries[:, j])[0]]

    def blocks_for_image(self, image_id) -> list:
        i = self.image_ids.index(image_id)
        return list(np.nonzero(self.entries[i])[0])


def bounds_contain(points, bounds_min, bounds_max) -> np.ndarray:
    """partition.bounds_contain (partition.py:172-181): lower-inclusive,
    upper-exclusive, an upper bound on the cube surface (== 2) inclusive."""
    p = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    lo = np.asarray(bounds_min, dtype=np.float64)
    hi = np.asarray(bounds_max, dtype=np.float64)
    below = np.where(hi == 2.0, p <= hi, p < hi)
    return ((p >= lo) & below).all(axis=1)


# ---------------------------------------------------------------------------
# device helpers


def _dev():
    return device.default_device()


def _contracted_dev(grid) -> torch.Tensor:
    """grid.contracted as a device float64 (K, 3) tensor (cached per grid)."""
    return device._cached(grid, ("contracted", _dev().index), lambda: torch.as_tensor(
        np.ascontiguousarray(np.asarray(grid.contracted, dtype=np.float64).reshape(-1, 3)), device=_dev()))


def _membership_dev(grid) -> torch.Tensor:
    return device._cached(grid, ("membership", _dev().index), lambda: torch.as_tensor(
        np.asarray(grid.membership).astype(np.int32), device=_dev()))


def _contain(points: torch.Tensor, lo, hi, mask: Optional[torch.Tensor] = None, p_min=None,
             p_max=None, count: bool = True) -> int:
    """cs_bounds_contain over device xyz points (contracted unless p_min/p_max given)."""
    lo = np.ascontiguousarray(lo, dtype=np.float64).reshape(3)
    hi = np.ascontiguousarray(hi, dtype=np.float64).reshape(3)
    pm = np.ascontiguousarray(p_min, dtype=np.float64).reshape(3) if p_min is not None else None
    px = np.ascontiguousarray(p_max, dtype=np.float64).reshape(3) if p_max is not None else None
    n = ctypes.c_int64(0)
    pts = points.contiguous()
    f32 = 1 if pts.dtype == torch.float32 else 0
    check(_lib.load().cs_bounds_contain(
        device.context(pts.device.index), pts.shape[0], pts.data_ptr(), f32, 3,
        pm.ctypes.data if pm is not None else None, px.ctypes.data if px is not None else None,
        lo.ctypes.data, hi.ctypes.data, mask.data_ptr() if mask is not None else None,
        ctypes.byref(n) if count else None, device.stream_handle(pts.device)), "cs_bounds_contain")
    return int(n.value)


def enlarge_bounds(j: int, grid, min_count: int, factor: float = ENLARGE_FACTOR):
    """partition.enlarge_bounds (partition.py:234-259); counts on the device."""
    if min_count <= 0:
        raise ValueError("min_count must be positive")
    lo = np.asarray(grid.bounds_min[j], dtype=np.float64).copy()
    hi = np.asarray(grid.bounds_max[j], dtype=np.float64).copy()
    total = int(np.asarray(grid.contracted).shape[0])
    if total < min_count:
        warnings.warn(
            f"scene holds {total} Gaussians, fewer than the enlargement "
            f"threshold {min_count}; using the whole contracted cube"
        )
        return np.full(3, -2.0), np.full(3, 2.0)
    pts = _contracted_dev(grid)
    while _contain(pts, lo, hi) < min_count:
        if (lo == -2.0).all() and (hi == 2.0).all():
            break
        center = 0.5 * (lo + hi)
        half = 0.5 * (hi - lo) * factor
        lo = np.maximum(center - half, -2.0)
        hi = np.minimum(center + half, 2.0)
    return lo, hi


def _scaled_camera(cam, scale: float):
    """partition._scaled_camera (partition.py:300-310)."""
    from .core import CameraView
    if scale == 1.0:
        return cam
    return CameraView(
        width=max(1, int(round(cam.width * scale))),
        height=max(1, int(round(cam.height * scale))),
        fx=cam.fx * scale, fy=cam.fy * scale,
        cx=cam.cx * scale, cy=cam.cy * scale,
        rotation_w2c=cam.rotation_w2c, translation_w2c=cam.translation_w2c,
    )


def _pose_view(pose, index: int):
    """partition._pose_view (partition.py:294-298)."""
    if hasattr(pose, "rotation_w2c"):
        return pose, index
    return pose.view, pose.image_id


class _Renderer:
    """Device renders of one cloud (float32 (H, W, 3) images), optionally with rows excluded."""

    def __init__(self, cloud, settings):
        from .render import RenderSettings
        self.settings = settings or RenderSettings()
        self.dc = device.device_cloud(cloud)
        self.cset = device.settings_struct(self.settings)

    def __call__(self, cam, exclude: Optional[torch.Tensor] = None) -> torch.Tensor:
        dev = self.dc.device
        out = torch.empty((int(cam.height), int(cam.width), 3), dtype=torch.float32, device=dev)
        src = _lib.CsSource()
        src.kind = _lib.CS_SRC_CLOUD
        src.force_level = -1
        src.cloud = self.dc.desc()
        src.exclude = exclude.data_ptr() if exclude is not None else None
        ccam = device.camera_struct(cam)
        check(_lib.load().cs_render(device.context(dev.index), ctypes.byref(src), ctypes.byref(ccam),
                                    ctypes.byref(self.cset), out.data_ptr(), _lib.CS_RENDER_SYNC, None,
                                    device.stream_handle(dev)), "cs_render")
        return out


def _ssim_into(a: torch.Tensor, b: torch.Tensor, acc4: torch.Tensor) -> None:
    """acc4[3] <- metrics.ssim(a, b) (metrics.py:70-96), asynchronously."""
    H, W = int(a.shape[0]), int(a.shape[1])
    if H < _WINDOW or W < _WINDOW:
        raise ValueError(f"images must be at least {_WINDOW}x{_WINDOW} for ssim")
    check(_lib.load().cs_ssim(device.context(a.device.index), a.data_ptr(), b.data_ptr(), H, W,
                              _W2D.ctypes.data, acc4.data_ptr(), device.stream_handle(a.device)),
          "cs_ssim")


def _image_tensor(img) -> torch.Tensor:
    px = getattr(img, "pixels", img)
    return torch.as_tensor(np.ascontiguousarray(np.asarray(px), dtype=np.float32), device=_dev())


def _l_ssim_host_images(a, b) -> float:
    acc = torch.zeros(4, dtype=torch.float64, device=_dev())
    ta, tb = _image_tensor(a), _image_tensor(b)
    if ta.shape != tb.shape:
        raise ValueError(f"image dimensions differ: {tuple(ta.shape)} vs {tuple(tb.shape)}")
    _ssim_into(ta, tb, acc)
    return 1.0 - float(acc[3].item())


def _mask_for(grid, j: int, bounds) -> torch.Tensor:
    if bounds is None:
        return (_membership_dev(grid) == j).to(torch.uint8)
    m = torch.empty(np.asarray(grid.contracted).shape[0], dtype=torch.uint8, device=_dev())
    _contain(_contracted_dev(grid), bounds[0], bounds[1], mask=m, count=False)
    return m


def _centers_in(views, grid, lo, hi) -> np.ndarray:
    """assign_b2 for every view against one box: contract(normalize_position(center))
    on the device, then the containment test."""
    c = np.ascontiguousarray(np.stack([np.asarray(v.camera_center, dtype=np.float64).reshape(3)
                                       for v in views]))
    pts = torch.as_tensor(c, device=_dev())
    m = torch.empty(len(views), dtype=torch.uint8, device=_dev())
    _contain(pts, lo, hi, mask=m, p_min=grid.map.p_min, p_max=grid.map.p_max, count=False)
    return m.cpu().numpy().astype(bool)


# ---------------------------------------------------------------------------
# public API


def assign_b1(pose, j: int, cloud, grid, epsilon: float, renderer: Optional[Callable] = None,
              bounds=None) -> bool:
    """partition.assign_b1 (partition.py:318-334): does removing block j's members
    change the render of this pose by more than epsilon in SSIM loss?"""
    if not 0.0 < epsilon < 1.0:
        raise ValueError("epsilon must be in (0, 1)")
    if bounds is None:
        member_mask = np.asarray(grid.membership) == j
    else:
        member_mask = bounds_contain(grid.contracted, bounds[0], bounds[1])
    if not member_mask.any():
        return False  # identical clouds render identically; the loss is zero
    if renderer is not None:
        full = renderer(cloud, pose)
        rest = renderer(cloud.take(np.nonzero(~member_mask)[0]), pose)
        return _l_ssim_host_images(full, rest) > epsilon
    r = _Renderer(cloud, None)
    acc = torch.zeros(4, dtype=torch.float64, device=_dev())
    full = r(pose)
    rest = r(pose, _mask_for(grid, j, bounds))
    _ssim_into(full, rest, acc)
    return (1.0 - float(acc[3].item())) > epsilon


def assign_b2(pose, j: int, grid, bounds=None) -> bool:
    """partition.assign_b2 (partition.py:337-345): camera centre inside block j."""
    if bounds is None:
        lo, hi = grid.bounds_min[j], grid.bounds_max[j]
    else:
        lo, hi = bounds
    return bool(_centers_in([pose], grid, lo, hi)[0])


def assign(poses: Sequence, grid, cloud, epsilon: float, *, settings=None,
           assignment_scale: float = 0.25, enlarge_min_count: int = 25_000,
           renderer: Optional[Callable] = None, return_l_ssim: bool = False):
    """partition.assign (partition.py:348-439): contribution (B1) OR containment
    (B2) per (pose, block); blocks no pose trains retry under enlarged bounds.

    With return_l_ssim the (poses, blocks) matrix of the B1 l_ssim values of
    the first (non-enlarged) pass is returned as well (NaN where not rendered)."""
    if not 0.0 < epsilon < 1.0:
        raise ValueError("epsilon must be in (0, 1)")
    n_blocks = int(np.asarray(grid.bounds_min).shape[0])
    counts = np.asarray(grid.counts)
    views, ids = [], []
    for i, pose in enumerate(poses):
        view, image_id = _pose_view(pose, i)
        views.append(view)
        ids.append(image_id)
    P = len(views)
    entries = np.zeros((P, n_blocks), dtype=bool)
    provenance = np.full((P, n_blocks), "", dtype="<U5")
    bounds_min_used = np.asarray(grid.bounds_min, dtype=np.float64).copy()
    bounds_max_used = np.asarray(grid.bounds_max, dtype=np.float64).copy()
    unassignable = []
    failed = set()

    def mark_failed(i, exc):
        failed.add(i)
        unassignable.append((ids[i], str(exc)))
        entries[i, :] = False
        provenance[i, :] = ""

    scaled_views = [_scaled_camera(v, assignment_scale) for v in views]
    dev_render = renderer is None
    r = _Renderer(cloud, settings) if dev_render else None
    full_images = [None] * P
    for i, scaled in enumerate(scaled_views):
        try:
            full_images[i] = r(scaled) if dev_render else _image_tensor(renderer(cloud, scaled))
        except Exception as exc:  # a broken pose must not sink the batch
            mark_failed(i, exc)

    def rest_image(i, mask_t, rest_host):
        if dev_render:
            return r(scaled_views[i], mask_t)
        return _image_tensor(renderer(rest_host, scaled_views[i]))

    def b1_values(blocks_masks):
        """l_ssim of every (pose, block) in blocks_masks: {j: (mask_t, rest_host)} -> (P, J) array."""
        acc = torch.zeros((P, n_blocks, 4), dtype=torch.float64, device=_dev())
        done = np.zeros((P, n_blocks), dtype=bool)
        for j, (mask_t, rest_host) in blocks_masks.items():
            for i in range(P):
                if i in failed or full_images[i] is None:
                    continue
                try:
                    img = rest_image(i, mask_t, rest_host)
                    if img.shape != full_images[i].shape:
                        raise ValueError("image dimensions differ")
                    _ssim_into(full_images[i], img, acc[i, j])
                    done[i, j] = True
                except Exception as exc:
                    mark_failed(i, exc)
        l = 1.0 - acc[:, :, 3].cpu().numpy()
        l[~done] = np.nan
        return l

    def rest_of(mask_np, mask_t):
        return (mask_t, None if dev_render else cloud.take(np.nonzero(~mask_np)[0]))

    def set_entry(i, j, b1, b2):
        if b1 or b2:
            entries[i, j] = True
            provenance[i, j] = "B1+B2" if (b1 and b2) else ("B1" if b1 else "B2")
        else:
            entries[i, j] = False
            provenance[i, j] = ""

    # first pass: original cells (rest clouds only for occupied blocks, partition.py:374-377)
    membership = np.asarray(grid.membership)
    masks = {}
    for j in range(n_blocks):
        if counts[j] > 0:
            mnp = membership == j
            masks[j] = rest_of(mnp, _mask_for(grid, j, None) if dev_render else None)
    l1 = b1_values(masks)
    for j in range(n_blocks):
        b2 = _centers_in(views, grid, grid.bounds_min[j], grid.bounds_max[j])
        for i in range(P):
            if i in failed:
                continue
            b1 = j in masks and not np.isnan(l1[i, j]) and l1[i, j] > epsilon
            set_entry(i, j, b1, bool(b2[i]))

    # blocks no pose trains: grow their bounds and retry both tests (partition.py:418-432)
    for j in range(n_blocks):
        if entries[:, j].any():
            continue
        lo, hi = enlarge_bounds(j, grid, enlarge_min_count)
        bounds_min_used[j] = lo
        bounds_max_used[j] = hi
        mnp = bounds_contain(grid.contracted, lo, hi)
        if mnp.any():
            lj = b1_values({j: rest_of(mnp, _mask_for(grid, j, (lo, hi)) if dev_render else None)})
        else:
            lj = np.full((P, n_blocks), np.nan)
        b2 = _centers_in(views, grid, lo, hi)
        for i in range(P):
            if i in failed:
                continue
            b1 = not np.isnan(lj[i, j]) and lj[i, j] > epsilon
            set_entry(i, j, b1, bool(b2[i]))

    for i in failed:
        entries[i, :] = False
        provenance[i, :] = ""
    out = AssignmentMatrix(entries=entries, provenance=provenance, bounds_min_used=bounds_min_used,
                           bounds_max_used=bounds_max_used, image_ids=tuple(ids),
                           unassignable=tuple(unassignable))
    return (out, l1) if return_l_ssim else out

"""Drop-in for citysplat.render (render.py:1-286), executed on the B200.

Compatibility tier -- same names, signatures, dataclasses and error
behaviour as the reference:

* ``RenderSettings``  (render.py:37-64)
* ``FrameStats``      (render.py:81-86)
* ``SplatPrimitive``  (render.py:67-78)
* ``project_gaussian``(render.py:191-214)
* ``rasterize_stats`` (render.py:252-280) -> (Image, FrameStats)
* ``rasterize``       (render.py:283-286) -> Image

Device tier -- ``render(...)`` returns the (H, W, 3) float32 CUDA tensor
without a host sync, readback or Image construction; FPS measurements and
training use it (the reference's host Image() alone costs ~50 ms at 1080p,
SURVEY.md section 8b).

Every frame runs the CUDA pipeline in libcsgpu.so (K1..K9, cs_api.h); there
is no CPU path.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib, device
from ._lib import CsFrameStats, CsSource
from ._lib import check as _check
from .core import GaussianCloud, Image

__all__ = ["RenderSettings", "SplatPrimitive", "FrameStats", "project_gaussian", "rasterize",
           "rasterize_stats", "render", "LOW_PASS"]

LOW_PASS = 0.3          # render.py:33
_SINGULAR_DET = 1e-12   # render.py:34


@dataclass(frozen=True)
class RenderSettings:
    background: tuple = (0.0, 0.0, 0.0)
    sh_degree: int = 3
    tile_size: int = 16
    alpha_floor: float = 1.0 / 255.0
    transmittance_floor: float = 1e-4
    near_plane: float = 0.2

    def __post_init__(self):
        object.__setattr__(self, "background", tuple(float(c) for c in self.background))
        if len(self.background) != 3 or any(not 0.0 <= c <= 1.0 for c in self.background):
            raise ValueError("background must be three channels in [0, 1]")
        if self.sh_degree not in (0, 1, 2, 3):
            raise ValueError("sh_degree must be 0..3")
        if self.tile_size < 8:
            raise ValueError("tile_size must be at least 8")
        for name in ("alpha_floor", "transmittance_floor"):
            v = getattr(self, name)
            if not 0.0 < v < 1.0:
                raise ValueError(f"{name} must be in (0, 1)")
        if self.near_plane <= 0:
            raise ValueError("near_plane must be positive")

    @property
    def support_sigmas(self) -> float:
        return math.sqrt(2.0 * math.log(1.0 / self.alpha_floor))


@dataclass(frozen=True)
class SplatPrimitive:
    mean2d: np.ndarray
    cov2d: np.ndarray
    depth: float
    color: np.ndarray
    opacity: float
    source_index: int
    radius: float


@dataclass(frozen=True)
class FrameStats:
    visible_splats: int
    blended_fragments: int
    skipped_singular: int
    wall_ms: float


def _source_for(cloud, dev_index: int, cam=None):
    """(cs_source, keepalive) for a cloud-like object or an AssembledCloud.

    An AssembledCloud is the fixed render set of the camera it was assembled
    for (assemble_render_set returns a concrete cloud, lod.py:360-401): when
    it is rendered from a different camera the selection still runs for the
    assembly camera (cs_source.select_cam)."""
    from .lod import AssembledCloud
    src = CsSource()
    if isinstance(cloud, AssembledCloud):
        src.kind = cloud.source_kind
        src.force_level = -1 if cloud.force_level is None else int(cloud.force_level)
        src.lod = cloud.scene.handle
        sel = device.camera_struct(cloud.cam)
        if cam is not None and bytes(device.camera_struct(cam)) != bytes(sel):
            src.select_cam = ctypes.pointer(sel)
        return src, (cloud, sel)
    dc = device.device_cloud(cloud, dev_index)
    src.kind = _lib.CS_SRC_CLOUD
    src.force_level = -1
    src.cloud = dc.desc()
    return src, dc


def _render_into(cloud, cam, settings, out: torch.Tensor, flags: int, stats: Optional[CsFrameStats]):
    dev_index = out.device.index
    src, keep = _source_for(cloud, dev_index, cam)
    cs_cam = device.camera_struct(cam)
    cs_set = device.settings_struct(settings)
    rc = _lib.load().cs_render(device.context(dev_index), ctypes.byref(src), ctypes.byref(cs_cam),
                               ctypes.byref(cs_set), out.data_ptr(), flags,
                               ctypes.byref(stats) if stats is not None else None,
                               device.stream_handle(out.device))
    _check(rc, "cs_render")
    return keep


def render(cloud, cam, settings: Optional[RenderSettings] = None, *, out: Optional[torch.Tensor] = None,
           device_index: Optional[int] = None, sync: bool = False) -> torch.Tensor:
    """Device tier: enqueue one frame on the current stream; returns the
    clipped (H, W, 3) float32 image tensor.  No host synchronisation.  A frame
    that overflows its tile-pair buffer is reported (MemoryError) by the
    context's next call at the latest -- ``check()`` synchronises and reports
    immediately.  ``sync=True`` renders synchronously, growing the pair
    buffers and re-rendering on overflow (for setup work such as targets)."""
    settings = settings or RenderSettings()
    dev = torch.device("cuda", device._device_index(device_index))
    if out is None:
        out = torch.empty((int(cam.height), int(cam.width), 3), dtype=torch.float32, device=dev)
    _render_into(cloud, cam, settings, out, _lib.CS_RENDER_SYNC if sync else 0, None)
    return out


def rasterize_stats(cloud, cam, settings: Optional[RenderSettings] = None):
    """(Image, FrameStats) exactly as render.rasterize_stats (render.py:252-280).
    wall_ms covers the device frame (selection excluded, as in the reference)
    up to the point the image is complete, before host Image construction."""
    settings = settings or RenderSettings()
    dev = torch.device("cuda", device._device_index())
    start = time.perf_counter()
    out = torch.empty((int(cam.height), int(cam.width), 3), dtype=torch.float64, device=dev)
    stats = CsFrameStats()
    _render_into(cloud, cam, settings, out,
                 _lib.CS_RENDER_SYNC | _lib.CS_RENDER_F64_OUT, stats)
    wall_ms = (time.perf_counter() - start) * 1000.0
    image = Image(out.cpu().numpy())
    return image, FrameStats(visible_splats=int(stats.visible),
                             blended_fragments=int(stats.fragments),
                             skipped_singular=int(stats.skipped_singular), wall_ms=wall_ms)


def check(device_index: Optional[int] = None) -> None:
    """Synchronise the current stream; MemoryError if an asynchronous frame on
    this thread's context overflowed its pair buffer (cs_check)."""
    dev = device._device_index(device_index)
    _lib.check(_lib.load().cs_check(device.context(dev), device.stream_handle(torch.device("cuda", dev))),
               "cs_check")


def rasterize(cloud, cam, settings: Optional[RenderSettings] = None) -> Image:
    image, _ = rasterize_stats(cloud, cam, settings)
    return image


def project_cloud(cloud, cam, settings: Optional[RenderSettings] = None) -> dict:
    """Depth-sorted projection of a cloud (the reference's private
    _Projected, render.py:89-188), computed by the projection kernel and read
    back: means, conics, covs, depths, colors, opacities, radii, source."""
    settings = settings or RenderSettings()
    dev = torch.device("cuda", device._device_index())
    out = torch.empty((1, 1, 3), dtype=torch.float32, device=dev)
    stats = CsFrameStats()
    _render_into(cloud, cam, settings, out, _lib.CS_RENDER_SYNC | _lib.CS_RENDER_PROJECT_ONLY, stats)
    return _dump_projected(dev.index, int(stats.visible), int(stats.skipped_singular))


def _dump_projected(dev_index: int, m: int, skipped: int) -> dict:
    n = max(m, 1)
    res = dict(means=np.zeros((n, 2)), conics=np.zeros((n, 3)), covs=np.zeros((n, 3)),
               depths=np.zeros(n), colors=np.zeros((n, 3)), opacities=np.zeros(n),
               radii=np.zeros((n, 2)), source=np.zeros(n, dtype=np.int64))
    p = lambda k: res[k].ctypes.data
    _check(_lib.load().cs_dump_projected(device.context(dev_index), p("means"), p("conics"),
                                        p("covs"), p("depths"), p("colors"), p("opacities"),
                                        p("radii"), p("source"), device.stream_handle()),
          "cs_dump_projected")
    out = {k: v[:m] for k, v in res.items()}
    out["count"] = m
    out["skipped_singular"] = skipped
    return out


def bin_tiles_last(cam, tile_size: int, dev_index: Optional[int] = None):
    """tile_ids / offsets of this thread's last frame, as render._bin_tiles returns them."""
    dev_index = device._device_index(dev_index)
    st = CsFrameStats()
    lib = _lib.load()
    ctx = device.context(dev_index)
    _check(lib.cs_frame_stats_get(ctx, ctypes.byref(st), device.stream_handle()))
    ntx = (int(cam.width) + tile_size - 1) // tile_size
    nty = (int(cam.height) + tile_size - 1) // tile_size
    tids = np.zeros(max(int(st.pairs), 1), dtype=np.int64)
    offs = np.zeros(ntx * nty + 1, dtype=np.int64)
    _check(lib.cs_dump_tiles(ctx, tids.ctypes.data, offs.ctypes.data, device.stream_handle()))
    return tids[:int(st.pairs)], offs


def project_gaussian(g, cam, settings: Optional[RenderSettings] = None,
                     source_index: int = 0) -> Optional[SplatPrimitive]:
    """render.project_gaussian (render.py:191-214): None when culled."""
    settings = settings or RenderSettings()
    cloud = GaussianCloud(positions=np.asarray(g.position)[None], opacities=[g.opacity],
                          scales=np.asarray(g.scale)[None], rotations=np.asarray(g.rotation)[None],
                          sh=np.asarray(g.sh)[None])
    p = project_cloud(device.DeviceCloud.from_arrays(cloud.positions, cloud.opacities, cloud.scales,
                                                     cloud.rotations, cloud.sh, force_fp64=True),
                      cam, settings)
    if p["count"] == 0:
        return None
    a, b, c = p["covs"][0]
    mid = 0.5 * (a + c)
    lam_max = mid + math.sqrt(max(mid * mid - (a * c - b * b), 0.0))
    # the device colour is float32; recompute it in float64 on the device for the
    # single-primitive API (core.sh_to_colors), direction as render.py:167-168
    d = np.asarray(g.position, dtype=np.float64) - np.asarray(cam.camera_center, dtype=np.float64)
    d = d / np.linalg.norm(d)
    from .core import sh_to_colors
    color = sh_to_colors(np.asarray(g.sh, dtype=np.float64)[None], d[None], settings.sh_degree)[0]
    return SplatPrimitive(
        mean2d=p["means"][0], cov2d=np.array([[a, b], [b, c]]), depth=float(p["depths"][0]),
        color=color, opacity=float(p["opacities"][0]), source_index=source_index,
        radius=settings.support_sigmas * math.sqrt(lam_max))

"""Drop-in for the selection/aggregation half of citysplat.lod (lod.py:150-401).

* ``LodScene``             (lod.py:150-208) -- same fields/validation; uploaded
                           once to HBM (device.DeviceLodScene) on first use.
* ``VisibilityDecision``   (lod.py:255-264)
* ``AssembledSet``         (lod.py:351-357)
* ``block_visible``        (lod.py:267-295)  -> device kernel
* ``select_level``         (lod.py:311-321)  -> device kernel
* ``decide_visibility``    (lod.py:330-348)  -> device kernel (K1)
* ``assemble_render_set``  (lod.py:360-401)  -> segment table on device (K2),
  no concatenation copy.  ``AssembledSet.cloud`` is an ``AssembledCloud``: a
  lazy, device-backed view that duck-types GaussianCloud (``count`` and the
  column arrays, materialised on access) and that ``rasterize_stats``
  recognises and renders straight from the scene in HBM.

Builder half (lod.py:54-248), on the CUDA LoD generator (lodgen.py, cs_lodgen.cu):

* ``significance_scores`` (lod.py:54-101), ``compress`` (lod.py:119-127),
  ``mad_bounds`` (lod.py:130-147), ``build_lod`` (lod.py:211-248) -- same
  signatures and exceptions; ``build_lod`` also leaves the device scene in the
  upload cache, so rendering the returned LodScene does not re-upload it.

Accepts the reference's own LodScene objects as well (duck-typed fields).
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib, device
from ._lib import CsDecision, CsFrameStats, check
from .core import GaussianCloud, pad_sh

__all__ = ["significance_scores", "compress", "mad_bounds", "build_lod",
           "LodScene", "VisibilityDecision", "AssembledSet", "AssembledCloud", "block_visible",
           "select_level", "decide_visibility", "assemble_render_set"]


def _device_settings(settings):
    from .render import RenderSettings
    return settings or RenderSettings()


def significance_scores(cloud, cameras: Sequence, settings=None) -> np.ndarray:
    """lod.significance_scores (lod.py:54-101) on the device; float64 (K,)."""
    from . import lodgen
    if _count(cloud) == 0:
        return np.zeros(0)
    dc = device.device_cloud(cloud)
    return lodgen.significance_scores(dc, cameras, _device_settings(settings)).cpu().numpy()


def _host_cloud(cloud):
    if hasattr(cloud, "take") and hasattr(cloud, "with_sh_degree"):
        return cloud
    return GaussianCloud(np.asarray(cloud.positions, dtype=np.float64),
                         np.asarray(cloud.opacities, dtype=np.float64),
                         np.asarray(cloud.scales, dtype=np.float64),
                         np.asarray(cloud.rotations, dtype=np.float64),
                         np.asarray(cloud.sh, dtype=np.float64))


def compress(cloud, rate: float, sh_degree: int = 3, cameras: Sequence = (), *,
             scores: Optional[np.ndarray] = None):
    """lod.compress (lod.py:119-127): the ceil(rate*K) highest-significance
    Gaussians in their original order, SH bands above sh_degree dropped."""
    from . import lodgen
    k = _count(cloud)
    keep = lodgen.keep_count(rate, k)
    if scores is None:
        sc = lodgen.significance_scores(device.device_cloud(cloud), cameras) if k else None
    else:
        sc = torch.as_tensor(np.asarray(scores, dtype=np.float64), device=device.default_device())
    if k == 0:
        return _host_cloud(cloud).take(np.zeros(0, dtype=np.int64)).with_sh_degree(sh_degree)
    order = lodgen.priority(sc)
    kept = torch.sort(order[:keep].long()).values.cpu().numpy()
    return _host_cloud(cloud).take(kept).with_sh_degree(sh_degree)


def mad_bounds(block_cloud, n_mad: float) -> Tuple[np.ndarray, np.ndarray]:
    """lod.mad_bounds (lod.py:130-147) on the device."""
    from . import lodgen
    if _count(block_cloud) == 0:
        raise ValueError("bounds of an empty block are undefined")
    if not n_mad > 0:
        raise ValueError("n_mad must be positive")
    dc = device.device_cloud(block_cloud)
    mem = torch.zeros(dc.count, dtype=torch.int32, device=dc.device)
    lo, hi = lodgen.block_bounds(dc, mem, 1, n_mad)
    return lo[0], hi[0]


def build_lod(cloud, grid, cameras: Sequence, config) -> "LodScene":
    """lod.build_lod (lod.py:211-248): every detail level of a partitioned scene."""
    from . import lodgen
    from .core import GaussianCloud
    dc = device.device_cloud(cloud)
    n_blocks = int(grid.n_blocks)
    mem = torch.as_tensor(np.asarray(grid.membership).astype(np.int32), device=dc.device)
    dscene = lodgen.build_lod_cloud(dc, mem, n_blocks, cameras, config.distance_intervals,
                                    config.compression_rates, config.lod_sh_degrees,
                                    float(config.n_mad))
    levels = []
    for L in range(dscene.n_levels):
        blocks = []
        for j in range(n_blocks):
            a = dscene.block_cloud_host(L, j)
            blocks.append(GaussianCloud(a["positions"], a["opacities"], a["scales"],
                                        a["rotations"], a["sh"]))
        levels.append(tuple(blocks))
    scene = LodScene(levels=tuple(levels), bounds_min=dscene.bounds_min,
                     bounds_max=dscene.bounds_max, distance_intervals=config.distance_intervals,
                     sh_degrees=dscene.sh_degrees, n_mad=float(config.n_mad), full=cloud)
    device.prime_lod_cache(scene, dscene)
    return scene


@dataclass(frozen=True)
class LodScene:
    """levels[L][j]: block j at level L (0 = coarsest); intervals nearest-first."""

    levels: tuple
    bounds_min: np.ndarray
    bounds_max: np.ndarray
    distance_intervals: tuple
    sh_degrees: tuple
    n_mad: float
    full: object

    def __post_init__(self):
        levels = tuple(tuple(level) for level in self.levels)
        object.__setattr__(self, "levels", levels)
        object.__setattr__(self, "distance_intervals",
                           tuple((float(a), float(b)) for a, b in self.distance_intervals))
        object.__setattr__(self, "sh_degrees", tuple(int(d) for d in self.sh_degrees))
        if not levels:
            raise ValueError("at least one level required")
        n_blocks = len(levels[0])
        if any(len(level) != n_blocks for level in levels):
            raise ValueError("every level must carry the same block set")
        if len(self.distance_intervals) != len(levels):
            raise ValueError("one distance interval per level required")
        if len(self.sh_degrees) != len(levels):
            raise ValueError("one sh_degree per level required")
        bmin = np.asarray(self.bounds_min, dtype=np.float64).reshape(n_blocks, 3)
        bmax = np.asarray(self.bounds_max, dtype=np.float64).reshape(n_blocks, 3)
        if not (np.isfinite(bmin).all() and np.isfinite(bmax).all()):
            raise ValueError("block bounds must be finite")
        object.__setattr__(self, "bounds_min", bmin)
        object.__setattr__(self, "bounds_max", bmax)

    @property
    def n_levels(self) -> int:
        return len(self.levels)

    @property
    def n_blocks(self) -> int:
        return len(self.levels[0])

    @property
    def finest(self) -> int:
        return self.n_levels - 1

    def level_size(self, level: int) -> int:
        return sum(_count(c) for c in self.levels[level])

    def occupied(self, j: int) -> bool:
        return _count(self.levels[self.finest][j]) > 0


def _count(c) -> int:
    return int(c.count) if hasattr(c, "count") else int(np.asarray(c.positions).shape[0])


@dataclass(frozen=True)
class VisibilityDecision:
    block: int
    visible: bool
    level: Optional[int]
    distance: float
    screen_box: Optional[tuple]


class AssembledSet:
    """AssembledSet (lod.py:351-357): ``cloud``, ``decisions``, ``selection_ms``.

    Block mode is lazy: the selection itself runs inside the frame that
    renders ``cloud`` (K1 in cs_render), so assembling costs no device round
    trip; ``decisions`` and ``cloud.count`` are computed (one synchronous
    K1 launch) only when read.  ``selection_ms`` is the host time of the
    assembly call."""

    __slots__ = ("cloud", "selection_ms", "_decisions")

    def __init__(self, cloud, decisions, selection_ms: float):
        self.cloud = cloud
        self.selection_ms = float(selection_ms)
        self._decisions = decisions

    @property
    def decisions(self) -> tuple:
        if self._decisions is None:
            self._decisions = self.cloud._resolve()[0]
        return self._decisions

    def __repr__(self):
        return f"AssembledSet(count={self.cloud.count}, selection_ms={self.selection_ms:.3f})"


class AssembledCloud:
    """The concatenated render set of one frame, kept on the device.

    Holds the scene handle plus the selection parameters; rendering it runs
    the selection kernel again inside the frame (it is deterministic, so the
    set is identical).  Column arrays are gathered to the host only when read.
    """

    def __init__(self, scene: device.DeviceLodScene, cam, mode: str, force_level, count, pieces):
        self.scene = scene
        self.cam = cam
        self.mode = mode
        self.force_level = force_level
        self._count = None if count is None else int(count)
        self._pieces = pieces  # [(level, block)] in assembled order (block mode); None until resolved
        self._decisions = None
        self._host = None
        self.source_kind = _lib.CS_SRC_LOD_BLOCK if mode == "block" else _lib.CS_SRC_LOD_POINT

    def _resolve(self):
        """(decisions, pieces, count) of a block-mode set, computed once."""
        if self._decisions is None:
            decisions = _decisions(self.scene, self.cam, self.force_level)
            self._pieces = [(d.level, d.block) for d in decisions
                            if d.visible and 0 <= d.level < self.scene.n_levels
                            and self.scene.counts[d.level, d.block] > 0]
            self._count = int(sum(self.scene.counts[L, j] for L, j in self._pieces))
            self._decisions = decisions
        return self._decisions, self._pieces, self._count

    @property
    def count(self) -> int:
        if self._count is None:
            self._resolve()
        return self._count

    def __len__(self) -> int:
        return self._count

    def _materialise(self):
        if self._host is None:
            if self.mode == "block":
                parts = [self.scene.block_cloud_host(L, j) for L, j in self._resolve()[1]]
            else:
                parts = _pointwise_host(self.scene, self.cam, self.force_level)
            if not parts:
                self._host = GaussianCloud.empty()
            else:
                width = max(p["sh"].shape[2] for p in parts)
                self._host = GaussianCloud(
                    np.concatenate([p["positions"] for p in parts]),
                    np.concatenate([p["opacities"] for p in parts]),
                    np.concatenate([p["scales"] for p in parts]),
                    np.concatenate([p["rotations"] for p in parts]),
                    np.concatenate([pad_sh(p["sh"], width) for p in parts]))
        return self._host

    positions = property(lambda self: self._materialise().positions)
    opacities = property(lambda self: self._materialise().opacities)
    scales = property(lambda self: self._materialise().scales)
    rotations = property(lambda self: self._materialise().rotations)
    sh = property(lambda self: self._materialise().sh)

    def to_cloud(self) -> GaussianCloud:
        return self._materialise()


def _pointwise_host(scene, cam, force_level):
    """Host copy of a pointwise render set: the device selection's packed
    (cloud << 40 | row) list, gathered from the level buffers."""
    n = _pointwise_count(scene, cam, force_level)
    packed = np.zeros(max(n, 1), dtype=np.uint64)
    got = ctypes.c_int64(0)
    check(_lib.load().cs_dump_assembled_list(device.context(scene.device_index), packed.ctypes.data,
                                             n, ctypes.byref(got), device.stream_handle()))
    packed = packed[:got.value]
    if packed.size == 0:
        return []
    cloud = (packed >> np.uint64(40)).astype(np.int64)
    row = (packed & np.uint64((1 << 40) - 1)).astype(np.int64)
    J = scene.n_blocks
    parts = []
    # runs of equal cloud index are contiguous (level-major, block order)
    cuts = np.flatnonzero(np.diff(cloud)) + 1
    for seg in np.split(np.arange(packed.size), cuts):
        ci = int(cloud[seg[0]])
        L, j = divmod(ci, J)
        host = scene.block_cloud_host(L, j)
        rows = row[seg]
        parts.append({k: v[rows] for k, v in host.items()})
    return parts


def block_visible(bounds, cam) -> Tuple[bool, float]:
    """lod.block_visible (lod.py:267-295) on the device."""
    lo = np.ascontiguousarray(np.asarray(bounds[0], dtype=np.float64).reshape(1, 3))
    hi = np.ascontiguousarray(np.asarray(bounds[1], dtype=np.float64).reshape(1, 3))
    vis = np.zeros(1, dtype=np.uint8)
    dist = np.zeros(1)
    c = device.camera_struct(cam)
    check(_lib.load().cs_block_visible(device.context(), 1, lo.ctypes.data, hi.ctypes.data,
                                       ctypes.byref(c), vis.ctypes.data, dist.ctypes.data,
                                       device.stream_handle()), "block_visible")
    return bool(vis[0]), float(dist[0])


def select_level(distance: float, intervals: Sequence) -> int:
    """lod.select_level (lod.py:311-321) on the device."""
    d = np.array([float(distance)])
    iv = np.ascontiguousarray(np.array([(float(a), float(b)) for a, b in intervals]).reshape(-1, 2))
    out = np.zeros(1, dtype=np.int32)
    rc = _lib.load().cs_select_level(device.context(), 1, d.ctypes.data, iv.shape[0],
                                     iv.ctypes.data, out.ctypes.data, device.stream_handle())
    if rc == _lib.CS_EINVAL:
        raise ValueError("distance must be nonnegative")
    if rc == _lib.CS_ERANGE:
        raise ValueError(f"no interval covers distance {float(distance)}")
    check(rc, "select_level")
    return int(out[0])


def _decisions(dscene: device.DeviceLodScene, cam, force_level) -> tuple:
    J = dscene.n_blocks
    arr = (CsDecision * J)()
    c = device.camera_struct(cam)
    rc = _lib.load().cs_decide_visibility(device.context(dscene.device_index), dscene.handle,
                                          ctypes.byref(c), -1 if force_level is None else int(force_level),
                                          arr, device.stream_handle())
    if rc == _lib.CS_ERANGE:
        raise ValueError("no interval covers a block distance")
    check(rc, "decide_visibility")
    out = []
    for j in range(J):
        d = arr[j]
        vis = bool(d.visible)
        out.append(VisibilityDecision(
            block=j, visible=vis, level=int(d.level) if vis else None,
            distance=float(d.distance),
            screen_box=tuple(float(v) for v in d.box) if d.has_box else None))
    return tuple(out)


def decide_visibility(scene, cam, force_level: Optional[int] = None) -> tuple:
    """lod.decide_visibility (lod.py:330-348) -> tuple of VisibilityDecision."""
    return _decisions(device.device_lod_scene(scene), cam, force_level)


def assemble_render_set(scene, cam, *, mode: str = "block",
                        force_level: Optional[int] = None) -> AssembledSet:
    """lod.assemble_render_set (lod.py:360-401) without the concatenation copy."""
    dscene = device.device_lod_scene(scene)
    start = time.perf_counter()
    if mode == "block":
        # lazy: the frame that renders the set runs the selection (K1).  Eager
        # when select_level could fail (intervals not covering [0, inf) without
        # gaps), so its ValueError surfaces here as in the reference.
        if force_level is not None and not 0 <= int(force_level) < dscene.n_levels:
            raise ValueError(f"force_level {force_level} outside the scene's levels")
        cloud = AssembledCloud(dscene, cam, mode, force_level, None, None)
        if force_level is None and not _covers_half_line(dscene.distance_intervals):
            cloud._resolve()
        return AssembledSet(cloud=cloud, decisions=cloud._decisions,
                            selection_ms=(time.perf_counter() - start) * 1000.0)
    elif mode == "pointwise":
        decisions = ()
        pieces = None
        count = _pointwise_count(dscene, cam, force_level)
    else:
        raise ValueError(f"unknown selection mode: {mode}")
    selection_ms = (time.perf_counter() - start) * 1000.0
    cloud = AssembledCloud(dscene, cam, mode, force_level, count, pieces)
    return AssembledSet(cloud=cloud, decisions=decisions, selection_ms=selection_ms)


def _covers_half_line(intervals) -> bool:
    """True when every distance >= 0 falls in exactly one [lo, hi) interval."""
    iv = sorted((float(a), float(b)) for a, b in intervals)
    if not iv or iv[0][0] > 0.0 or iv[-1][1] != math.inf:
        return False
    return all(iv[i][1] == iv[i + 1][0] for i in range(len(iv) - 1))


def _pointwise_count(dscene, cam, force_level) -> int:
    from ._lib import CsSource
    from .render import RenderSettings
    src = CsSource()
    src.kind = _lib.CS_SRC_LOD_POINT
    src.force_level = -1 if force_level is None else int(force_level)
    src.lod = dscene.handle
    out = torch.empty((1, 1, 3), dtype=torch.float32, device=torch.device("cuda", dscene.device_index))
    stats = CsFrameStats()
    c = device.camera_struct(cam)
    s = device.settings_struct(RenderSettings())
    check(_lib.load().cs_render(device.context(dscene.device_index), ctypes.byref(src), ctypes.byref(c),
                                ctypes.byref(s), out.data_ptr(),
                                _lib.CS_RENDER_SYNC | _lib.CS_RENDER_PROJECT_ONLY,
                                ctypes.byref(stats), device.stream_handle()), "pointwise")
    return int(stats.assembled)

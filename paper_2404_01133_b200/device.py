"""Device residency: contexts, HBM-resident clouds and LoD scenes.

* One ``cs_ctx`` per (thread, device): the C side is re-entrant per context,
  ctypes releases the GIL, so service threads render concurrently
  (the reference renders on threads without a lock, service.py:213-223).
* ``DeviceCloud`` keeps one GaussianCloud in HBM as 16-byte quads
  (x, y, z, opacity), (sx, sy, sz, 0), (w, x, y, z) plus float32 SH rows.
  Geometry is stored in float32 when every decision input is exactly
  representable (then the float64 device math sees identical values), else in
  float64 -- the bit-exact contract never depends on a lossy cast.
* ``DeviceLodScene`` keeps every level's blocks contiguous per level
  (levels[L] concatenated in block order) and registers the (level, block)
  descriptor table with the C side once (cs_lod_create).
* Host clouds are immutable (core.py:59-64), so uploads are cached per object.

torch is used only for device memory and the current stream.
"""

from __future__ import annotations

import ctypes
import math
import threading
import weakref
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import CsCamera, CsCloud, CsLodDesc, CsSettings, check

_tls = threading.local()
_ctx_lock = threading.Lock()
_all_ctx = []


def _device_index(device=None) -> int:
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2404_01133_b200 needs a CUDA device (sm_100a); none is visible")
        return torch.cuda.current_device()
    return torch.device(device).index or 0


def context(device=None) -> ctypes.c_void_p:
    """The calling thread's cs_ctx for `device` (created on first use)."""
    dev = _device_index(device)
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    h = ctxs.get(dev)
    if h is None:
        lib = _lib.load()
        h = ctypes.c_void_p()
        torch.cuda.init()
        check(lib.cs_create(dev, ctypes.byref(h)), "cs_create")
        ctxs[dev] = h
        with _ctx_lock:
            _all_ctx.append(h)
    return h


def stream_handle(device=None) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def camera_struct(cam) -> CsCamera:
    c = CsCamera()
    R = np.asarray(cam.rotation_w2c, dtype=np.float64).reshape(9)
    t = np.asarray(cam.translation_w2c, dtype=np.float64).reshape(3)
    center = np.asarray(cam.camera_center, dtype=np.float64).reshape(3)
    c.R[:] = R.tolist()
    c.t[:] = t.tolist()
    c.center[:] = center.tolist()
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    return c


def settings_struct(settings) -> CsSettings:
    s = CsSettings()
    s.background[:] = [float(v) for v in settings.background]
    s.alpha_floor = float(settings.alpha_floor)
    s.transmittance_floor = float(settings.transmittance_floor)
    s.near_plane = float(settings.near_plane)
    s.support_sigmas = math.sqrt(2.0 * math.log(1.0 / s.alpha_floor))  # render.py:61-64
    s.low_pass = 0.3           # LOW_PASS, render.py:33
    s.singular_det = 1e-12     # _SINGULAR_DET, render.py:34
    s.sh_degree = int(settings.sh_degree)
    s.tile_size = int(settings.tile_size)
    return s


def _f32_exact(*arrays) -> bool:
    for a in arrays:
        a = np.asarray(a, dtype=np.float64)
        if a.size and not np.array_equal(a.astype(np.float32).astype(np.float64), a):
            return False
    return True


def sh_stride(coeffs: int) -> int:
    return (3 * coeffs + 3) // 4 * 4


class DeviceCloud:
    """A GaussianCloud resident in HBM (see module docstring for the layout)."""

    def __init__(self, pos_op: torch.Tensor, scale: torch.Tensor, quat: torch.Tensor,
                 sh: torch.Tensor, sh_coeffs: int, count: int):
        self.pos_op, self.scale, self.quat, self.sh = pos_op, scale, quat, sh
        self.sh_coeffs = int(sh_coeffs)
        self._count = int(count)
        self.fp64 = pos_op.dtype == torch.float64

    @property
    def count(self) -> int:
        return self._count

    @property
    def device(self):
        return self.pos_op.device

    def desc(self, offset: int = 0, count: Optional[int] = None) -> CsCloud:
        """cs_cloud for rows [offset, offset + count)."""
        n = self._count - offset if count is None else int(count)
        d = CsCloud()
        es = self.pos_op.element_size() * 4
        d.pos_op = self.pos_op.data_ptr() + offset * es
        d.scale = self.scale.data_ptr() + offset * es
        d.quat = self.quat.data_ptr() + offset * es
        d.sh = self.sh.data_ptr() + offset * self.sh.shape[1] * 4
        d.count = n
        d.sh_coeffs = self.sh_coeffs
        d.sh_stride = int(self.sh.shape[1])
        d.fp64 = 1 if self.fp64 else 0
        return d

    @classmethod
    def from_arrays(cls, positions, opacities, scales, rotations, sh, device=None,
                    force_fp64: bool = False, sh_width: Optional[int] = None) -> "DeviceCloud":
        dev = torch.device("cuda", _device_index(device))
        pos = np.asarray(positions)
        k = int(pos.shape[0])
        shn = np.asarray(sh)
        C = int(shn.shape[2]) if shn.ndim == 3 else 1
        width = int(sh_width or C)
        fp32 = (not force_fp64) and _f32_exact(positions, opacities, scales, rotations)
        dt = np.float32 if fp32 else np.float64
        quads = np.zeros((3, k, 4), dtype=dt)
        quads[0, :, :3] = np.asarray(positions).reshape(k, 3)
        quads[0, :, 3] = np.asarray(opacities).reshape(k)
        quads[1, :, :3] = np.asarray(scales).reshape(k, 3)
        quads[2] = np.asarray(rotations).reshape(k, 4)
        stride = sh_stride(width)
        rows = np.zeros((k, stride), dtype=np.float32)
        if k:
            src = np.zeros((k, 3, width), dtype=np.float32)
            src[:, :, :C] = shn.reshape(k, 3, C)
            rows[:, :3 * width] = src.reshape(k, 3 * width)
        t = torch.from_numpy(quads).to(dev, non_blocking=False)
        shd = torch.from_numpy(rows).to(dev)
        return cls(t[0], t[1], t[2], shd, width, k)

    @classmethod
    def from_torch(cls, positions: torch.Tensor, opacities: torch.Tensor, scales: torch.Tensor,
                   rotations: torch.Tensor, sh: torch.Tensor) -> "DeviceCloud":
        """Pack device tensors (K,3),(K,),(K,3),(K,4),(K,3,C) into quads (any float dtype:
        float64 keeps float64 geometry, anything else is stored as float32)."""
        k = positions.shape[0]
        dt = torch.float64 if positions.dtype == torch.float64 else torch.float32
        dev = positions.device
        quads = torch.zeros((3, k, 4), dtype=dt, device=dev)
        quads[0, :, :3] = positions
        quads[0, :, 3] = opacities.reshape(k)
        quads[1, :, :3] = scales
        quads[2] = rotations
        C = sh.shape[2]
        stride = sh_stride(C)
        rows = torch.zeros((k, stride), dtype=torch.float32, device=dev)
        rows[:, :3 * C] = sh.reshape(k, 3 * C).to(torch.float32)
        return cls(quads[0], quads[1], quads[2], rows, C, k)


_cloud_cache: dict = {}
_cache_lock = threading.Lock()


def _cached(obj, key, build):
    """Upload cache keyed by object identity (host clouds are immutable)."""
    k = (id(obj), key)
    with _cache_lock:
        hit = _cloud_cache.get(k)
        if hit is not None and hit[0]() is obj:
            return hit[1]
    val = build()
    try:
        ref = weakref.ref(obj, lambda _r, k=k: _cloud_cache.pop(k, None))
    except TypeError:
        return val
    with _cache_lock:
        _cloud_cache[k] = (ref, val)
    return val


def device_cloud(cloud, device=None) -> DeviceCloud:
    """DeviceCloud for any object with the GaussianCloud fields."""
    if isinstance(cloud, DeviceCloud):
        return cloud
    dev = _device_index(device)
    return _cached(cloud, ("cloud", dev), lambda: DeviceCloud.from_arrays(
        cloud.positions, cloud.opacities, cloud.scales, cloud.rotations, cloud.sh, dev))


class DeviceLodScene:
    """LodScene (lod.py:150-208) resident in HBM with its C-side handle."""

    def __init__(self, levels, bounds_min, bounds_max, distance_intervals, sh_degrees,
                 device=None, full=None):
        self.device_index = _device_index(device)
        self.n_levels = len(levels)
        self.n_blocks = len(levels[0])
        self.bounds_min = np.ascontiguousarray(bounds_min, dtype=np.float64).reshape(self.n_blocks, 3)
        self.bounds_max = np.ascontiguousarray(bounds_max, dtype=np.float64).reshape(self.n_blocks, 3)
        self.distance_intervals = tuple((float(a), float(b)) for a, b in distance_intervals)
        self.sh_degrees = tuple(int(d) for d in sh_degrees)
        self.level_clouds = []     # one DeviceCloud per level (blocks concatenated)
        self.block_offsets = []    # [L][j] row offset inside the level cloud
        self.counts = np.zeros((self.n_levels, self.n_blocks), dtype=np.int64)
        self.full = full
        descs = (CsCloud * (self.n_levels * self.n_blocks))()
        self._levels_src = levels
        self._build(descs)
        del self._levels_src
        self._descs = descs
        ints = np.ascontiguousarray(np.array(self.distance_intervals, dtype=np.float64).reshape(-1, 2))
        if ints.shape[0] != self.n_levels:
            raise ValueError("one distance interval per level required")
        self._ints = ints
        d = CsLodDesc()
        d.n_levels = self.n_levels
        d.n_blocks = self.n_blocks
        d.clouds = ctypes.cast(descs, ctypes.POINTER(CsCloud))
        d.bounds_min = self.bounds_min.ctypes.data_as(_lib.c_double_p)
        d.bounds_max = self.bounds_max.ctypes.data_as(_lib.c_double_p)
        d.intervals = ints.ctypes.data_as(_lib.c_double_p)
        h = ctypes.c_void_p()
        check(_lib.load().cs_lod_create(context(self.device_index), ctypes.byref(d),
                                        ctypes.byref(h)), "cs_lod_create")
        self.handle = h
        self._finalizer = weakref.finalize(self, _lib.load().cs_lod_destroy, h)

    def _build(self, descs):
        levels = self._levels_src
        J = self.n_blocks
        self.level_clouds = []
        self.block_offsets = []
        for L, blocks in enumerate(levels):
            if len(blocks) != J:
                raise ValueError("every level must carry the same block set")
            if all(isinstance(b, DeviceCloud) for b in blocks) and len(blocks) == 1:
                lc = blocks[0]
                offs = [0]
            else:
                arrs = [(np.asarray(b.positions), np.asarray(b.opacities), np.asarray(b.scales),
                         np.asarray(b.rotations), np.asarray(b.sh)) for b in blocks]
                width = max(a[4].shape[2] for a in arrs)
                offs = np.cumsum([0] + [a[0].shape[0] for a in arrs])[:-1].tolist()
                cat = lambda i: np.concatenate([a[i] for a in arrs]) if arrs else np.zeros((0, 3))
                sh = np.concatenate([_pad_sh(a[4], width) for a in arrs])
                lc = DeviceCloud.from_arrays(cat(0), cat(1), cat(2), cat(3), sh, self.device_index)
            self.level_clouds.append(lc)
            self.block_offsets.append(offs)
            for j, b in enumerate(blocks):
                n = int(np.asarray(b.positions).shape[0]) if not isinstance(b, DeviceCloud) else b.count
                self.counts[L, j] = n
                descs[L * J + j] = lc.desc(offs[j], n)

    @classmethod
    def from_device_levels(cls, level_clouds, counts, bounds_min, bounds_max, distance_intervals,
                           sh_degrees, device=None, full=None) -> "DeviceLodScene":
        """Build from per-level DeviceClouds whose rows are grouped by block
        (counts[L][j] rows of block j, in block order)."""
        self = cls.__new__(cls)
        self.device_index = _device_index(device)
        self.n_levels = len(level_clouds)
        counts = np.asarray(counts, dtype=np.int64)
        self.n_blocks = counts.shape[1]
        self.bounds_min = np.ascontiguousarray(bounds_min, dtype=np.float64).reshape(self.n_blocks, 3)
        self.bounds_max = np.ascontiguousarray(bounds_max, dtype=np.float64).reshape(self.n_blocks, 3)
        self.distance_intervals = tuple((float(a), float(b)) for a, b in distance_intervals)
        self.sh_degrees = tuple(int(d) for d in sh_degrees)
        self.level_clouds = list(level_clouds)
        self.counts = counts
        self.full = full
        J = self.n_blocks
        descs = (CsCloud * (self.n_levels * J))()
        self.block_offsets = []
        for L, lc in enumerate(level_clouds):
            offs = np.concatenate([[0], np.cumsum(counts[L])[:-1]]).astype(np.int64).tolist()
            self.block_offsets.append(offs)
            for j in range(J):
                descs[L * J + j] = lc.desc(int(offs[j]), int(counts[L, j]))
        self._descs = descs
        ints = np.ascontiguousarray(np.array(self.distance_intervals, dtype=np.float64).reshape(-1, 2))
        self._ints = ints
        d = CsLodDesc()
        d.n_levels = self.n_levels
        d.n_blocks = J
        d.clouds = ctypes.cast(descs, ctypes.POINTER(CsCloud))
        d.bounds_min = self.bounds_min.ctypes.data_as(_lib.c_double_p)
        d.bounds_max = self.bounds_max.ctypes.data_as(_lib.c_double_p)
        d.intervals = ints.ctypes.data_as(_lib.c_double_p)
        h = ctypes.c_void_p()
        check(_lib.load().cs_lod_create(context(self.device_index), ctypes.byref(d),
                                        ctypes.byref(h)), "cs_lod_create")
        self.handle = h
        self._finalizer = weakref.finalize(self, _lib.load().cs_lod_destroy, h)
        return self

    @property
    def finest(self) -> int:
        return self.n_levels - 1

    def occupied(self, j: int) -> bool:
        return bool(self.counts[self.finest, j] > 0)

    def level_size(self, level: int) -> int:
        return int(self.counts[level].sum())

    def block_cloud_host(self, level: int, j: int):
        """Materialise levels[level][j] on the host (arrays as stored on device)."""
        lc = self.level_clouds[level]
        o = int(self.block_offsets[level][j])
        n = int(self.counts[level, j])
        return _host_arrays(lc, o, n)


def _pad_sh(sh, width):
    sh = np.asarray(sh)
    if sh.shape[2] == width:
        return sh
    out = np.zeros(sh.shape[:2] + (width,), dtype=sh.dtype)
    out[:, :, :sh.shape[2]] = sh
    return out


def _host_arrays(lc: DeviceCloud, o: int, n: int):
    q = lambda t: t[o:o + n].double().cpu().numpy()
    pos_op = q(lc.pos_op)
    C = lc.sh_coeffs
    sh = lc.sh[o:o + n, :3 * C].double().cpu().numpy().reshape(n, 3, C)
    return dict(positions=pos_op[:, :3], opacities=pos_op[:, 3], scales=q(lc.scale)[:, :3],
                rotations=q(lc.quat), sh=sh)


def prime_lod_cache(scene, dscene: DeviceLodScene) -> None:
    """Register an already-built DeviceLodScene for the host LodScene `scene`."""
    _cached(scene, ("lod", dscene.device_index), lambda: dscene)


def default_device() -> torch.device:
    return torch.device("cuda", _device_index(None))


def device_lod_scene(scene, device=None) -> DeviceLodScene:
    if isinstance(scene, DeviceLodScene):
        return scene
    dev = _device_index(device)
    return _cached(scene, ("lod", dev), lambda: DeviceLodScene(
        scene.levels, scene.bounds_min, scene.bounds_max, scene.distance_intervals,
        scene.sh_degrees, dev, full=getattr(scene, "full", None)))


# ---------------------------------------------------------------------------
# small device utilities used by the core API mirror


def build_covariances(scales: np.ndarray, quats: np.ndarray) -> np.ndarray:
    n = scales.shape[0]
    dev = torch.device("cuda", _device_index())
    s = torch.from_numpy(np.ascontiguousarray(scales.reshape(n, 3))).to(dev)
    q = torch.from_numpy(np.ascontiguousarray(quats.reshape(n, 4))).to(dev)
    out = torch.empty((n, 3, 3), dtype=torch.float64, device=dev)
    check(_lib.load().cs_build_covariances(context(), n, s.data_ptr(), q.data_ptr(),
                                           out.data_ptr(), stream_handle()))
    return out.cpu().numpy()


def sh_to_colors(sh: np.ndarray, dirs: np.ndarray, degree: int) -> np.ndarray:
    n = sh.shape[0]
    dev = torch.device("cuda", _device_index())
    s = torch.from_numpy(np.ascontiguousarray(sh)).to(dev)
    d = torch.from_numpy(np.ascontiguousarray(dirs.reshape(n, 3))).to(dev)
    out = torch.empty((n, 3), dtype=torch.float64, device=dev)
    check(_lib.load().cs_sh_to_colors(context(), n, s.data_ptr(), sh.shape[2], d.data_ptr(),
                                      degree, out.data_ptr(), stream_handle()))
    return out.cpu().numpy()

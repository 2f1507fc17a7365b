"""RenderService drop-in (service.py:114-238) over the device-resident scene
(SURVEY.md 8f row f4).

Same request handling as the reference's ``RenderService`` -- camera JSON
validation naming the broken field (``camera_from_json``, service.py:59-88),
the ``max_dim`` 413 guard, per-request LoD overrides that do not persist,
atomic interval / enable swaps (``update_lod``), ``scene_info`` /
``block_geometry`` metadata and the ``last_stats`` payload
(``_stats_payload``, service.py:91-112) -- but a frame is: block selection and
rasterisation by ``cs_render`` on the scene uploaded once to HBM, the
float64 image quantised to 8 bits on the device (``rint(255 x)`` clipped,
images.to_uint8), and only the 8-bit frame read back for the PNG encoder
(PIL, as images.encode_png).  Interval overrides reuse the resident level
buffers through a second selection table (no re-upload).

``render_ms`` covers selection + rasterisation up to the finished device
image, like the reference's timer (service.py:213-223) minus its host Image
construction; readback and PNG encoding are outside it.  The HTTP layer
(``create_app``, FastAPI) is networking and out of scope.
"""

from __future__ import annotations

import ctypes
import io
import math
import threading
import time
from collections import OrderedDict
from typing import Optional

import numpy as np

from .core import CameraView

__all__ = ["RenderService", "BadRequest", "Oversized", "ConfigError", "camera_from_json",
           "validate_intervals", "encode_png", "to_uint8", "MAX_DIM_DEFAULT"]

MAX_DIM_DEFAULT = 1920  # service.py:33


class ConfigError(ValueError):
    """errors.ConfigError: invalid run configuration."""


class BadRequest(Exception):
    """service._BadRequest: a 400 naming the offending field."""

    def __init__(self, field: str, message: str):
        super().__init__(message)
        self.field = field


class Oversized(Exception):
    """service._Oversized: a 413 (image larger than max_dim)."""

    def __init__(self, max_dim: int):
        super().__init__(f"image dimensions exceed the configured maximum {max_dim}")
        self.max_dim = max_dim


def validate_intervals(intervals) -> None:
    """config.validate_intervals (config.py:37-51)."""
    iv = tuple((float(a), float(b)) for a, b in intervals)
    if not iv:
        raise ConfigError("at least one distance interval is required")
    if iv[0][0] != 0.0:
        raise ConfigError("the first distance interval must start at 0")
    if iv[-1][1] != math.inf:
        raise ConfigError("the last distance interval must be unbounded")
    for (lo, hi), (lo2, _) in zip(iv, iv[1:]):
        if hi != lo2:
            raise ConfigError("distance intervals must be contiguous and non-overlapping")
    if any(not lo < hi for lo, hi in iv):
        raise ConfigError("distance intervals must be ascending")


def _json_intervals(intervals) -> list:
    # JSON has no Infinity literal: an unbounded upper edge travels as null
    return [[lo, hi if math.isfinite(hi) else None] for lo, hi in intervals]


def _number(body: dict, field: str) -> float:
    try:
        v = float(body[field])
    except KeyError:
        raise BadRequest(f"camera.{field}", "missing required field") from None
    except (TypeError, ValueError):
        raise BadRequest(f"camera.{field}", "must be a number") from None
    if not math.isfinite(v):
        raise BadRequest(f"camera.{field}", "must be finite")
    return v


def camera_from_json(body) -> CameraView:
    """service.camera_from_json (service.py:59-88)."""
    if not isinstance(body, dict):
        raise BadRequest("camera", "must be an object")
    width = _number(body, "width")
    height = _number(body, "height")
    if width != int(width) or height != int(height):
        raise BadRequest("camera.width", "dimensions must be integers")
    try:
        rotation = np.asarray(body["rotation"], dtype=np.float64).reshape(3, 3)
    except KeyError:
        raise BadRequest("camera.rotation", "missing required field") from None
    except (TypeError, ValueError):
        raise BadRequest("camera.rotation", "must be a 3x3 matrix") from None
    try:
        translation = np.asarray(body["translation"], dtype=np.float64).reshape(3)
    except KeyError:
        raise BadRequest("camera.translation", "missing required field") from None
    except (TypeError, ValueError):
        raise BadRequest("camera.translation", "must be a 3-vector") from None
    try:
        return CameraView(width=int(width), height=int(height),
                          fx=_number(body, "fx"), fy=_number(body, "fy"),
                          cx=_number(body, "cx"), cy=_number(body, "cy"),
                          rotation_w2c=rotation, translation_w2c=translation)
    except ValueError as exc:
        raise BadRequest("camera", str(exc)) from None


def to_uint8(pixels) -> np.ndarray:
    """images.to_uint8 (images.py:16-17) for host arrays."""
    return np.clip(np.rint(np.asarray(pixels) * 255.0), 0, 255).astype(np.uint8)


def encode_png(pixels_u8: np.ndarray) -> bytes:
    """images.encode_png (images.py:20-25) from an already quantised frame."""
    from PIL import Image as PilImage
    buf = io.BytesIO()
    PilImage.fromarray(np.ascontiguousarray(pixels_u8), mode="RGB").save(buf, format="PNG")
    return buf.getvalue()


def _stats_payload(render_ms, cloud_count, visible, decisions, lod_enabled, want_overlay) -> dict:
    """service._stats_payload (service.py:91-112)."""
    blocks = []
    for d in decisions:
        if not d.visible:
            continue
        entry = {"id": d.block, "level": d.level, "distance": d.distance}
        if want_overlay:
            entry["screen_box"] = list(d.screen_box) if d.screen_box else None
        blocks.append(entry)
    return {
        "render_ms": render_ms,
        "visible_gaussians": int(visible),
        "assembled_gaussians": int(cloud_count),
        "fps_estimate": 1000.0 / max(render_ms, 1e-6),
        "lod_enabled": lod_enabled,
        "blocks": blocks,
    }


class RenderService:
    """Request handling of the reference's render service, rendering on the
    B200.  ``scene`` is a LodScene (host clouds, e.g. bundle.load_lod) or a
    DeviceLodScene (bundle.load_lod_device / lodgen.build_lod_device); the
    upload happens on the first frame, so metadata calls need no device."""

    _VARIANTS = 8  # interval-override selection tables kept resident

    def __init__(self, scene, settings=None, max_dim: int = MAX_DIM_DEFAULT):
        from .render import RenderSettings
        self.scene = scene
        self.settings = settings or RenderSettings()
        self.max_dim = int(max_dim)
        self._lock = threading.Lock()
        self._frame_lock = threading.Lock()  # one frame at a time per service
        self._intervals = tuple((float(a), float(b)) for a, b in scene.distance_intervals)
        self._enabled = True
        self._last_stats: Optional[dict] = None
        self._dscene = None
        self._variants: "OrderedDict[tuple, object]" = OrderedDict()

    # -- metadata (service.py:126-161) ------------------------------------
    def snapshot(self):
        with self._lock:
            return self._intervals, self._enabled

    def _full_count(self) -> int:
        full = getattr(self.scene, "full", None)
        return int(full.count) if full is not None else 0

    def scene_info(self) -> dict:
        scene = self.scene
        intervals, enabled = self.snapshot()
        return {
            "n_blocks": scene.n_blocks,
            "n_levels": scene.n_levels,
            "level_sizes": [int(scene.level_size(level)) for level in range(scene.n_levels)],
            "full_size": self._full_count(),
            "sh_degrees": list(scene.sh_degrees),
            "intervals": _json_intervals(intervals),
            "lod_enabled": enabled,
            "n_mad": getattr(scene, "n_mad", None),
            "bounds_min": np.asarray(scene.bounds_min).tolist(),
            "bounds_max": np.asarray(scene.bounds_max).tolist(),
            "max_dim": self.max_dim,
        }

    def block_geometry(self) -> dict:
        scene = self.scene
        blocks = []
        for j in range(scene.n_blocks):
            if hasattr(scene, "levels"):
                size = int(scene.levels[scene.finest][j].count)
            else:
                size = int(scene.counts[scene.finest, j])
            blocks.append({"id": j, "min": np.asarray(scene.bounds_min)[j].tolist(),
                           "max": np.asarray(scene.bounds_max)[j].tolist(),
                           "occupied": bool(scene.occupied(j)), "size": size})
        return {"blocks": blocks}

    # -- LoD configuration (service.py:163-193) ---------------------------
    def update_lod(self, body: dict) -> dict:
        if not isinstance(body, dict):
            raise BadRequest("lod", "must be an object")
        intervals = None
        if body.get("intervals") is not None:
            intervals = self._parse_intervals(body["intervals"])
        with self._lock:
            if intervals is not None:
                self._intervals = intervals
            if "enabled" in body and body["enabled"] is not None:
                self._enabled = bool(body["enabled"])
            return {"ok": True, "intervals": _json_intervals(self._intervals),
                    "enabled": self._enabled}

    def _parse_intervals(self, raw):
        try:
            intervals = tuple((float(lo), float(hi if hi is not None else math.inf))
                              for lo, hi in raw)
        except (TypeError, ValueError):
            raise BadRequest("lod.intervals", "must be a list of [lo, hi] pairs") from None
        try:
            validate_intervals(intervals)
        except ConfigError as exc:
            raise BadRequest("lod.intervals", str(exc)) from None
        if len(intervals) != self.scene.n_levels:
            raise BadRequest("lod.intervals",
                             f"need exactly {self.scene.n_levels} intervals for this scene")
        return intervals

    # -- frames (service.py:195-230) --------------------------------------
    def _device_scene(self, intervals):
        from . import device
        if self._dscene is None:
            self._dscene = device.device_lod_scene(self.scene)
        ds = self._dscene
        if intervals == ds.distance_intervals:
            return ds
        hit = self._variants.get(intervals)
        if hit is None:
            # same resident level buffers, another selection table
            hit = device.DeviceLodScene.from_device_levels(
                ds.level_clouds, ds.counts, ds.bounds_min, ds.bounds_max, intervals,
                ds.sh_degrees, ds.device_index, full=ds.full)
            self._variants[intervals] = hit
            while len(self._variants) > self._VARIANTS:
                self._variants.popitem(last=False)
        else:
            self._variants.move_to_end(intervals)
        return hit

    def _full_source(self):
        from . import device
        full = getattr(self.scene, "full", None)
        if full is None and self._dscene is not None:
            full = self._dscene.full
        if full is None:
            raise BadRequest("lod", "this scene carries no full cloud (LoD cannot be disabled)")
        return full if isinstance(full, device.DeviceCloud) else device.device_cloud(full)

    def render(self, body: dict):
        """(png bytes, stats) as service.RenderService.render."""
        import torch
        from . import _lib, device
        from ._lib import CsFrameStats, CsSource, check
        from .lod import _decisions
        if not isinstance(body, dict):
            raise BadRequest("request", "must be a JSON object")
        cam = camera_from_json(body.get("camera"))
        if cam.width > self.max_dim or cam.height > self.max_dim:
            raise Oversized(self.max_dim)
        want_overlay = bool(body.get("want_overlay", False))

        intervals, enabled = self.snapshot()
        override = body.get("lod")
        if override is not None:
            if not isinstance(override, dict):
                raise BadRequest("lod", "must be an object")
            if override.get("intervals") is not None:
                intervals = self._parse_intervals(override["intervals"])
            if "enabled" in override and override["enabled"] is not None:
                enabled = bool(override["enabled"])

        with self._frame_lock:
            dev = device.default_device()
            src = CsSource()
            keep = None
            start = time.perf_counter()
            if enabled:
                ds = self._device_scene(intervals)
                decisions = _decisions(ds, cam, None)
                count = int(sum(ds.counts[d.level, d.block] for d in decisions
                                if d.visible and ds.counts[d.level, d.block] > 0))
                src.kind = _lib.CS_SRC_LOD_BLOCK
                src.force_level = -1
                src.lod = ds.handle
                keep = ds
            else:
                decisions = ()
                dc = self._full_source()
                count = dc.count
                src.kind = _lib.CS_SRC_CLOUD
                src.force_level = -1
                src.cloud = dc.desc()
                keep = dc
            out = torch.empty((cam.height, cam.width, 3), dtype=torch.float64, device=dev)
            stats = CsFrameStats()
            c = device.camera_struct(cam)
            s = device.settings_struct(self.settings)
            check(_lib.load().cs_render(device.context(dev.index), ctypes.byref(src), ctypes.byref(c),
                                        ctypes.byref(s), out.data_ptr(),
                                        _lib.CS_RENDER_SYNC | _lib.CS_RENDER_F64_OUT,
                                        ctypes.byref(stats), device.stream_handle(dev)), "cs_render")
            render_ms = (time.perf_counter() - start) * 1000.0
            # images.to_uint8 on the device: rint (half-even, as np.rint) of
            # 255 x in float64, clipped; only the 8-bit frame is read back
            u8 = torch.round(out * 255.0).clamp_(0, 255).to(torch.uint8).cpu().numpy()
            del keep
        result = _stats_payload(render_ms, count, stats.visible, decisions, enabled, want_overlay)
        png = encode_png(u8)
        with self._lock:
            self._last_stats = result
        return png, result

    def last_stats(self) -> Optional[dict]:
        with self._lock:
            return self._last_stats

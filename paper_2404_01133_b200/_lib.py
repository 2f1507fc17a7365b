"""ctypes binding of libcsgpu.so (include/cs_api.h).

The product path has no CPU fallback: importing the package without the built
library, or calling into it without an sm_100 device, raises.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libcsgpu.so"

CS_OK, CS_EINVAL, CS_ECUDA, CS_ENOMEM, CS_ERANGE = 0, -1, -2, -3, -4
CS_SRC_CLOUD, CS_SRC_LOD_BLOCK, CS_SRC_LOD_POINT = 0, 1, 2
CS_RENDER_SYNC, CS_RENDER_F64_OUT, CS_RENDER_NO_CLIP, CS_RENDER_KEEP_STATE = 1, 2, 4, 8
CS_RENDER_PROJECT_ONLY = 16
CS_RENDER_DEBUG = 32
CS_RENDER_DIAG = 64

c_double_p = ctypes.POINTER(ctypes.c_double)
vp = ctypes.c_void_p
i32 = ctypes.c_int32
i64 = ctypes.c_int64


class CsCamera(ctypes.Structure):
    _fields_ = [("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3),
                ("center", ctypes.c_double * 3), ("fx", ctypes.c_double),
                ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("width", i32), ("height", i32)]


class CsSettings(ctypes.Structure):
    _fields_ = [("background", ctypes.c_double * 3), ("alpha_floor", ctypes.c_double),
                ("transmittance_floor", ctypes.c_double), ("near_plane", ctypes.c_double),
                ("support_sigmas", ctypes.c_double), ("low_pass", ctypes.c_double),
                ("singular_det", ctypes.c_double), ("sh_degree", i32), ("tile_size", i32)]


class CsCloud(ctypes.Structure):
    _fields_ = [("pos_op", vp), ("scale", vp), ("quat", vp), ("sh", vp), ("count", i64),
                ("sh_coeffs", i32), ("sh_stride", i32), ("fp64", i32), ("reserved", i32)]


class CsFrameStats(ctypes.Structure):
    _fields_ = [("assembled", i64), ("visible", i64), ("skipped_singular", i64),
                ("pairs", i64), ("fragments", i64), ("n_segments", i32), ("status", i32),
                ("evals", i64), ("warp_hits", i64), ("warp_hits_empty", i64),
                ("blend_max_item_cycles", i64), ("blend_item_cycles", i64),
                ("blend_exact_hits", i64), ("blend_floor_resolved", i64), ("blend_replays", i64)]


class CsDecision(ctypes.Structure):
    _fields_ = [("distance", ctypes.c_double), ("box", ctypes.c_double * 4), ("level", i32),
                ("visible", ctypes.c_uint8), ("has_box", ctypes.c_uint8),
                ("pad", ctypes.c_uint8 * 2)]


class CsLodDesc(ctypes.Structure):
    _fields_ = [("n_levels", i32), ("n_blocks", i32), ("clouds", ctypes.POINTER(CsCloud)),
                ("bounds_min", c_double_p), ("bounds_max", c_double_p),
                ("intervals", c_double_p)]


class CsGrads(ctypes.Structure):
    _fields_ = [("positions", vp), ("scales", vp), ("rotations", vp), ("opacities", vp), ("sh", vp)]


class CsAdamHparams(ctypes.Structure):
    _fields_ = [("lr_position", ctypes.c_float), ("lr_scale", ctypes.c_float),
                ("lr_rotation", ctypes.c_float), ("lr_opacity", ctypes.c_float),
                ("lr_sh", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("eps", ctypes.c_float), ("step", i32), ("reserved", i32)]


class CsSource(ctypes.Structure):
    _fields_ = [("kind", i32), ("force_level", i32), ("cloud", CsCloud), ("lod", vp), ("exclude", vp),
                ("select_cam", ctypes.POINTER(CsCamera))]


_SIGS = {
    "cs_version": (ctypes.c_int, []),
    "cs_last_error": (ctypes.c_char_p, []),
    "cs_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(vp)]),
    "cs_destroy": (None, [vp]),
    "cs_lod_create": (ctypes.c_int, [vp, ctypes.POINTER(CsLodDesc), ctypes.POINTER(vp)]),
    "cs_lod_destroy": (None, [vp]),
    "cs_decide_visibility": (ctypes.c_int, [vp, vp, ctypes.POINTER(CsCamera), i32,
                                            ctypes.POINTER(CsDecision), vp]),
    "cs_block_visible": (ctypes.c_int, [vp, i32, vp, vp, ctypes.POINTER(CsCamera), vp, vp, vp]),
    "cs_select_level": (ctypes.c_int, [vp, i32, vp, i32, vp, vp, vp]),
    "cs_render": (ctypes.c_int, [vp, ctypes.POINTER(CsSource), ctypes.POINTER(CsCamera),
                                 ctypes.POINTER(CsSettings), vp, ctypes.c_uint32,
                                 ctypes.POINTER(CsFrameStats), vp]),
    "cs_frame_stats_get": (ctypes.c_int, [vp, ctypes.POINTER(CsFrameStats), vp]),
    "cs_check": (ctypes.c_int, [vp, vp]),
    "cs_render_train": (ctypes.c_int, [vp, ctypes.POINTER(CsSource), ctypes.POINTER(CsCamera),
                                       ctypes.POINTER(CsSettings), vp, ctypes.c_uint32, ctypes.POINTER(vp),
                                       vp]),
    "cs_render_backward": (ctypes.c_int, [vp, vp, vp, ctypes.POINTER(CsGrads), vp]),
    "cs_state_release": (None, [vp]),
    "cs_timing_begin": (ctypes.c_int, [vp, i32]),
    "cs_timing_end": (ctypes.c_int, [vp, vp, vp]),
    "cs_frame_graphs": (ctypes.c_int, [vp]),
    "cs_dump_projected": (ctypes.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "cs_dump_tiles": (ctypes.c_int, [vp, vp, vp, vp]),
    "cs_dump_segments": (ctypes.c_int, [vp, vp, vp, i32, vp, vp]),
    "cs_dump_assembled_list": (ctypes.c_int, [vp, vp, i64, vp, vp]),
    "cs_blend_tiles": (ctypes.c_int, [vp, vp, vp, i64, vp, vp, vp, vp, i64, vp, i32, i32, i32,
                                      i32, ctypes.c_double, ctypes.c_double, vp, vp, vp]),
    "cs_build_covariances": (ctypes.c_int, [vp, i64, vp, vp, vp, vp]),
    "cs_sh_to_colors": (ctypes.c_int, [vp, i64, vp, i32, vp, i32, vp, vp]),
    "cs_training_loss": (ctypes.c_int, [vp, vp, vp, i32, i32, ctypes.c_double, vp, vp, vp]),
    "cs_block_adam": (ctypes.c_int, [vp, i64, i32, vp, vp, vp, vp, vp, vp, ctypes.POINTER(CsGrads),
                                     ctypes.POINTER(CsAdamHparams), vp, vp, vp, vp]),
    "cs_block_activate": (ctypes.c_int, [vp, i64, vp, vp, vp, vp, vp]),
    "cs_block_of_points": (ctypes.c_int, [vp, i64, vp, i32, vp, vp, i32, i32, i32, vp, vp]),
    "cs_fuse_filter": (ctypes.c_int, [vp, i64, vp, i32, vp, vp, i32, i32, i32, i32, vp, vp, vp]),
    "cs_significance": (ctypes.c_int, [vp, ctypes.POINTER(CsCloud), vp, i32, ctypes.POINTER(CsSettings),
                                       vp, vp, vp]),
    "cs_priority": (ctypes.c_int, [vp, i64, vp, vp, vp]),
    "cs_lod_rows": (ctypes.c_int, [vp, i64, vp, vp, i32, vp, i32, vp, vp, vp]),
    "cs_mad_bounds": (ctypes.c_int, [vp, ctypes.POINTER(CsCloud), vp, i32, ctypes.c_double, vp, vp, vp]),
    "cs_gather_cloud": (ctypes.c_int, [vp, ctypes.POINTER(CsCloud), vp, i64, ctypes.POINTER(CsCloud), vp]),
    "cs_bounds_contain": (ctypes.c_int, [vp, i64, vp, i32, i32, vp, vp, vp, vp, vp, vp, vp]),
    "cs_ssim": (ctypes.c_int, [vp, vp, vp, i32, i32, vp, vp, vp]),
    "cs_measure_fp64_peak": (ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_double), vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def library_path() -> Path:
    return _LIB_PATH


def load():
    """Load libcsgpu.so; raises ImportError when it has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            if not _LIB_PATH.exists():
                raise ImportError(
                    f"{_LIB_PATH} is missing: build it with `python -m paper_2404_01133_b200._build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(str(_LIB_PATH))
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class CsError(RuntimeError):
    pass


def check(rc: int, what: str = ""):
    """Map C return codes to the reference's exception types (cs_api.h)."""
    if rc == CS_OK:
        return
    msg = load().cs_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc in (CS_EINVAL, CS_ERANGE):
        raise ValueError(msg)
    if rc == CS_ENOMEM:
        raise MemoryError(msg)
    raise CsError(msg)

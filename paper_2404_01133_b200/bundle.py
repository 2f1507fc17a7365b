"""Checkpoint and LoD-bundle loading straight into HBM.

Drop-ins for ``ply.load_ply`` (ply.py:73-137) and ``lod.load_lod``
(lod.py:432-455), plus ``load_lod_device``: the bundle's detail levels are
read once, concatenated per level on the host and uploaded as the
DeviceLodScene the renderer uses (one H2D copy per level, no per-frame host
work), so a render service or benchmark starts rendering from a bundle
without materialising a LodScene of host clouds.

PLY semantics follow the reference: binary little-endian float32 vertex
rows ``x y z nx ny nz f_dc_0..2 f_rest_* opacity scale_0..2 rot_0..3``, stored
pre-activation; loading applies sigmoid (opacity) and exp (scales, clamped to
MIN_SCALE with a warning) in float64 with numpy/scipy -- the same library
calls the reference makes, so the activated values are bit-identical -- and
renormalises quaternions that miss unit norm by more than QUAT_NORM_TOL.
The decode stays on the host on purpose: a device exp would differ in the
last ulp and break the bit-exact decision parity of PLY-loaded scenes
(SURVEY.md Appendix B.4).
"""

from __future__ import annotations

import json
import warnings
from pathlib import Path
from typing import Tuple

import numpy as np

from .core import QUAT_NORM_TOL, GaussianCloud

__all__ = ["DataError", "PlySchemaError", "load_ply", "load_lod", "load_lod_device"]

MIN_SCALE = 1e-8                 # ply.py:27
_FREST_WIDTHS = (0, 9, 24, 45)   # SH bands above band 0, channel-major


class DataError(ValueError):
    """errors.DataError: invalid input data."""


class PlySchemaError(DataError):
    """errors.PlySchemaError: a PLY file is not a Gaussian checkpoint."""


def _header(blob: bytes, path) -> Tuple[int, list, int]:
    marker = b"end_header\n"
    end = blob.find(marker)
    if not blob.startswith(b"ply\n") or end < 0:
        raise PlySchemaError(f"{path}: not a PLY file")
    fmt, count, props, in_vertex = None, None, [], False
    for line in blob[:end].decode("ascii", "replace").splitlines()[1:]:
        tok = line.split()
        if not tok or tok[0] in ("comment", "obj_info"):
            continue
        if tok[0] == "format":
            fmt = tok[1]
        elif tok[0] == "element":
            if in_vertex:
                raise PlySchemaError(f"{path}: unsupported extra element '{tok[1]}'")
            if tok[1] != "vertex":
                raise PlySchemaError(f"{path}: expected a vertex element, got '{tok[1]}'")
            in_vertex, count = True, int(tok[2])
        elif tok[0] == "property":
            if not in_vertex:
                raise PlySchemaError(f"{path}: property declared before the vertex element")
            if tok[1] not in ("float", "float32"):
                raise PlySchemaError(f"{path}: property '{tok[-1]}' is not float32")
            props.append(tok[2])
    if fmt != "binary_little_endian":
        raise PlySchemaError(f"{path}: format must be binary_little_endian, got {fmt}")
    if count is None:
        raise PlySchemaError(f"{path}: missing vertex element")
    return count, props, end + len(marker)


def _columns(path):
    """Raw float32 columns of a checkpoint PLY -> (count, n_rest, structured array)."""
    blob = Path(path).read_bytes()
    count, props, off = _header(blob, path)
    rest = sorted(int(p[7:]) for p in props if p.startswith("f_rest_"))
    n_rest = len(rest)
    if n_rest not in _FREST_WIDTHS or rest != list(range(n_rest)):
        raise PlySchemaError(f"{path}: f_rest properties must be a 0/9/24/45-wide prefix")
    need = (["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"]
            + [f"f_rest_{i}" for i in range(n_rest)]
            + ["opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"])
    for name in need:
        if name not in props:
            raise PlySchemaError(f"{path}: missing property '{name}'")
    dt = np.dtype([(p, "<f4") for p in props])
    body = blob[off:]
    if len(body) < count * dt.itemsize:
        raise DataError(f"{path}: truncated body, expected {count} vertices")
    return count, n_rest, props, np.frombuffer(body[:count * dt.itemsize], dtype=dt)


def load_ply(path) -> GaussianCloud:
    """ply.load_ply (ply.py:73-137): activated float64 GaussianCloud."""
    from scipy.special import expit
    count, n_rest, props, raw = _columns(path)
    if count:
        full = np.stack([raw[p].astype(np.float64) for p in props], axis=1)
        bad = ~np.isfinite(full).all(axis=1)
        if bad.any():
            raise DataError(f"{path}: non-finite value at row {int(np.argmax(bad))}")
    stack = lambda *names: np.stack([raw[n].astype(np.float64) for n in names], axis=1)
    positions = stack("x", "y", "z")
    opacities = expit(raw["opacity"].astype(np.float64)) if count else np.zeros(0)
    scales = np.exp(stack("scale_0", "scale_1", "scale_2"))
    small = scales <= MIN_SCALE
    if small.any():
        warnings.warn(f"{path}: clamped {int(small.sum())} degenerate scale components to {MIN_SCALE}")
        scales = np.where(small, MIN_SCALE, scales)
    rotations = stack("rot_0", "rot_1", "rot_2", "rot_3")
    norms = np.linalg.norm(rotations, axis=1)
    if count and norms.min() == 0.0:
        raise DataError(f"{path}: zero-norm quaternion at row {int(np.argmin(norms))}")
    off = np.abs(norms - 1.0) > QUAT_NORM_TOL
    if off.any():
        rotations = np.where(off[:, None], rotations / norms[:, None], rotations)
    C = 1 + n_rest // 3
    sh = np.zeros((count, 3, C))
    for ch in range(3):
        sh[:, ch, 0] = raw[f"f_dc_{ch}"]
        for i in range(C - 1):
            sh[:, ch, 1 + i] = raw[f"f_rest_{ch * (C - 1) + i}"]
    return GaussianCloud(positions, opacities, scales, rotations, sh)


def _index(root: Path) -> dict:
    try:
        return json.loads((root / "index.json").read_text())
    except FileNotFoundError:
        raise DataError(f"not a detail-level bundle: {root} has no index.json") from None


def _block_paths(root: Path, index: dict):
    out = []
    for level in range(int(index["n_levels"])):
        row = []
        for j in range(int(index["n_blocks"])):
            path = root / "levels" / str(level) / "blocks" / f"{j}.ply"
            if not path.exists():
                raise DataError(f"bundle is missing {path.relative_to(root)}")
            row.append(path)
        out.append(row)
    return out


def load_lod(in_dir):
    """lod.load_lod (lod.py:432-455): a LodScene of host clouds (bundle layout
    index.json, full.ply, levels/<L>/blocks/<j>.ply)."""
    from .lod import LodScene
    root = Path(in_dir)
    index = _index(root)
    levels = tuple(tuple(load_ply(p) for p in row) for row in _block_paths(root, index))
    return LodScene(
        levels=levels,
        bounds_min=np.array(index["bounds"]["min"], dtype=np.float64),
        bounds_max=np.array(index["bounds"]["max"], dtype=np.float64),
        distance_intervals=tuple((a, b) for a, b in index["intervals"]),
        sh_degrees=tuple(index["sh_degrees"]),
        n_mad=float(index["n_mad"]),
        full=load_ply(root / "full.ply"),
    )


def load_lod_device(in_dir, device=None, with_full: bool = False):
    """The bundle as a DeviceLodScene: each level's blocks are decoded (as
    load_ply) and uploaded once as one level cloud; ``full.ply`` is uploaded
    only when ``with_full`` (the no-LoD path of the render service)."""
    from . import device as dev
    root = Path(in_dir)
    index = _index(root)
    levels = [[load_ply(p) for p in row] for row in _block_paths(root, index)]
    full = dev.device_cloud(load_ply(root / "full.ply"), device) if with_full else None
    return dev.DeviceLodScene(levels, np.array(index["bounds"]["min"], dtype=np.float64),
                              np.array(index["bounds"]["max"], dtype=np.float64),
                              tuple((a, b) for a, b in index["intervals"]),
                              tuple(index["sh_degrees"]), device, full=full)

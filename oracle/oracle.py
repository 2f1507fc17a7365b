"""CPU parity oracle for the citysplat rendering hot path.

TEST INFRASTRUCTURE ONLY -- the checker, never the thing measured or shipped.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.  The product package
(paper_2404_01133_b200) never imports it and has no CPU fallback.

Thin numpy/ctypes wrapper over cs_oracle.c, which restates the reference
functions in their exact float64 operation order.  The
wrapper mirrors the reference call structure:

* project_cloud      -> render._project_cloud  (render.py:111-188)
* bin_tiles          -> render._bin_tiles      (render.py:217-249)
* blend_tiles        -> _kernels.blend_tiles   (_kernels.py:17-76)
* rasterize_stats    -> render.rasterize_stats (render.py:252-280)
* decide_visibility  -> lod.decide_visibility  (lod.py:330-348)
* assemble           -> lod.assemble_render_set(lod.py:360-401)
* block_of_points/fuse -> partition.py:155-169, 570-587

Pinning: tests/test_oracle_golden.py checks every function here against the
golden vectors in tests/golden/*.npz, which tests/golden/make_golden.py
produced by running the reference package itself (OPENBLAS_CORETYPE=Sandybridge).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libcsoracle.so"
_lib = None

LOW_PASS = 0.3          # render.py:33
SINGULAR_DET = 1e-12    # render.py:34


class _Cam(ctypes.Structure):
    _fields_ = [("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3),
                ("center", ctypes.c_double * 3), ("fx", ctypes.c_double),
                ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("width", ctypes.c_int64), ("height", ctypes.c_int64)]


class _Settings(ctypes.Structure):
    _fields_ = [("background", ctypes.c_double * 3), ("alpha_floor", ctypes.c_double),
                ("transmittance_floor", ctypes.c_double), ("near_plane", ctypes.c_double),
                ("support_sigmas", ctypes.c_double), ("low_pass", ctypes.c_double),
                ("singular_det", ctypes.c_double), ("sh_degree", ctypes.c_int64),
                ("tile_size", ctypes.c_int64)]


def build(force: bool = False) -> Path:
    """Compile cs_oracle.c (gcc, -ffp-contract=off, OpenMP)."""
    src = _HERE / "cs_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(
            ["gcc", "-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
             "-std=c11", "-shared", "-o", str(_LIB_PATH), str(src), "-lm"],
            check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(str(_LIB_PATH))
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        _lib.or_project.restype = i64
        _lib.or_project.argtypes = [i64, P, P, P, P, ctypes.c_int, P, ctypes.c_int, i64, P, P,
                                    P, P, P, P, P, P, P, P, P, ctypes.c_int]
        _lib.or_depth_argsort.argtypes = [i64, P, P]
        _lib.or_tile_rects.restype = i64
        _lib.or_tile_rects.argtypes = [i64, P, P, i64, i64, i64, P]
        _lib.or_bin_tiles.argtypes = [i64, P, i64, i64, i64, P, P]
        _lib.or_blend_tiles.argtypes = [P, P, i64, P, P, P, P, P, i64, i64, i64, i64,
                                        ctypes.c_double, ctypes.c_double, P, P, P, P,
                                        ctypes.c_int]
        _lib.or_blend_fragments.argtypes = [P, P, i64, P, P, P, i64, i64, i64, i64, ctypes.c_double,
                                            ctypes.c_double, P, P, P, ctypes.c_int]
        _lib.or_decide_visibility.restype = ctypes.c_int
        _lib.or_decide_visibility.argtypes = [i64, P, P, P, i64, P, P, i64, P, P, P, P, P]
        _lib.or_pointwise_keep.argtypes = [i64, P, ctypes.c_int, P, i64, P, i64, P]
        _lib.or_block_of_points.argtypes = [i64, P, ctypes.c_int, P, P, i64, i64, i64, P]
        _lib.or_significance_hits.argtypes = [i64, P, P, P, ctypes.c_int, i64, P, P, P, ctypes.c_int]
        _lib.or_rasterize.restype = ctypes.c_int
        _lib.or_rasterize.argtypes = [i64, P, P, P, P, ctypes.c_int, P, ctypes.c_int, i64, P, P,
                                      P, P, P, ctypes.c_int]
    return _lib


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _f64(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a.reshape(shape) if shape is not None else a


def _geom(a):
    """Keep float32 arrays as float32 (the oracle upcasts exactly), else float64."""
    a = np.asarray(a)
    if a.dtype == np.float32:
        return np.ascontiguousarray(a), 1
    return np.ascontiguousarray(a, dtype=np.float64), 0


def camera_struct(cam) -> _Cam:
    c = _Cam()
    R = _f64(cam.rotation_w2c).reshape(9)
    t = _f64(cam.translation_w2c).reshape(3)
    center = _f64(cam.camera_center).reshape(3)
    c.R[:] = list(R)
    c.t[:] = list(t)
    c.center[:] = list(center)
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    return c


def settings_struct(settings) -> _Settings:
    s = _Settings()
    bg = getattr(settings, "background", (0.0, 0.0, 0.0))
    s.background[:] = [float(v) for v in bg]
    s.alpha_floor = float(getattr(settings, "alpha_floor", 1.0 / 255.0))
    s.transmittance_floor = float(getattr(settings, "transmittance_floor", 1e-4))
    s.near_plane = float(getattr(settings, "near_plane", 0.2))
    s.support_sigmas = math.sqrt(2.0 * math.log(1.0 / s.alpha_floor))  # render.py:61-64
    s.low_pass = LOW_PASS
    s.singular_det = SINGULAR_DET
    s.sh_degree = int(getattr(settings, "sh_degree", 3))
    s.tile_size = int(getattr(settings, "tile_size", 16))
    return s


class DefaultSettings:
    background = (0.0, 0.0, 0.0)
    sh_degree = 3
    tile_size = 16
    alpha_floor = 1.0 / 255.0
    transmittance_floor = 1e-4
    near_plane = 0.2


def project_cloud(cloud, cam, settings=None, nthreads: int = 0) -> dict:
    """render._project_cloud (render.py:111-188): depth-sorted projection."""
    settings = settings or DefaultSettings()
    pos, gf = _geom(cloud.positions)
    opac, _ = _geom(cloud.opacities)
    scl, _ = _geom(cloud.scales)
    rot, _ = _geom(cloud.rotations)
    if gf:
        opac = opac.astype(np.float32)
        scl = scl.astype(np.float32)
        rot = rot.astype(np.float32)
    sh, sf = _geom(cloud.sh)
    k = pos.shape[0]
    C = sh.shape[2] if sh.ndim == 3 else 1
    n = max(k, 1)
    out = dict(means=np.zeros((n, 2)), conics=np.zeros((n, 3)), covs=np.zeros((n, 3)),
               depths=np.zeros(n), colors=np.zeros((n, 3)), opacities=np.zeros(n),
               radii=np.zeros((n, 2)), source=np.zeros(n, dtype=np.int64))
    skipped = ctypes.c_int64(0)
    cs = camera_struct(cam)
    ss = settings_struct(settings)
    m = lib().or_project(k, _ptr(pos), _ptr(opac), _ptr(scl), _ptr(rot), gf, _ptr(sh), sf, C,
                         ctypes.byref(cs), ctypes.byref(ss), _ptr(out["means"]),
                         _ptr(out["conics"]), _ptr(out["covs"]), _ptr(out["depths"]),
                         _ptr(out["colors"]), _ptr(out["opacities"]), _ptr(out["radii"]),
                         _ptr(out["source"]), ctypes.byref(skipped), nthreads)
    order = np.zeros(max(m, 1), dtype=np.int64)
    depths = np.ascontiguousarray(out["depths"][:m])
    lib().or_depth_argsort(m, _ptr(depths), _ptr(order))
    order = order[:m]
    res = {key: np.ascontiguousarray(v[:m][order]) for key, v in out.items()}
    res["skipped_singular"] = int(skipped.value)
    res["count"] = int(m)
    return res


def bin_tiles(proj: dict, cam, tile_size: int):
    """render._bin_tiles (render.py:217-249) -> (tile_ids, offsets, ntx, nty)."""
    ntx = (int(cam.width) + tile_size - 1) // tile_size
    nty = (int(cam.height) + tile_size - 1) // tile_size
    n_tiles = ntx * nty
    m = proj["count"]
    rects = np.zeros((max(m, 1), 4), dtype=np.int64)
    means = _f64(proj["means"]) if m else np.zeros((1, 2))
    radii = _f64(proj["radii"]) if m else np.zeros((1, 2))
    total = lib().or_tile_rects(m, _ptr(means), _ptr(radii), tile_size, int(cam.width),
                                int(cam.height), _ptr(rects))
    tile_ids = np.zeros(max(total, 1), dtype=np.int64)
    offsets = np.zeros(n_tiles + 1, dtype=np.int64)
    lib().or_bin_tiles(m, _ptr(rects), int(cam.width), tile_size, n_tiles, _ptr(tile_ids),
                       _ptr(offsets))
    return tile_ids[:total], offsets, ntx, nty


def blend_tiles(tile_ids, offsets, proj, cam, settings, nthreads: int = 0, want_state=False):
    """_kernels.blend_tiles (_kernels.py:17-76)."""
    ts = int(settings.tile_size)
    ntx = (int(cam.width) + ts - 1) // ts
    n_tiles = offsets.shape[0] - 1
    out = np.empty((int(cam.height), int(cam.width), 3))
    frags = np.zeros(n_tiles, dtype=np.int64)
    m = proj["count"]
    pad = lambda a, w: _f64(a) if m else np.zeros((1, w))
    means, conics, colors = pad(proj["means"], 2), pad(proj["conics"], 3), pad(proj["colors"], 3)
    opac = _f64(proj["opacities"]) if m else np.zeros(1)
    bg = _f64(settings.background)
    tid = np.ascontiguousarray(tile_ids, dtype=np.int64) if tile_ids.size else np.zeros(1, np.int64)
    final_t = np.empty((int(cam.height), int(cam.width))) if want_state else None
    last = np.empty((int(cam.height), int(cam.width)), dtype=np.int64) if want_state else None
    lib().or_blend_tiles(_ptr(tid), _ptr(offsets), n_tiles, _ptr(means), _ptr(conics),
                         _ptr(colors), _ptr(opac), _ptr(bg), ts, int(cam.width),
                         int(cam.height), ntx, float(settings.alpha_floor),
                         float(settings.transmittance_floor), _ptr(out), _ptr(frags),
                         _ptr(final_t), _ptr(last), nthreads)
    if want_state:
        return out, frags, final_t, last
    return out, frags


def blend_fragments(tile_ids, offsets, proj, cam, settings, nthreads: int = 0):
    """The accepted fragments of _kernels.blend_tiles (_kernels.py:46-72) per
    pixel, in blend order -> (pixel_offsets int64[H*W+1], splat int64[F]) with
    splat indices into the depth-sorted projection."""
    ts = int(settings.tile_size)
    W, H = int(cam.width), int(cam.height)
    ntx = (W + ts - 1) // ts
    n_tiles = offsets.shape[0] - 1
    m = proj["count"]
    pad = lambda a, w: _f64(a) if m else np.zeros((1, w))
    means, conics = pad(proj["means"], 2), pad(proj["conics"], 3)
    opac = _f64(proj["opacities"]) if m else np.zeros(1)
    tid = np.ascontiguousarray(tile_ids, dtype=np.int64) if tile_ids.size else np.zeros(1, np.int64)
    cnt = np.zeros(W * H, dtype=np.int64)
    args = (_ptr(tid), _ptr(offsets), n_tiles, _ptr(means), _ptr(conics), _ptr(opac), ts, W, H, ntx,
            float(settings.alpha_floor), float(settings.transmittance_floor))
    lib().or_blend_fragments(*args, _ptr(cnt), None, None, nthreads)
    off = np.zeros(W * H + 1, dtype=np.int64)
    np.cumsum(cnt, out=off[1:])
    splat = np.zeros(max(int(off[-1]), 1), dtype=np.int64)
    lib().or_blend_fragments(*args, _ptr(cnt), _ptr(off), _ptr(splat), nthreads)
    return off, splat[:int(off[-1])]


def rasterize_stats(cloud, cam, settings=None, nthreads: int = 0):
    """render.rasterize_stats (render.py:252-280) -> (clipped image, stats dict)."""
    settings = settings or DefaultSettings()
    proj = project_cloud(cloud, cam, settings, nthreads)
    tile_ids, offsets, _, _ = bin_tiles(proj, cam, int(settings.tile_size))
    out, frags = blend_tiles(tile_ids, offsets, proj, cam, settings, nthreads)
    stats = dict(visible_splats=proj["count"], blended_fragments=int(frags.sum()),
                 skipped_singular=proj["skipped_singular"], pairs=int(tile_ids.shape[0]))
    return np.clip(out, 0.0, 1.0), stats


def rasterize_frame_c(cloud, cam, settings=None, nthreads: int = 0):
    """All four stages inside C (used for the timed CPU baseline)."""
    settings = settings or DefaultSettings()
    pos, gf = _geom(cloud.positions)
    opac, scl, rot = (np.ascontiguousarray(np.asarray(a), dtype=pos.dtype)
                      for a in (cloud.opacities, cloud.scales, cloud.rotations))
    sh, sf = _geom(cloud.sh)
    out = np.empty((int(cam.height), int(cam.width), 3))
    counts = np.zeros(4, dtype=np.int64)
    stage = np.zeros(4)
    cs, ss = camera_struct(cam), settings_struct(settings)
    rc = lib().or_rasterize(pos.shape[0], _ptr(pos), _ptr(opac), _ptr(scl), _ptr(rot), gf,
                            _ptr(sh), sf, sh.shape[2], ctypes.byref(cs), ctypes.byref(ss),
                            _ptr(out), _ptr(counts), _ptr(stage), nthreads)
    if rc != 0:
        raise MemoryError("oracle rasterize failed")
    return np.clip(out, 0.0, 1.0), dict(visible_splats=int(counts[0]), pairs=int(counts[1]),
                                        blended_fragments=int(counts[2]),
                                        skipped_singular=int(counts[3]),
                                        stage_ms=dict(project=stage[0], sort=stage[1],
                                                      bin=stage[2], blend=stage[3]))


# ---------------------------------------------------------------------------
# LoD selection / assembly (lod.py:267-401)


def decide_visibility(scene, cam, force_level=None):
    """lod.decide_visibility -> list of (block, visible, level|None, distance, box|None)."""
    J = len(scene.levels[0])
    finest = len(scene.levels) - 1
    occupied = np.array([scene.levels[finest][j].count > 0 if hasattr(scene.levels[finest][j], "count")
                         else len(scene.levels[finest][j].positions) > 0 for j in range(J)],
                        dtype=np.uint8)
    bmin = _f64(scene.bounds_min).reshape(J, 3)
    bmax = _f64(scene.bounds_max).reshape(J, 3)
    ints = _f64(np.array(scene.distance_intervals, dtype=np.float64)).reshape(-1, 2)
    vis = np.zeros(J, dtype=np.uint8)
    lev = np.zeros(J, dtype=np.int64)
    dist = np.zeros(J)
    box = np.zeros((J, 4))
    has = np.zeros(J, dtype=np.uint8)
    cs = camera_struct(cam)
    rc = lib().or_decide_visibility(J, _ptr(bmin), _ptr(bmax), _ptr(occupied), ints.shape[0],
                                    _ptr(ints), ctypes.byref(cs),
                                    -1 if force_level is None else int(force_level),
                                    _ptr(vis), _ptr(lev), _ptr(dist), _ptr(box), _ptr(has))
    if rc != 0:
        raise ValueError("no interval covers a block distance")
    out = []
    for j in range(J):
        out.append((j, bool(vis[j]), None if lev[j] < 0 else int(lev[j]), float(dist[j]),
                    tuple(float(v) for v in box[j]) if has[j] else None))
    return out


class Arrays:
    """Plain columnar cloud (duck-types GaussianCloud for the oracle)."""

    def __init__(self, positions, opacities, scales, rotations, sh):
        self.positions, self.opacities, self.scales = positions, opacities, scales
        self.rotations, self.sh = rotations, sh

    @property
    def count(self):
        return int(np.asarray(self.positions).shape[0])


def concat(clouds):
    """GaussianCloud.concat (core.py:281-294): SH zero-padded to the widest."""
    clouds = list(clouds)
    if not clouds:
        return Arrays(np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3)), np.zeros((0, 4)),
                      np.zeros((0, 3, 16)))
    width = max(np.asarray(c.sh).shape[2] for c in clouds)

    def pad(sh):
        sh = np.asarray(sh)
        if sh.shape[2] == width:
            return sh
        o = np.zeros(sh.shape[:2] + (width,), dtype=sh.dtype)
        o[:, :, :sh.shape[2]] = sh
        return o

    return Arrays(np.concatenate([np.asarray(c.positions) for c in clouds]),
                  np.concatenate([np.asarray(c.opacities) for c in clouds]),
                  np.concatenate([np.asarray(c.scales) for c in clouds]),
                  np.concatenate([np.asarray(c.rotations) for c in clouds]),
                  np.concatenate([pad(c.sh) for c in clouds]))


def assemble(scene, cam, mode="block", force_level=None):
    """lod.assemble_render_set (lod.py:360-401) -> (Arrays, decisions)."""
    if mode == "block":
        dec = decide_visibility(scene, cam, force_level)
        pieces = [scene.levels[d[2]][d[0]] for d in dec
                  if d[1] and np.asarray(scene.levels[d[2]][d[0]].positions).shape[0]]
    elif mode == "pointwise":
        dec = ()
        center = _f64(cam.camera_center)
        los = _f64([lo for lo, _ in scene.distance_intervals])
        pieces = []
        for level in range(len(scene.levels)):
            want = level if force_level is None else int(force_level)
            for block in scene.levels[level]:
                pos, f32 = _geom(block.positions)
                k = pos.shape[0]
                if k == 0:
                    continue
                keep = np.zeros(k, dtype=np.uint8)
                lib().or_pointwise_keep(k, _ptr(pos), f32, _ptr(center), los.shape[0], _ptr(los),
                                        want, _ptr(keep))
                if level == want and keep.any():
                    idx = np.nonzero(keep)[0]
                    pieces.append(Arrays(np.asarray(block.positions)[idx],
                                         np.asarray(block.opacities)[idx],
                                         np.asarray(block.scales)[idx],
                                         np.asarray(block.rotations)[idx],
                                         np.asarray(block.sh)[idx]))
    else:
        raise ValueError(f"unknown selection mode: {mode}")
    if len(pieces) == 1:
        return pieces[0], dec
    return concat(pieces), dec


def block_of_points(positions, p_min, p_max, dims):
    """partition.block_of_points(contract(normalize_position(p)))."""
    dims = tuple(int(d) for d in dims)
    if len(dims) == 2:
        dims = dims + (1,)
    pos, f32 = _geom(positions)
    k = pos.shape[0]
    out = np.zeros(max(k, 1), dtype=np.int64)
    lib().or_block_of_points(k, _ptr(pos), f32, _ptr(_f64(p_min)), _ptr(_f64(p_max)),
                             dims[0], dims[1], dims[2], _ptr(out))
    return out[:k]


def fuse(block_clouds, p_min, p_max, dims):
    """partition.fuse (partition.py:570-587)."""
    pieces = []
    for cloud, j in sorted(block_clouds, key=lambda item: item[1]):
        pos = np.asarray(cloud.positions)
        if pos.shape[0] == 0:
            continue
        keep = block_of_points(pos, p_min, p_max, dims) == j
        if keep.any():
            idx = np.nonzero(keep)[0]
            pieces.append(Arrays(pos[idx], np.asarray(cloud.opacities)[idx],
                                 np.asarray(cloud.scales)[idx], np.asarray(cloud.rotations)[idx],
                                 np.asarray(cloud.sh)[idx]))
    return concat(pieces)


def significance_scores(cloud, cameras, settings=None, nthreads: int = 0):
    """lod.significance_scores (lod.py:54-101): C hit counts (or_significance_hits)
    times opacity times the percentile-clamped volume^0.1, the last two in numpy
    exactly as the reference writes them (lod.py:97-100).  Returns (scores, hits)."""
    settings = settings or DefaultSettings()
    k = int(np.asarray(cloud.positions).shape[0])
    if k == 0:
        return np.zeros(0), np.zeros(0, dtype=np.int64)
    geo = [_geom(a) for a in (cloud.positions, cloud.scales, cloud.rotations)]
    f32 = int(all(f for _, f in geo))
    pos, scl, rot = (g if f32 else _f64(g) for g, _ in geo)
    cams = list(cameras)
    arr = (_Cam * max(len(cams), 1))()
    for i, c in enumerate(cams):
        arr[i] = camera_struct(c)
    ss = settings_struct(settings)
    hits = np.zeros(k, dtype=np.int64)
    lib().or_significance_hits(k, _ptr(pos), _ptr(scl), _ptr(rot), f32, len(cams),
                               ctypes.cast(arr, ctypes.c_void_p), ctypes.byref(ss), _ptr(hits),
                               nthreads)
    scales = np.asarray(cloud.scales, dtype=np.float64)
    volume = np.prod(scales, axis=1)
    cap = np.percentile(volume, 90.0)
    clamped = np.minimum(volume, cap)
    scores = hits.astype(np.float64) * np.asarray(cloud.opacities, dtype=np.float64) * clamped ** 0.1
    return scores, hits


def priority(scores):
    """lod._priority (lod.py:114-116): descending score, ties -> lower index."""
    return np.argsort(-np.asarray(scores, dtype=np.float64), kind="stable")


def keep_count(rate: float, k: int) -> int:
    """lod._keep_count (lod.py:104-111)."""
    import math
    if not 0.0 < rate <= 1.0:
        raise ValueError("compression rate must be in (0, 1]")
    if k == 0:
        return 0
    return min(k, max(1, math.ceil(rate * k - 1e-9 * k)))


def level_rows(order, membership, n_blocks, rates_finest_first):
    """build_lod's kept rows (lod.py:222-234): [L][j] ascending indices, L coarsest first."""
    k = len(order)
    out = []
    membership = np.asarray(membership)
    for rate in reversed(tuple(rates_finest_first)):
        mask = np.zeros(k, dtype=bool)
        mask[np.asarray(order)[:keep_count(rate, k)]] = True
        out.append([np.nonzero(mask & (membership == j))[0] for j in range(n_blocks)])
    return out


def mad_bounds(positions, n_mad):
    """lod.mad_bounds (lod.py:130-147) restated with numpy."""
    import math
    p = np.asarray(positions, dtype=np.float64)
    if p.shape[0] == 0:
        raise ValueError("bounds of an empty block are undefined")
    lo = p.min(axis=0).copy()
    hi = p.max(axis=0).copy()
    med = np.median(p, axis=0)
    mad = np.median(np.abs(p - med), axis=0)
    for axis in range(3):
        if mad[axis] > 0.0 and math.isfinite(n_mad):
            lo[axis] = max(lo[axis], med[axis] - n_mad * mad[axis])
            hi[axis] = min(hi[axis], med[axis] + n_mad * mad[axis])
    return lo, hi


def build_lod(cloud, membership, n_blocks, cameras, distance_intervals,
              compression_rates=(0.5, 0.34, 0.25), lod_sh_degrees=(3, 2, 1), n_mad=4.0,
              settings=None, nthreads: int = 0):
    """lod.build_lod (lod.py:211-248) on the host: one global significance
    ranking over the training views, level L keeps the top
    _keep_count(rate_L, K) rows split by block (ascending index inside a
    block), SH truncated to the level degree; per-block MAD bounds of the full
    cloud's members.  Rates and degrees are finest-first, reversed here.
    Returns a namespace with levels[L][j] (Arrays, coarsest level first),
    bounds_min/bounds_max (J, 3), distance_intervals and sh_degrees."""
    from types import SimpleNamespace
    k = int(np.asarray(cloud.positions).shape[0])
    scores, _ = significance_scores(cloud, cameras, settings, nthreads)
    order = priority(scores)
    mem = np.asarray(membership).astype(np.int64)
    rates = tuple(reversed(tuple(compression_rates)))
    degrees = tuple(reversed(tuple(lod_sh_degrees)))
    sh = np.asarray(cloud.sh)
    cols = [np.asarray(cloud.positions), np.asarray(cloud.opacities), np.asarray(cloud.scales),
            np.asarray(cloud.rotations)]
    levels = []
    for rate, deg in zip(rates, degrees):
        mask = np.zeros(k, dtype=bool)
        mask[order[:keep_count(rate, k)]] = True
        idx = np.nonzero(mask)[0]
        # np.nonzero(mask & (membership == j)) for every j at once: stable split by block
        by_block = idx[np.argsort(mem[idx], kind="stable")]
        counts = np.bincount(mem[idx], minlength=n_blocks)
        width = min((deg + 1) ** 2, sh.shape[2])
        blocks = []
        start = 0
        for j in range(n_blocks):
            rows = by_block[start:start + counts[j]]
            start += counts[j]
            blocks.append(Arrays(*(c[rows] for c in cols), sh[rows][:, :, :width]))
        levels.append(tuple(blocks))
    bmin = np.zeros((n_blocks, 3))
    bmax = np.zeros((n_blocks, 3))
    members = np.argsort(mem, kind="stable")
    mcount = np.bincount(mem, minlength=n_blocks)
    start = 0
    for j in range(n_blocks):
        rows = members[start:start + mcount[j]]
        start += mcount[j]
        if rows.size:
            bmin[j], bmax[j] = mad_bounds(cols[0][rows], n_mad)
    return SimpleNamespace(levels=tuple(levels), bounds_min=bmin, bounds_max=bmax,
                           distance_intervals=tuple(tuple(map(float, iv)) for iv in distance_intervals),
                           sh_degrees=degrees)


# ---------------------------------------------------------------------------
# training-data assignment (partition.py:172-439, metrics.py:61-101)

def ssim(a, b):
    """metrics.ssim (metrics.py:70-96), restated with scipy.signal.convolve as the reference."""
    from scipy.signal import convolve
    g = np.exp(-((np.arange(11) - 5) ** 2) / (2.0 * 1.5 ** 2))
    w = np.outer(g, g)
    w = w / w.sum()
    pa, pb = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    vals = []
    for ch in range(3):
        x, y = pa[:, :, ch], pb[:, :, ch]
        mu_x = convolve(x, w, mode="valid")
        mu_y = convolve(y, w, mode="valid")
        e_xx = convolve(x * x, w, mode="valid")
        e_yy = convolve(y * y, w, mode="valid")
        e_xy = convolve(x * y, w, mode="valid")
        var_x = e_xx - mu_x ** 2
        var_y = e_yy - mu_y ** 2
        cov = e_xy - mu_x * mu_y
        num = (2 * mu_x * mu_y + 0.01 ** 2) * (2 * cov + 0.03 ** 2)
        den = (mu_x ** 2 + mu_y ** 2 + 0.01 ** 2) * (var_x + var_y + 0.03 ** 2)
        vals.append(np.mean(num / den))
    return float(np.mean(vals))


def bounds_contain(points, bounds_min, bounds_max):
    """partition.bounds_contain (partition.py:172-181)."""
    p = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    lo = np.asarray(bounds_min, dtype=np.float64)
    hi = np.asarray(bounds_max, dtype=np.float64)
    below = np.where(hi == 2.0, p <= hi, p < hi)
    return ((p >= lo) & below).all(axis=1)


def contract_normalized(p, p_min, p_max):
    """contract(normalize_position(p)) (partition.py:110-126)."""
    p = np.asarray(p, dtype=np.float64)
    ph = 2.0 * (p - np.asarray(p_min)) / (np.asarray(p_max) - np.asarray(p_min)) - 1.0
    m = np.abs(ph).max(axis=-1, keepdims=True)
    safe = np.maximum(m, 1.0)
    return np.where(m <= 1.0, ph, (2.0 - 1.0 / safe) * ph / safe)


def enlarge_bounds(j, bounds_min, bounds_max, contracted, min_count, factor=1.2):
    """partition.enlarge_bounds (partition.py:234-259)."""
    lo = np.asarray(bounds_min[j], dtype=np.float64).copy()
    hi = np.asarray(bounds_max[j], dtype=np.float64).copy()
    if contracted.shape[0] < min_count:
        return np.full(3, -2.0), np.full(3, 2.0)
    while bounds_contain(contracted, lo, hi).sum() < min_count:
        if (lo == -2.0).all() and (hi == 2.0).all():
            break
        center = 0.5 * (lo + hi)
        half = 0.5 * (hi - lo) * factor
        lo = np.maximum(center - half, -2.0)
        hi = np.minimum(center + half, 2.0)
    return lo, hi


def scaled_camera(cam, scale):
    """partition._scaled_camera (partition.py:300-310) as a plain namespace."""
    from types import SimpleNamespace
    if scale == 1.0:
        return cam
    return SimpleNamespace(width=max(1, int(round(cam.width * scale))),
                           height=max(1, int(round(cam.height * scale))),
                           fx=cam.fx * scale, fy=cam.fy * scale, cx=cam.cx * scale, cy=cam.cy * scale,
                           rotation_w2c=cam.rotation_w2c, translation_w2c=cam.translation_w2c,
                           camera_center=cam.camera_center)


def take(cloud, idx):
    return Arrays(np.asarray(cloud.positions)[idx], np.asarray(cloud.opacities)[idx],
                  np.asarray(cloud.scales)[idx], np.asarray(cloud.rotations)[idx],
                  np.asarray(cloud.sh)[idx])


def assign(views, grid, cloud, epsilon, settings=None, assignment_scale=0.25, enlarge_min_count=25_000):
    """partition.assign (partition.py:348-439) -> (entries, provenance, bmin_used, bmax_used, l_ssim)."""
    settings = settings or DefaultSettings()
    J = np.asarray(grid.bounds_min).shape[0]
    P = len(views)
    entries = np.zeros((P, J), dtype=bool)
    prov = np.full((P, J), "", dtype="<U5")
    bmin = np.asarray(grid.bounds_min, dtype=np.float64).copy()
    bmax = np.asarray(grid.bounds_max, dtype=np.float64).copy()
    scaled = [scaled_camera(v, assignment_scale) for v in views]
    fulls = [rasterize_stats(cloud, s, settings)[0] for s in scaled]
    centers = contract_normalized(np.stack([np.asarray(v.camera_center, dtype=np.float64) for v in views]),
                                  grid.map.p_min, grid.map.p_max)
    lmat = np.full((P, J), np.nan)

    def evaluate(j, rest, lo, hi, record):
        b2 = bounds_contain(centers, lo, hi)
        for i in range(P):
            b1 = False
            if rest is not None:
                l = 1.0 - ssim(fulls[i], rasterize_stats(rest, scaled[i], settings)[0])
                if record:
                    lmat[i, j] = l
                b1 = l > epsilon
            if b1 or b2[i]:
                entries[i, j] = True
                prov[i, j] = "B1+B2" if (b1 and b2[i]) else ("B1" if b1 else "B2")
            else:
                entries[i, j] = False
                prov[i, j] = ""

    mem = np.asarray(grid.membership)
    for j in range(J):
        rest = take(cloud, np.nonzero(mem != j)[0]) if np.asarray(grid.counts)[j] > 0 else None
        evaluate(j, rest, grid.bounds_min[j], grid.bounds_max[j], True)
    for j in range(J):
        if entries[:, j].any():
            continue
        lo, hi = enlarge_bounds(j, grid.bounds_min, grid.bounds_max, np.asarray(grid.contracted),
                                enlarge_min_count)
        bmin[j], bmax[j] = lo, hi
        m = bounds_contain(grid.contracted, lo, hi)
        rest = take(cloud, np.nonzero(~m)[0]) if m.any() else None
        evaluate(j, rest, lo, hi, False)
    return entries, prov, bmin, bmax, lmat

"""Generate the golden vectors in tests/golden/ by running the REFERENCE itself.

    OPENBLAS_CORETYPE=Sandybridge python tests/golden/make_golden.py

Imports citysplat from /root/reference/pkg/src (read-only; only present in
the build container, never on the GPU box) and records, for seeded inputs,
the reference's own outputs of the hot-path functions:

  render.npz   _project_cloud (render.py:111-188), _bin_tiles (render.py:217-249),
               rasterize_stats (render.py:252-280) on the closed-form cases of
               tests/test_render.py and on random cloud_in_view scenes
               (tests/conftest.py:37-54), tile sizes 8/16/32
  city.npz     a synthetic city (synthetic.py:96-203) cut into a 2x2 / 3-level
               LodScene (build_lod, lod.py:211-248): decide_visibility,
               assemble_render_set (block, forced, pointwise) and the render of
               the assembled cloud, for several cameras
  fuse.npz     partition.fuse (partition.py:570-587) of perturbed block clouds
  assign.npz   training-data assignment (partition.assign, partition.py:348-439)
               with the per-(pose, block) l_ssim of the contribution test
               (partition.py:318-334, metrics.py:70-101); a 5x5 grid with
               sparse / unassigned blocks (enlarged-bounds retry)
  bundle/      an on-disk LoD bundle written by lod.save_lod (lod.py:405-429)
  bundle.npz   the reference's lod.load_lod (lod.py:432-455) of it
  lodgen.npz   LoD generation: significance_scores
               (lod.py:54-101), the stable priority order (lod.py:114-116),
               build_lod's per-level / per-block kept rows (lod.py:211-248) and
               mad_bounds (lod.py:130-147), on a 3x3-block city with exact
               duplicate Gaussians (score ties)

OPENBLAS_CORETYPE=Sandybridge pins numpy's dgemm to the no-FMA kernel
(SURVEY.md Appendix B.1); the script refuses to run without it.
"""

import os
import sys

if os.environ.get("OPENBLAS_CORETYPE") != "Sandybridge":
    os.environ["OPENBLAS_CORETYPE"] = "Sandybridge"
    os.execv(sys.executable, [sys.executable] + sys.argv)

import math  # noqa: E402
from pathlib import Path  # noqa: E402

import numpy as np  # noqa: E402

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

from citysplat.config import RunConfig  # noqa: E402
from citysplat.core import CameraView, Gaussian, GaussianCloud, SH_C0  # noqa: E402
from citysplat.lod import (_keep_count, _priority, assemble_render_set, build_lod,  # noqa: E402
                           decide_visibility, load_lod, mad_bounds, save_lod, significance_scores)
from citysplat.metrics import l_ssim  # noqa: E402
from citysplat.partition import (ContractionMap, _scaled_camera, assign, fuse,  # noqa: E402
                                 grid_partition)
from citysplat.render import rasterize  # noqa: E402
from citysplat.render import RenderSettings, _bin_tiles, _project_cloud, rasterize_stats  # noqa: E402
from citysplat.synthetic import generate_synthetic_city, look_at  # noqa: E402
from conftest import cloud_in_view, identity_camera, random_camera  # noqa: E402

OUT = Path(__file__).resolve().parent


def q32(a):
    """Round to float32-representable float64."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def quantize(cloud: GaussianCloud) -> GaussianCloud:
    rot = q32(cloud.rotations)
    return GaussianCloud(positions=q32(cloud.positions), opacities=q32(cloud.opacities),
                         scales=q32(cloud.scales), rotations=rot, sh=q32(cloud.sh))


def cam_dict(cam):
    return dict(R=np.asarray(cam.rotation_w2c), t=np.asarray(cam.translation_w2c),
                center=np.asarray(cam.camera_center),
                intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy]),
                size=np.array([cam.width, cam.height], dtype=np.int64))


def settings_dict(s):
    return dict(bg=np.array(s.background), sh_degree=np.int64(s.sh_degree),
                tile_size=np.int64(s.tile_size), alpha_floor=np.float64(s.alpha_floor),
                t_floor=np.float64(s.transmittance_floor), near=np.float64(s.near_plane))


def cloud_dict(c):
    return dict(positions=c.positions, opacities=c.opacities, scales=c.scales,
                rotations=c.rotations, sh=c.sh)


def render_record(cloud, cam, settings):
    p = _project_cloud(cloud, cam, settings)
    tid, off, _, _ = _bin_tiles(p, cam, settings.tile_size)
    img, st = rasterize_stats(cloud, cam, settings)
    rec = dict(
        p_means=p.means, p_conics=p.conics, p_covs=p.covs, p_depths=p.depths,
        p_colors=p.colors, p_opacities=p.opacities, p_radii=p.radii, p_source=p.source,
        p_skipped=np.int64(p.skipped_singular), tile_ids=tid, offsets=off,
        image=img.pixels, visible=np.int64(st.visible_splats),
        fragments=np.int64(st.blended_fragments), skipped=np.int64(st.skipped_singular))
    return rec


def put(store, prefix, d):
    for k, v in d.items():
        store[f"{prefix}/{k}"] = np.asarray(v)


def on_axis(z, opacity=1.0, scale=0.3, color=None):
    sh = np.zeros((3, 16))
    if color is not None:
        sh[:, 0] = (np.asarray(color) - 0.5) / SH_C0
    return Gaussian(position=np.array([0.0, 0.0, z]), opacity=opacity, scale=np.full(3, scale),
                    rotation=np.array([1.0, 0.0, 0.0, 0.0]), sh=sh)


def make_render():
    store = {}
    cases = []
    # closed-form cases (tests/test_render.py:145-200)
    cases.append(("empty", GaussianCloud.empty(), identity_camera(40, 30),
                  RenderSettings(background=(0.1, 0.5, 0.9))))
    cases.append(("opaque_center", GaussianCloud.from_gaussians([on_axis(5.0, 1.0, color=(1.0, 0.5, 0.0))]),
                  identity_camera(65, 49, 60.0), RenderSettings(background=(0.2, 0.2, 0.2))))
    cases.append(("two_coincident", GaussianCloud.from_gaussians([
        on_axis(8.0, 0.5, color=(0.0, 1.0, 0.0)), on_axis(5.0, 0.5, color=(1.0, 0.0, 0.0))]),
        identity_camera(65, 49, 60.0), RenderSettings(background=(0.0, 0.0, 1.0))))
    cases.append(("t_floor_drop", GaussianCloud.from_gaussians([
        on_axis(float(z), 1.0, color=c) for z, c in
        ((1, (1.0, 0.0, 0.0)), (2, (0.0, 1.0, 0.0)), (3, (0.0, 0.0, 1.0)))]),
        identity_camera(1, 1, 10.0), RenderSettings()))
    cases.append(("faint_skip", GaussianCloud.from_gaussians([on_axis(5.0, 1.0 / 300.0, color=(1, 1, 1))]),
                  identity_camera(65, 49, 60.0), RenderSettings()))
    cases.append(("near_cull", GaussianCloud.from_gaussians([on_axis(-5.0), on_axis(0.1), on_axis(0.25)]),
                  identity_camera(), RenderSettings()))
    cases.append(("occluder", GaussianCloud.from_gaussians([
        on_axis(4.0, 1.0, 30.0, (0.1, 0.1, 0.1)), on_axis(8.0, 1.0, 30.0, (1.0, 1.0, 1.0))]),
        identity_camera(33, 25, 30.0), RenderSettings()))
    # random scenes like tests/test_render.py:207-221 (tile sizes 8/16/32)
    rng = np.random.default_rng(20260814)
    for i in range(24):
        cam = random_camera(rng)
        cloud = cloud_in_view(rng, cam, int(rng.integers(0, 41)))
        settings = RenderSettings(background=tuple(rng.uniform(0.0, 1.0, 3)),
                                  tile_size=int(rng.choice([8, 16, 32])),
                                  transmittance_floor=float(rng.choice([1e-4, 1e-12])),
                                  sh_degree=int(rng.integers(0, 4)))
        cases.append((f"random{i:02d}", cloud, cam, settings))
    # a denser scene with many tile pairs
    cam = identity_camera(width=96, height=72, f=70.0)
    cases.append(("dense", cloud_in_view(np.random.default_rng(99), cam, 300), cam, RenderSettings()))
    names = []
    for name, cloud, cam, settings in cases:
        put(store, name, cloud_dict(cloud))
        put(store, name, cam_dict(cam))
        put(store, name, settings_dict(settings))
        put(store, name, render_record(cloud, cam, settings))
        names.append(name)
    store["cases"] = np.array(names)
    np.savez_compressed(OUT / "render.npz", **store)
    print("render.npz", len(names), "cases")


def make_city():
    bundle = generate_synthetic_city(seed=7, extent=60.0, n_buildings=8, n_cameras=16,
                                     target_gaussians=4000, image_size=(64, 48))
    cloud = quantize(bundle.cloud)
    cmap = ContractionMap.central_third(cloud)
    grid = grid_partition(cloud, cmap, (2, 2))
    config = RunConfig(block_dims=(2, 2), distance_intervals=((0.0, 20.0), (20.0, 45.0), (45.0, math.inf)))
    cams = [r.view for r in bundle.train_cameras()]
    lod = build_lod(cloud, grid, cams, config)
    store = {}
    L, J = lod.n_levels, lod.n_blocks
    store["n_levels"] = np.int64(L)
    store["n_blocks"] = np.int64(J)
    store["bounds_min"] = lod.bounds_min
    store["bounds_max"] = lod.bounds_max
    store["intervals"] = np.array(lod.distance_intervals)
    store["sh_degrees"] = np.array(lod.sh_degrees)
    for l in range(L):
        for j in range(J):
            put(store, f"level{l}/block{j}", cloud_dict(lod.levels[l][j]))
    views = [r.view for r in bundle.cameras]
    center = cloud.positions.mean(axis=0)
    views.append(look_at(center + np.array([0.0, 0.0, 2000.0]), center, 64, 48, 54.0))  # far: coarse
    bc = 0.5 * (lod.bounds_min[0] + lod.bounds_max[0])
    views.append(CameraView(64, 48, 50.0, 50.0, 32.0, 24.0, np.eye(3), -bc))  # inside block 0
    names = []
    for i, cam in enumerate(views):
        name = f"cam{i:02d}"
        put(store, name, cam_dict(cam))
        dec = decide_visibility(lod, cam)
        store[f"{name}/dec_visible"] = np.array([d.visible for d in dec])
        store[f"{name}/dec_level"] = np.array([-1 if d.level is None else d.level for d in dec])
        store[f"{name}/dec_distance"] = np.array([d.distance for d in dec])
        store[f"{name}/dec_box"] = np.array([d.screen_box if d.screen_box else (np.nan,) * 4 for d in dec])
        for tag, kw in (("block", dict()), ("forced", dict(force_level=lod.finest)),
                        ("point", dict(mode="pointwise"))):
            a = assemble_render_set(lod, cam, **kw)
            store[f"{name}/{tag}_count"] = np.int64(a.cloud.count)
            if i % 4 == 0:
                store[f"{name}/{tag}_positions"] = a.cloud.positions.astype(np.float32)
            if tag == "block" or i % 4 == 0:
                put(store, f"{name}/{tag}", render_record(a.cloud, cam, RenderSettings()))
        names.append(name)
    store["cases"] = np.array(names)
    np.savez_compressed(OUT / "city.npz", **store)
    print("city.npz", len(names), "cameras")


def make_fuse():
    bundle = generate_synthetic_city(seed=3, extent=80.0, n_buildings=10, n_cameras=8,
                                     target_gaussians=3000, image_size=(32, 24))
    cloud = bundle.cloud
    cmap = ContractionMap.central_third(cloud)
    grid = grid_partition(cloud, cmap, (3, 3))
    rng = np.random.default_rng(5)
    blocks = []
    store = {"p_min": cmap.p_min, "p_max": cmap.p_max, "dims": np.array([3, 3])}
    for j in range(grid.n_blocks):
        m = grid.members(j)
        if j == 4:
            continue  # a missing block
        sub = cloud.take(m)
        moved = GaussianCloud(positions=sub.positions + rng.normal(0, 1.5, sub.positions.shape),
                              opacities=sub.opacities, scales=sub.scales,
                              rotations=sub.rotations, sh=sub.sh)
        blocks.append((moved, j))
        put(store, f"block{j}", cloud_dict(moved))
    fused = fuse(list(reversed(blocks)), grid)
    put(store, "fused", cloud_dict(fused))
    store["block_ids"] = np.array([j for _, j in blocks])
    np.savez_compressed(OUT / "fuse.npz", **store)
    print("fuse.npz", fused.count, "fused of", sum(b.count for b, _ in blocks))


def make_assign():
    bundle = generate_synthetic_city(seed=21, extent=80.0, n_buildings=12, n_cameras=12,
                                     target_gaussians=6000, image_size=(160, 120))
    cloud = quantize(bundle.cloud)
    # foreground box over the x-y centre third; a 5x5 grid leaves corner
    # blocks empty or sparse so the enlarged-bounds retry runs
    cmap = ContractionMap.central_third(cloud)
    grid = grid_partition(cloud, cmap, (5, 5))
    poses = bundle.train_cameras()
    scale = 0.5
    settings = RenderSettings()
    views = [p.view for p in poses]
    scaled = [_scaled_camera(v, scale) for v in views]
    P, J = len(poses), grid.n_blocks
    l = np.full((P, J), np.nan)
    fulls = [rasterize(cloud, s, settings) for s in scaled]
    for j in range(J):
        if grid.counts[j] == 0:
            continue
        rest = cloud.take(np.nonzero(grid.membership != j)[0])
        for i in range(P):
            l[i, j] = l_ssim(fulls[i], rasterize(rest, scaled[i], settings))
    # epsilon in the widest gap of the middle half of the finite values: no
    # decision sits on a knife edge
    v = np.sort(l[np.isfinite(l)])
    lo_i, hi_i = len(v) // 4, 3 * len(v) // 4
    gaps = np.diff(v[lo_i:hi_i + 1])
    g = int(np.argmax(gaps))
    eps = float(0.5 * (v[lo_i + g] + v[lo_i + g + 1]))
    min_count = 900
    res = assign(poses, grid, cloud, eps, settings=settings, assignment_scale=scale,
                 enlarge_min_count=min_count)
    store = dict(positions=cloud.positions.astype(np.float32), opacities=cloud.opacities.astype(np.float32),
                 scales=cloud.scales.astype(np.float32), rotations=cloud.rotations.astype(np.float32),
                 sh=cloud.sh.astype(np.float32), membership=grid.membership, counts=grid.counts,
                 contracted=grid.contracted, bounds_min=grid.bounds_min, bounds_max=grid.bounds_max,
                 p_min=cmap.p_min, p_max=cmap.p_max, dims=np.array(grid.dims),
                 epsilon=np.float64(eps), scale=np.float64(scale), min_count=np.int64(min_count),
                 l_ssim=l, entries=res.entries, provenance=res.provenance.astype("U5"),
                 bounds_min_used=res.bounds_min_used, bounds_max_used=res.bounds_max_used,
                 image_ids=np.array(res.image_ids), n_poses=np.int64(P))
    assert np.array_equal(store["positions"].astype(np.float64), cloud.positions)
    assert np.array_equal(store["sh"].astype(np.float64), cloud.sh)
    for i, vw in enumerate(views):
        put(store, f"pose{i:02d}", cam_dict(vw))
    np.savez_compressed(OUT / "assign.npz", **store)
    enlarged = int((~np.all(res.bounds_min_used == grid.bounds_min, axis=1)).sum())
    print("assign.npz", P, "poses", J, "blocks; counts", grid.counts.tolist(), "eps", eps,
          "gap", float(gaps[g]), "B1", int((res.provenance == "B1").sum()),
          "B2", int((res.provenance == "B2").sum()), "B1+B2", int((res.provenance == "B1+B2").sum()),
          "enlarged", enlarged)


def make_bundle():
    import shutil
    bundle = generate_synthetic_city(seed=5, extent=50.0, n_buildings=6, n_cameras=8,
                                     target_gaussians=1500, image_size=(64, 48))
    cloud = bundle.cloud
    cmap = ContractionMap.central_third(cloud)
    grid = grid_partition(cloud, cmap, (2, 2))
    config = RunConfig(block_dims=(2, 2), distance_intervals=((0.0, 15.0), (15.0, 35.0), (35.0, math.inf)))
    lod = build_lod(cloud, grid, [r.view for r in bundle.train_cameras()], config)
    out = OUT / "bundle"
    shutil.rmtree(out, ignore_errors=True)
    save_lod(lod, out)
    back = load_lod(out)
    store = {"n_levels": np.int64(back.n_levels), "n_blocks": np.int64(back.n_blocks),
             "bounds_min": back.bounds_min, "bounds_max": back.bounds_max,
             "intervals": np.array(back.distance_intervals), "sh_degrees": np.array(back.sh_degrees),
             "n_mad": np.float64(back.n_mad)}
    put(store, "full", cloud_dict(back.full))
    for l in range(back.n_levels):
        for j in range(back.n_blocks):
            put(store, f"level{l}/block{j}", cloud_dict(back.levels[l][j]))
    cam = bundle.cameras[3].view
    put(store, "cam", cam_dict(cam))
    a = assemble_render_set(back, cam)
    put(store, "render", render_record(a.cloud, cam, RenderSettings()))
    np.savez_compressed(OUT / "bundle.npz", **store)
    print("bundle/", sum(f.stat().st_size for f in out.rglob("*") if f.is_file()) // 1024, "KiB")


def make_lodgen():
    bundle = generate_synthetic_city(seed=11, extent=120.0, n_buildings=30, n_cameras=24,
                                     target_gaussians=20_000, image_size=(320, 240))
    c = quantize(bundle.cloud)
    # append exact duplicates of 500 Gaussians: identical scores, ties broken by index
    dup = np.arange(0, 20_000, 40)
    cloud = GaussianCloud(positions=np.concatenate([c.positions, c.positions[dup]]),
                          opacities=np.concatenate([c.opacities, c.opacities[dup]]),
                          scales=np.concatenate([c.scales, c.scales[dup]]),
                          rotations=np.concatenate([c.rotations, c.rotations[dup]]),
                          sh=np.concatenate([c.sh, c.sh[dup]]))
    cmap = ContractionMap.central_third(cloud)
    grid = grid_partition(cloud, cmap, (3, 3))
    config = RunConfig(block_dims=(3, 3), n_mad=2.5)
    cams = [r.view for r in bundle.train_cameras()]
    scores = significance_scores(cloud, cams)
    order = _priority(scores)
    lod = build_lod(cloud, grid, cams, config)
    store = dict(positions=cloud.positions.astype(np.float32), opacities=cloud.opacities.astype(np.float32),
                 scales=cloud.scales.astype(np.float32), rotations=cloud.rotations.astype(np.float32),
                 membership=grid.membership.astype(np.int32), n_blocks=np.int64(grid.n_blocks),
                 rates=np.array(config.compression_rates), sh_degrees=np.array(config.lod_sh_degrees),
                 n_mad=np.float64(config.n_mad), scores=scores, order=order.astype(np.int32),
                 bounds_min=lod.bounds_min, bounds_max=lod.bounds_max,
                 n_cams=np.int64(len(cams)))
    assert np.array_equal(store["positions"].astype(np.float64), cloud.positions)
    for i, cam in enumerate(cams):
        put(store, f"cam{i:02d}", cam_dict(cam))
    rates = tuple(reversed(config.compression_rates))
    for L, rate in enumerate(rates):
        keep = _keep_count(rate, cloud.count)
        mask = np.zeros(cloud.count, dtype=bool)
        mask[order[:keep]] = True
        for j in range(grid.n_blocks):
            idx = np.nonzero(mask & (grid.membership == j))[0]
            assert np.array_equal(lod.levels[L][j].positions, cloud.positions[idx])
            store[f"level{L}/block{j}"] = idx.astype(np.int32)
    # mad_bounds with clipping disabled (n_mad = inf) for one block
    lo, hi = mad_bounds(cloud.take(grid.members(4)), math.inf)
    store["block4_inf_lo"], store["block4_inf_hi"] = lo, hi
    np.savez_compressed(OUT / "lodgen.npz", **store)
    print("lodgen.npz", cloud.count, "Gaussians,", len(cams), "views, ties:", len(dup),
          "zero scores:", int((scores == 0).sum()))


def make_service():
    """RenderService.render (service.py:195-230) of the reference on the
    bundle scene: request bodies, decoded PNG pixels and the stats payload
    (render_ms / fps_estimate dropped: wall-clock)."""
    import io
    import json
    from PIL import Image as PilImage
    from citysplat.service import RenderService
    from citysplat.lod import load_lod as ref_load_lod
    bundle = generate_synthetic_city(seed=5, extent=50.0, n_buildings=6, n_cameras=8,
                                     target_gaussians=1500, image_size=(64, 48))
    scene = ref_load_lod(OUT / "bundle")
    svc = RenderService(scene, max_dim=256)

    def cam_json(cam):
        return {"width": cam.width, "height": cam.height, "fx": cam.fx, "fy": cam.fy,
                "cx": cam.cx, "cy": cam.cy, "rotation": cam.rotation_w2c.tolist(),
                "translation": cam.translation_w2c.tolist()}

    reqs = []
    for i in range(8):
        reqs.append({"camera": cam_json(bundle.cameras[i].view), "want_overlay": i % 2 == 1})
    reqs.append({"camera": cam_json(bundle.cameras[3].view), "lod": {"enabled": False}})
    reqs.append({"camera": cam_json(bundle.cameras[5].view),
                 "lod": {"intervals": [[0, 5], [5, 10], [10, None]]}, "want_overlay": True})
    store = {"n": np.int64(len(reqs))}
    for k, body in enumerate(reqs):
        png, stats = svc.render(body)
        px = np.asarray(PilImage.open(io.BytesIO(png)).convert("RGB"))
        stats = {key: v for key, v in stats.items() if key not in ("render_ms", "fps_estimate")}
        store[f"req{k}/body"] = np.array(json.dumps(body))
        store[f"req{k}/pixels"] = px
        store[f"req{k}/png"] = np.frombuffer(png, dtype=np.uint8)
        store[f"req{k}/stats"] = np.array(json.dumps(stats))
    store["scene_info"] = np.array(json.dumps(svc.scene_info()))
    store["blocks"] = np.array(json.dumps(svc.block_geometry()))
    np.savez_compressed(OUT / "service.npz", **store)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()["make_" + name]()
        sys.exit(0)
    make_render()
    make_city()
    make_fuse()
    make_lodgen()
    make_assign()
    make_bundle()
    make_service()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size // 1024, "KiB")

"""BASELINE.json configs as parity cases (needs a B200), every one against the
C oracle on identical inputs:

* C1 -- synthetic 100k-Gaussian scene, one block, 3 LoD levels built on the
  device (cs_significance / cs_lod_rows / cs_mad_bounds), 256x256 views:
  LoD decisions, assembled counts, visible / fragment counts and images for
  every camera of the set;
* C2 -- synthetic 1.1M-Gaussian scene, 1080p, no LoD: projection fields,
  the full tile list and the image, at orbit, top-down and low-altitude views.

Bar (north star): visible set and sorted tile lists bit-exact, fragment counts
equal, images within max-abs 1e-4.
"""

import math
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu
IMG_TOL = 1e-4


def _host_scene(scene):
    levels = []
    for L in range(scene.n_levels):
        lc = scene.level_clouds[L]
        pos_op = lc.pos_op.float().cpu().numpy()
        scl = lc.scale.float().cpu().numpy()
        quat = lc.quat.float().cpu().numpy()
        C = lc.sh_coeffs
        sh = lc.sh[:, :3 * C].cpu().numpy().reshape(-1, 3, C)
        blocks = []
        for j in range(scene.n_blocks):
            o, n = int(scene.block_offsets[L][j]), int(scene.counts[L, j])
            blocks.append(SimpleNamespace(positions=pos_op[o:o + n, :3], opacities=pos_op[o:o + n, 3],
                                          scales=scl[o:o + n, :3], rotations=quat[o:o + n], sh=sh[o:o + n],
                                          count=n))
        levels.append(tuple(blocks))
    return SimpleNamespace(levels=tuple(levels), bounds_min=scene.bounds_min, bounds_max=scene.bounds_max,
                           distance_intervals=scene.distance_intervals)


@pytest.fixture(scope="module")
def c1():
    from paper_2404_01133_b200 import lodgen
    from paper_2404_01133_b200.synth import city_cameras, generate_city_torch
    dev = torch.device("cuda", 0)
    pos, op, sc, q, sh = generate_city_torch(0, 100.0, 40, 100_000, device=dev)
    pmin, pmax = lodgen.central_third(pos)
    mem = lodgen.block_membership(pos, pmin, pmax, (1, 1))
    cams = city_cameras(16, 100.0, 256, 256, seed=0)
    train = [c for i, c in enumerate(cams) if i % 8 != 0]
    scene = lodgen.build_lod_device(pos, op, sc, q, sh, mem, 1, train,
                                    distance_intervals=((0.0, 40.0), (40.0, 80.0), (80.0, math.inf)))
    return scene, _host_scene(scene), cams


def test_c1_lod_render_all_cameras(c1):
    import paper_2404_01133_b200 as cs
    scene, hs, cams = c1
    st = cs.RenderSettings()
    for i, cam in enumerate(cams):
        dec = cs.decide_visibility(scene, cam)
        odec = O.decide_visibility(hs, cam)
        assert [(d.visible, d.level) for d in dec] == [(o[1], o[2]) for o in odec]
        # the camera's own level, and every level forced in turn (lod.py:330-348)
        for force in (None, i % 3):
            a = cs.assemble_render_set(scene, cam, force_level=force)
            ocloud, _ = O.assemble(hs, cam, force_level=force)
            assert a.cloud.count == ocloud.count
            img, stats = cs.rasterize_stats(a.cloud, cam, st)
            rimg, rstats = O.rasterize_stats(ocloud, cam, st)
            assert stats.visible_splats == rstats["visible_splats"]
            assert stats.blended_fragments == rstats["blended_fragments"]
            assert np.abs(img.pixels - rimg).max() <= IMG_TOL


@pytest.fixture(scope="module")
def c2():
    from paper_2404_01133_b200.synth import city_cameras, generate_city, look_at
    cloud = generate_city(seed=2, extent=100.0, n_buildings=40, n_gaussians=1_100_000)
    cams = city_cameras(16, 100.0, 1920, 1080, seed=2)
    center = np.asarray(cloud.positions).mean(axis=0)
    low = look_at(center + np.array([0.15 * 100.0, 0.0, 0.15 * 100.0]), center, 1920, 1080, 1600.0)
    return cloud, [cams[1], cams[12], low]


@pytest.mark.parametrize("ci", [0, 1, 2])
def test_c2_1080p_full_cloud(c2, ci):
    import paper_2404_01133_b200 as cs
    from paper_2404_01133_b200.render import bin_tiles_last, project_cloud
    cloud, cams = c2
    cam = cams[ci]
    st = cs.RenderSettings()
    p = project_cloud(cloud, cam, st)
    rp = O.project_cloud(cloud, cam, st)
    assert p["count"] == rp["count"] > 1000
    for f in ("means", "conics", "depths", "radii", "source"):
        assert np.array_equal(p[f], rp[f]), f
    img, stats = cs.rasterize_stats(cloud, cam, st)
    tid, off = bin_tiles_last(cam, 16)
    rtid, roff, _, _ = O.bin_tiles(rp, cam, 16)
    assert np.array_equal(off, roff) and np.array_equal(tid, rtid)
    rimg, rstats = O.rasterize_stats(cloud, cam, st)
    assert stats.blended_fragments == rstats["blended_fragments"]
    assert np.abs(img.pixels - rimg).max() <= IMG_TOL

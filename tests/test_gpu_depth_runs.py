"""Exact depth order through the 32-bit depth sort + run fix-up (K4/K4b), needs a B200.

Splats whose float64 depths share a 32-bit sort key (the top bits of
bits(z) - bits(near), ~2^28 steps per octave) form runs after the 32-bit radix
sort; K4b re-sorts each run by (float64 depth, assembled index).
These scenes force every fix-up path -- short runs (<= 8, one thread), runs
handled by one CTA in shared memory (<= 2048) and longer runs merged through
global scratch -- with shuffled sub-ulp depth offsets and exact ties, and
compare the depth order (source indices), the tile lists and the image with
the C oracle (np.argsort(depths, kind="stable"), render.py:176-177).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _scene(seed, groups, width=320, height=240):
    from paper_2404_01133_b200.core import CameraView, GaussianCloud
    rng = np.random.default_rng(seed)
    f = 0.9 * width
    cam = CameraView(width, height, f, f, width / 2.0, height / 2.0, np.eye(3), np.zeros(3))
    zs = []
    for base, n, spread, ties in groups:
        d = rng.uniform(0.0, spread, n)
        if ties:  # a share of exact duplicates
            d[: n // 3] = d[n // 3: 2 * (n // 3)]
        zs.append(base + d)
    z = np.concatenate(zs)
    perm = rng.permutation(z.size)          # depth order unrelated to index order
    z = z[perm]
    k = z.size
    u = rng.uniform(0.05 * width, 0.95 * width, k)
    v = rng.uniform(0.05 * height, 0.95 * height, k)
    pos = np.stack([(u - cam.cx) / f * z, (v - cam.cy) / f * z, z], axis=1)
    q = rng.normal(size=(k, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    cloud = GaussianCloud(pos, rng.uniform(0.1, 0.6, k), rng.uniform(0.002, 0.02, (k, 3)) * z[:, None] / 10,
                          q, rng.normal(0.0, 0.2, (k, 3, 4)))
    return cloud, cam


@pytest.mark.parametrize("seed", [0, 1])
def test_depth_runs_exact(seed):
    import paper_2404_01133_b200 as cs
    from oracle import oracle as O
    from paper_2404_01133_b200.render import bin_tiles_last, project_cloud
    groups = [
        (5.0, 600, 1e-2, False),     # spread out: mostly singleton runs, some short runs
        (7.0, 24, 1e-7, True),       # ~7 keys at 7: short runs with ties
        (10.0, 1500, 4e-7, True),    # ~13 keys at 10: runs of ~100 (CTA bitonic)
        (30.0, 5000, 0.0, False),    # 5000 exactly equal depths (merge path, order by index)
        (40.0, 4500, 1.5e-6, True),  # ~12 keys at 40: runs of ~400, shuffled, with ties
    ]
    cloud, cam = _scene(seed, groups)
    st = cs.RenderSettings()
    p = project_cloud(cloud, cam, st)
    r = O.project_cloud(cloud, cam, st)
    assert p["count"] == r["count"] > 10000
    assert np.array_equal(p["source"], r["source"][: r["count"]])
    assert np.array_equal(p["depths"], r["depths"][: r["count"]])
    img, stats = cs.rasterize_stats(cloud, cam, st)
    tid, off = bin_tiles_last(cam, st.tile_size)
    rtid, roff, _, _ = O.bin_tiles(r, cam, st.tile_size)
    assert np.array_equal(tid, rtid) and np.array_equal(off, roff)
    rimg, rstats = O.rasterize_stats(cloud, cam, st)
    assert stats.blended_fragments == rstats["blended_fragments"]
    assert np.abs(img.pixels - rimg).max() <= 1e-4


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_needle_splats_box_masks(seed):
    """Thin, long, randomly rotated splats stress K8's exact ellipse-vs-box
    mask: a box the alpha-floor ellipse reaches must never be skipped, so the
    accepted-fragment count and image must still equal the oracle's."""
    import paper_2404_01133_b200 as cs
    from oracle import oracle as O
    from paper_2404_01133_b200.core import CameraView, GaussianCloud
    rng = np.random.default_rng(100 + seed)
    W, H = 256, 192
    f = 0.9 * W
    cam = CameraView(W, H, f, f, W / 2.0 + 0.37, H / 2.0 - 0.21, np.eye(3), np.zeros(3))
    k = 3000
    z = rng.uniform(2.0, 30.0, k)
    u = rng.uniform(-0.1 * W, 1.1 * W, k)
    v = rng.uniform(-0.1 * H, 1.1 * H, k)
    pos = np.stack([(u - cam.cx) / f * z, (v - cam.cy) / f * z, z], axis=1)
    q = rng.normal(size=(k, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sc = np.stack([rng.uniform(0.001, 0.01, k), rng.uniform(0.2, 3.0, k), rng.uniform(0.001, 0.01, k)], axis=1)
    cloud = GaussianCloud(pos, rng.uniform(0.05, 1.0, k), sc, q, rng.normal(0.0, 0.3, (k, 3, 4)))
    st = cs.RenderSettings()
    img, stats = cs.rasterize_stats(cloud, cam, st)
    rimg, rstats = O.rasterize_stats(cloud, cam, st)
    assert stats.visible_splats == rstats["visible_splats"]
    assert stats.blended_fragments == rstats["blended_fragments"]
    assert np.abs(img.pixels - rimg).max() <= 1e-4

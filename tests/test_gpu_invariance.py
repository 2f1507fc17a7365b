"""Bitwise determinism of the forward (needs a B200).

* Fused-vs-original: a 50k-Gaussian city partitioned into 2x2 blocks
  (central-third contraction, grid_partition membership) and fused back with
  the device fusion (fusion.fuse_device, partition.fuse partition.py:570-587)
  renders BYTE-identically to the original cloud from the 16 seam-straddling
  views of the reference's acceptance gate (test_acceptance.py:240-268), and
  so does its device-tier (float32) image.
* Permutation invariance: a random row permutation of a cloud without exact
  depth ties renders byte-identically (the reference asserts 1e-6,
  test_render.py:234-243; the north star asks for a bitwise
  permutation-invariant forward: no atomics on colour, the same per-element
  math wherever a row sits), with the same fragment count and the same tile
  list up to the permutation.
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def city():
    from paper_2404_01133_b200.synth import generate_city
    return generate_city(seed=0, extent=100.0, n_buildings=40, n_gaussians=50_000)


def _central_third(p):
    lo, hi = p.min(axis=0), p.max(axis=0)
    c = 0.5 * (lo + hi)
    six = np.maximum((hi - lo) / 6.0, 1e-6)
    return np.array([c[0] - six[0], c[1] - six[1], lo[2]]), np.array([c[0] + six[0], c[1] + six[1], hi[2]])


def _seam_views(pmin, pmax):
    from paper_2404_01133_b200.synth import look_at
    center = 0.5 * (pmin + pmax)
    span = float(np.max(pmax[:2] - pmin[:2]))
    cams = []
    for i in range(16):     # test_acceptance.py:253-263
        along = (i / 15.0 - 0.5) * 2.0 * span
        altitude = 8.0 + 3.0 * (i % 4)
        eye = center + (np.array([along, -1.5 * span, altitude]) if i % 2 == 0
                        else np.array([-1.5 * span, along, altitude]))
        cams.append(look_at(eye, center, 96, 72, 80.0))
    return cams


def test_fused_renders_byte_identical_to_original(city):
    import paper_2404_01133_b200 as cs
    from paper_2404_01133_b200 import fusion
    from paper_2404_01133_b200.core import GaussianCloud
    cloud = GaussianCloud(city.positions, city.opacities, city.scales, city.rotations, city.sh)
    pmin, pmax = _central_third(np.asarray(cloud.positions))
    mem = O.block_of_points(cloud.positions, pmin, pmax, (2, 2))
    slices = [(cloud.take(np.nonzero(mem == j)[0]), j) for j in range(4)]
    fused = fusion.fuse_device(slices, pmin, pmax, (2, 2))
    assert fused.count == cloud.count
    fused_cloud = GaussianCloud(fused.positions, fused.opacities, fused.scales, fused.rotations, fused.sh)
    st = cs.RenderSettings()
    n_diff_order = 0
    for i, cam in enumerate(_seam_views(pmin, pmax)):
        a, sa = cs.rasterize_stats(cloud, cam, st)
        b, sb = cs.rasterize_stats(fused_cloud, cam, st)
        assert sa.visible_splats == sb.visible_splats and sa.blended_fragments == sb.blended_fragments, i
        assert np.array_equal(a.pixels, b.pixels), f"seam view {i}"
        da = cs.render(cloud, cam, st).cpu().numpy()
        db = cs.render(fused_cloud, cam, st).cpu().numpy()
        assert da.tobytes() == db.tobytes(), f"seam view {i} (device tier)"
        n_diff_order += sa.visible_splats > 0
    assert n_diff_order >= 12


def test_permutation_invariance_bitwise(city):
    import paper_2404_01133_b200 as cs
    from paper_2404_01133_b200.core import GaussianCloud
    from paper_2404_01133_b200.render import bin_tiles_last, project_cloud
    from paper_2404_01133_b200.synth import city_cameras
    cloud = GaussianCloud(city.positions, city.opacities, city.scales, city.rotations, city.sh)
    perm = np.random.default_rng(3).permutation(cloud.count)
    inv = np.argsort(perm)
    shuffled = cloud.take(perm)
    st = cs.RenderSettings()
    for cam in city_cameras(8, 100.0, 320, 240, seed=0)[:6]:
        p = project_cloud(cloud, cam, st)
        if len(np.unique(p["depths"])) != p["count"]:
            continue          # exact depth ties: the index tie-break legitimately differs
        a, sa = cs.rasterize_stats(cloud, cam, st)
        ta, oa = bin_tiles_last(cam, st.tile_size)
        b, sb = cs.rasterize_stats(shuffled, cam, st)
        tb, ob = bin_tiles_last(cam, st.tile_size)
        assert a.pixels.tobytes() == b.pixels.tobytes()
        assert sa.blended_fragments == sb.blended_fragments and sa.visible_splats == sb.visible_splats
        assert np.array_equal(oa, ob) and np.array_equal(ta, tb)   # depth-rank lists are identical
        q = project_cloud(shuffled, cam, st)
        assert np.array_equal(perm[q["source"]], p["source"])      # same splats, same order
        assert np.array_equal(inv[perm], np.arange(cloud.count))

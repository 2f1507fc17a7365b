"""Tile-local binning (cs_tiles.cu) vs the global tile sort and the oracle.

Both binning paths must give render._bin_tiles' lists (render.py:217-249)
bit for bit: the tile-local path sorts each tile's depth ranks in shared
memory (one piece up to 16384 entries, two pieces + merge up to 32768), the
global path emits pairs in depth order and sorts them stably by tile.
CS_TL_MAX lowers the tile-local limit per call (0 forces the global path)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _tile_local_on(monkeypatch):
    """The tile-local path is opt-in (CS_TILE_LOCAL=1, read per frame)."""
    monkeypatch.setenv("CS_TILE_LOCAL", "1")


@pytest.fixture(scope="module")
def city():
    from paper_2404_01133_b200.synth import city_cameras, generate_city
    c = generate_city(seed=5, extent=80.0, n_buildings=30, n_gaussians=150_000)
    cams = city_cameras(6, 80.0, 1280, 720, seed=5)
    return c, cams


def _render(cloud, cam, tl_max=None):
    import paper_2404_01133_b200 as cs
    from paper_2404_01133_b200.render import bin_tiles_last, binning_path_last
    old = os.environ.get("CS_TL_MAX")
    if tl_max is None:
        os.environ.pop("CS_TL_MAX", None)
    else:
        os.environ["CS_TL_MAX"] = str(tl_max)
    try:
        img, stats = cs.rasterize_stats(cloud, cam, cs.RenderSettings())
        tid, off = bin_tiles_last(cam, 16)
        path = binning_path_last()
    finally:
        if old is None:
            os.environ.pop("CS_TL_MAX", None)
        else:
            os.environ["CS_TL_MAX"] = old
    return img, stats, tid, off, path


@pytest.mark.parametrize("ci", [0, 3, 5])
def test_tile_local_equals_global_and_oracle(city, ci):
    from oracle import oracle as O
    import paper_2404_01133_b200 as cs
    cloud, cams = city
    cam = cams[ci]
    img_t, st_t, tid_t, off_t, path_t = _render(cloud, cam)
    img_g, st_g, tid_g, off_g, path_g = _render(cloud, cam, tl_max=0)
    assert path_t == "tile_local" and path_g == "global"
    assert np.array_equal(off_t, off_g) and np.array_equal(tid_t, tid_g)
    assert np.array_equal(img_t.pixels, img_g.pixels)
    assert st_t.blended_fragments == st_g.blended_fragments
    ref_p = O.project_cloud(cloud, cam, cs.RenderSettings())
    rtid, roff, _, _ = O.bin_tiles(ref_p, cam, 16)
    assert np.array_equal(off_t, roff) and np.array_equal(tid_t, rtid)


@pytest.mark.parametrize("limit", [300, 1500, 5000])
def test_size_classes_and_fallback(city, limit):
    """Frames whose largest tile exceeds the limit take the global path; below
    it every size class of the per-tile sort is exercised."""
    cloud, cams = city
    cam = cams[1]
    _, _, tid_ref, off_ref, _ = _render(cloud, cam, tl_max=0)
    n_max = int(np.diff(off_ref).max())
    _, _, tid, off, path = _render(cloud, cam, tl_max=limit)
    assert path == ("tile_local" if n_max <= limit else "global")
    assert np.array_equal(off, off_ref) and np.array_equal(tid, tid_ref)


@pytest.mark.parametrize("n", [90_000, 150_000])
def test_two_piece_merge_tiles(n):
    """Tiles above 16384 entries (two sorted pieces + merge path): a dense
    cluster in front of the camera piles > 16k splats onto a few tiles; at
    150k the largest tile passes 32768 and the frame takes the global path."""
    from oracle import oracle as O
    import paper_2404_01133_b200 as cs
    from paper_2404_01133_b200.core import CameraView, GaussianCloud
    rng = np.random.default_rng(11)
    pos = np.column_stack([rng.normal(0, 0.4, n), rng.normal(0, 0.4, n), rng.uniform(4, 30, n)])
    cloud = GaussianCloud(positions=pos, opacities=rng.uniform(0.05, 0.3, n),
                          scales=np.full((n, 3), 0.02) * rng.uniform(0.5, 2, (n, 1)),
                          rotations=np.tile([1.0, 0, 0, 0], (n, 1)),
                          sh=rng.normal(0, 0.3, (n, 3, 1)))
    f = 120.0 / np.tan(np.radians(10.0))
    cam = CameraView(width=320, height=240, fx=f, fy=f, cx=160.0, cy=120.0,
                     rotation_w2c=np.eye(3), translation_w2c=np.zeros(3))
    img, st, tid, off, path = _render(cloud, cam)
    n_max = int(np.diff(off).max())
    assert n_max > 16384, n_max
    assert path == ("tile_local" if n_max <= 32768 else "global")
    assert (n_max <= 32768) == (n == 90_000), n_max
    ref_p = O.project_cloud(cloud, cam, cs.RenderSettings())
    rtid, roff, _, _ = O.bin_tiles(ref_p, cam, 16)
    assert np.array_equal(off, roff) and np.array_equal(tid, rtid)
    rimg, rst = O.rasterize_stats(cloud, cam, cs.RenderSettings())
    assert np.abs(img.pixels - rimg).max() <= 1e-4
    assert st.blended_fragments == rst["blended_fragments"]

"""CUDA path vs the reference's golden vectors and the CPU oracle (needs a B200).

Bar (BASELINE.json north star): visible set, LoD levels and sorted tile-key
lists bit-exact; images within max-abs 1e-4; fragment counts equal.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4      # north-star image tolerance (max-abs)
COLOR_TOL = 1e-6    # float32 SH rows, float64 evaluation
EXACT = ("means", "conics", "covs", "depths", "opacities", "radii", "source")


@pytest.fixture(scope="module")
def cs():
    import paper_2404_01133_b200 as cs
    return cs


def test_golden_projection_bitexact(cs, golden_render):
    from paper_2404_01133_b200.render import project_cloud
    for name in golden_render.cases():
        cloud = golden_render.cloud(name)
        cam = golden_render.camera(name)
        st = golden_render.settings(name)
        p = project_cloud(cloud, cam, st)
        assert p["count"] == int(golden_render[f"{name}/visible"]), name
        assert p["skipped_singular"] == int(golden_render[f"{name}/p_skipped"]), name
        for f in EXACT:
            ref = golden_render[f"{name}/p_{f}"]
            assert np.array_equal(p[f].reshape(ref.shape), ref), (name, f)
        if p["count"]:
            np.testing.assert_allclose(p["colors"], golden_render[f"{name}/p_colors"], atol=COLOR_TOL)


def test_golden_tiles_image_stats(cs, golden_render):
    from paper_2404_01133_b200.render import bin_tiles_last
    for name in golden_render.cases():
        cloud = golden_render.cloud(name)
        cam = golden_render.camera(name)
        st = golden_render.settings(name)
        img, stats = cs.rasterize_stats(cloud, cam, st)
        tid, off = bin_tiles_last(cam, st.tile_size)
        assert np.array_equal(tid, golden_render[f"{name}/tile_ids"]), name
        assert np.array_equal(off, golden_render[f"{name}/offsets"]), name
        ref = golden_render[f"{name}/image"]
        assert img.pixels.shape == ref.shape
        assert np.abs(img.pixels - ref).max() <= IMG_TOL, name
        assert stats.visible_splats == int(golden_render[f"{name}/visible"]), name
        assert stats.blended_fragments == int(golden_render[f"{name}/fragments"]), name
        assert stats.skipped_singular == int(golden_render[f"{name}/skipped"]), name


def test_closed_forms(cs, golden_render):
    # test_render.py:155-191 at the north-star tolerance
    img, _ = cs.rasterize_stats(golden_render.cloud("opaque_center"), golden_render.camera("opaque_center"),
                                golden_render.settings("opaque_center"))
    np.testing.assert_allclose(img.pixels[24, 32], 0.99 * np.array([1.0, 0.5, 0.0]) + 0.01 * 0.2, atol=1e-6)
    img, st = cs.rasterize_stats(golden_render.cloud("t_floor_drop"), golden_render.camera("t_floor_drop"),
                                 golden_render.settings("t_floor_drop"))
    assert st.blended_fragments == 2 and st.visible_splats == 3


def _lod(golden_city):
    return golden_city.lod()


def test_golden_lod_decisions(cs, golden_city):
    lod = _lod(golden_city)
    for name in golden_city.cases():
        cam = golden_city.camera(name)
        dec = cs.decide_visibility(lod, cam)
        assert np.array_equal(np.array([d.visible for d in dec]), golden_city[f"{name}/dec_visible"]), name
        assert np.array_equal(np.array([-1 if d.level is None else d.level for d in dec]),
                              golden_city[f"{name}/dec_level"]), name
        assert np.array_equal(np.array([d.distance for d in dec]), golden_city[f"{name}/dec_distance"]), name
        box = np.array([d.screen_box if d.screen_box else (np.nan,) * 4 for d in dec])
        assert np.array_equal(box, golden_city[f"{name}/dec_box"], equal_nan=True), name


@pytest.mark.parametrize("tag,kw", [("block", {}), ("forced", {"force_level": 2}),
                                    ("point", {"mode": "pointwise"})])
def test_golden_lod_assembly_render(cs, golden_city, tag, kw):
    from paper_2404_01133_b200.render import bin_tiles_last, project_cloud
    lod = _lod(golden_city)
    for name in golden_city.cases():
        cam = golden_city.camera(name)
        a = cs.assemble_render_set(lod, cam, **kw)
        assert a.cloud.count == int(golden_city[f"{name}/{tag}_count"]), (name, tag)
        if golden_city.has(f"{name}/{tag}_positions"):
            ref = golden_city[f"{name}/{tag}_positions"]
            assert np.array_equal(np.asarray(a.cloud.positions, dtype=np.float32), ref), name
        if golden_city.has(f"{name}/{tag}/image"):
            p = project_cloud(a.cloud, cam)
            for f in EXACT:
                ref = golden_city[f"{name}/{tag}/p_{f}"]
                assert np.array_equal(p[f].reshape(ref.shape), ref), (name, tag, f)
            img, stats = cs.rasterize_stats(a.cloud, cam)
            tid, off = bin_tiles_last(cam, 16)
            assert np.array_equal(tid, golden_city[f"{name}/{tag}/tile_ids"]), name
            assert np.abs(img.pixels - golden_city[f"{name}/{tag}/image"]).max() <= IMG_TOL
            assert stats.blended_fragments == int(golden_city[f"{name}/{tag}/fragments"])


def test_select_level_and_block_visible(cs):
    ints = ((0.0, 200.0), (200.0, 400.0), (400.0, float("inf")))
    assert cs.select_level(100.0, ints) == 2
    assert cs.select_level(250.0, ints) == 1
    assert cs.select_level(10_000.0, ints) == 0
    assert cs.select_level(0.0, ints) == 2 and cs.select_level(200.0, ints) == 1
    with pytest.raises(ValueError):
        cs.select_level(-1.0, ints)
    from paper_2404_01133_b200.core import CameraView
    cam = CameraView(64, 48, 55.0, 55.0, 32.0, 24.0, np.eye(3), np.zeros(3))
    v, d = cs.block_visible((np.full(3, -1.0), np.full(3, 1.0)), cam)
    assert v and d == 0.0
    v, d = cs.block_visible((np.array([-1.0, -1, -9]), np.array([1.0, 1, -5])), cam)
    assert not v and d == pytest.approx(np.sqrt(27.0))
    v, _ = cs.block_visible((np.array([8.0, -1.0, 9.0]), np.array([10.0, 1.0, 11.0])), cam)
    assert not v


def test_fuse_filter_matches_golden(cs, golden_fuse):
    from paper_2404_01133_b200.fusion import fuse_device
    ids = [int(j) for j in golden_fuse["block_ids"]]
    blocks = [(golden_fuse.cloud(f"block{j}"), j) for j in ids]
    fused = fuse_device(list(reversed(blocks)), golden_fuse["p_min"], golden_fuse["p_max"],
                        tuple(int(d) for d in golden_fuse["dims"]))
    ref = golden_fuse.cloud("fused")
    for f in ("positions", "opacities", "scales", "rotations", "sh"):
        assert np.array_equal(np.asarray(getattr(fused, f)), getattr(ref, f)), f


# ---------------------------------------------------------------------------
# larger scenes vs the oracle (same arrays on both sides)

@pytest.fixture(scope="module")
def city200k():
    from paper_2404_01133_b200.synth import city_cameras, generate_city
    c = generate_city(seed=1, extent=100.0, n_buildings=40, n_gaussians=200_000)
    cams = city_cameras(8, 100.0, 1920, 1080, seed=1)
    return c, cams


@pytest.mark.parametrize("ci", [0, 2, 5, 7])
def test_city_1080p_vs_oracle(cs, city200k, ci):
    from oracle import oracle as O
    from paper_2404_01133_b200.render import bin_tiles_last, project_cloud
    cloud, cams = city200k
    cam = cams[ci]
    st = cs.RenderSettings()
    ref_p = O.project_cloud(cloud, cam, st)
    p = project_cloud(cloud, cam, st)
    assert p["count"] == ref_p["count"]
    for f in EXACT:
        assert np.array_equal(p[f], ref_p[f]), f
    img, stats = cs.rasterize_stats(cloud, cam, st)
    tid, off = bin_tiles_last(cam, 16)
    rtid, roff, _, _ = O.bin_tiles(ref_p, cam, 16)
    assert np.array_equal(off, roff)
    assert np.array_equal(tid, rtid)
    rimg, rstats = O.rasterize_stats(cloud, cam, st)
    assert np.abs(img.pixels - rimg).max() <= IMG_TOL
    assert stats.blended_fragments == rstats["blended_fragments"]
    assert stats.visible_splats == rstats["visible_splats"]


def test_device_tier_matches_compat(cs, city200k):
    cloud, cams = city200k
    img, _ = cs.rasterize_stats(cloud, cams[3])
    t = cs.render(cloud, cams[3])
    torch.cuda.synchronize()
    assert t.dtype == torch.float32 and tuple(t.shape) == (1080, 1920, 3)
    assert np.abs(t.cpu().numpy().astype(np.float64) - img.pixels).max() <= 1e-6


def test_blend_tiles_mirror_vs_oracle(cs, golden_render):
    """cs_blend_tiles has the numba kernel's exact argument list (_kernels.py:18-30)."""
    from oracle import oracle as O
    from paper_2404_01133_b200 import _lib, device
    name = "dense"
    cloud, cam, st = golden_render.cloud(name), golden_render.camera(name), golden_render.settings(name)
    p = O.project_cloud(cloud, cam, st)
    tid, off, ntx, nty = O.bin_tiles(p, cam, st.tile_size)
    ref_out, ref_frag = O.blend_tiles(tid, off, p, cam, st)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    out = torch.empty((cam.height, cam.width, 3), dtype=torch.float64, device="cuda")
    frag = torch.zeros(ntx * nty, dtype=torch.int64, device="cuda")
    args = [d(tid), d(off), ntx * nty, d(p["means"]), d(p["conics"]), d(p["colors"]), d(p["opacities"]),
            p["count"], d(np.array(st.background)), st.tile_size, cam.width, cam.height, ntx,
            st.alpha_floor, st.transmittance_floor, out, frag]
    ptrs = [a.data_ptr() if isinstance(a, torch.Tensor) else a for a in args]
    _lib.check(_lib.load().cs_blend_tiles(device.context(), *ptrs, device.stream_handle()))
    torch.cuda.synchronize()
    assert np.abs(out.cpu().numpy() - ref_out).max() <= 1e-6
    assert np.array_equal(frag.cpu().numpy(), ref_frag)

"""Pin the CPU oracle against the reference's own outputs (tests/golden/).

The oracle (oracle/cs_oracle.c) is the parity checker for the CUDA path, so it
is itself checked bit for bit against vectors the reference produced
(tests/golden/make_golden.py).  Decision quantities must be bit-identical;
images within 1e-12 (both are float64 with the same op order; only libm exp
may differ in the last ulp).
"""

import math

import numpy as np
import pytest

from oracle import oracle as O

FIELDS = ("means", "conics", "covs", "depths", "opacities", "radii", "source")


def test_render_cases_projection_bitexact(golden_render):
    for name in golden_render.cases():
        cloud = golden_render.cloud(name)
        cam = golden_render.camera(name)
        st = golden_render.settings(name)
        p = O.project_cloud(cloud, cam, st)
        assert p["count"] == int(golden_render[f"{name}/visible"]), name
        assert p["skipped_singular"] == int(golden_render[f"{name}/p_skipped"]), name
        for f in FIELDS:
            ref = golden_render[f"{name}/p_{f}"]
            assert np.array_equal(p[f].reshape(ref.shape), ref), (name, f)
        np.testing.assert_allclose(p["colors"].reshape(-1, 3) if p["count"] else np.zeros((0, 3)),
                                   golden_render[f"{name}/p_colors"].reshape(-1, 3), atol=1e-12)


def test_render_cases_tiles_and_image(golden_render):
    for name in golden_render.cases():
        cloud = golden_render.cloud(name)
        cam = golden_render.camera(name)
        st = golden_render.settings(name)
        p = O.project_cloud(cloud, cam, st)
        tid, off, _, _ = O.bin_tiles(p, cam, st.tile_size)
        assert np.array_equal(tid, golden_render[f"{name}/tile_ids"]), name
        assert np.array_equal(off, golden_render[f"{name}/offsets"]), name
        img, stats = O.rasterize_stats(cloud, cam, st)
        np.testing.assert_allclose(img, golden_render[f"{name}/image"], atol=1e-12, err_msg=name)
        assert stats["blended_fragments"] == int(golden_render[f"{name}/fragments"]), name
        assert stats["visible_splats"] == int(golden_render[f"{name}/visible"]), name


def test_closed_form_cases(golden_render):
    # test_render.py:155-191 closed forms, through the oracle
    img = golden_render["opaque_center/image"]
    np.testing.assert_allclose(img[24, 32], 0.99 * np.array([1.0, 0.5, 0.0]) + 0.01 * 0.2, atol=1e-12)
    img = golden_render["two_coincident/image"]
    np.testing.assert_allclose(img[24, 32], [0.5, 0.25, 0.25], atol=1e-12)
    assert int(golden_render["t_floor_drop/fragments"]) == 2
    assert int(golden_render["t_floor_drop/visible"]) == 3
    assert int(golden_render["near_cull/visible"]) == 1


def test_city_decisions_bitexact(golden_city):
    lod = golden_city.lod()
    for name in golden_city.cases():
        cam = golden_city.camera(name)
        dec = O.decide_visibility(lod, cam)
        vis = np.array([d[1] for d in dec])
        lev = np.array([-1 if d[2] is None else d[2] for d in dec])
        dist = np.array([d[3] for d in dec])
        assert np.array_equal(vis, golden_city[f"{name}/dec_visible"]), name
        assert np.array_equal(lev, golden_city[f"{name}/dec_level"]), name
        assert np.array_equal(dist, golden_city[f"{name}/dec_distance"]), name
        box = np.array([d[4] if d[4] is not None else (np.nan,) * 4 for d in dec])
        assert np.array_equal(box, golden_city[f"{name}/dec_box"], equal_nan=True), name


@pytest.mark.parametrize("tag,kw", [("block", {}), ("forced", {"force_level": 2}),
                                    ("point", {"mode": "pointwise"})])
def test_city_assembly_and_render(golden_city, tag, kw):
    lod = golden_city.lod()
    for i, name in enumerate(golden_city.cases()):
        cam = golden_city.camera(name)
        cloud, _ = O.assemble(lod, cam, **kw)
        assert cloud.count == int(golden_city[f"{name}/{tag}_count"]), name
        if golden_city.has(f"{name}/{tag}_positions"):
            ref = golden_city[f"{name}/{tag}_positions"]
            assert np.array_equal(np.asarray(cloud.positions, dtype=np.float32), ref), name
        if golden_city.has(f"{name}/{tag}/image"):
            p = O.project_cloud(cloud, cam, None)
            for f in FIELDS:
                ref = golden_city[f"{name}/{tag}/p_{f}"]
                assert np.array_equal(p[f].reshape(ref.shape), ref), (name, tag, f)
            tid, off, _, _ = O.bin_tiles(p, cam, 16)
            assert np.array_equal(tid, golden_city[f"{name}/{tag}/tile_ids"]), name
            img, stats = O.rasterize_stats(cloud, cam, None)
            np.testing.assert_allclose(img, golden_city[f"{name}/{tag}/image"], atol=1e-12)
            assert stats["blended_fragments"] == int(golden_city[f"{name}/{tag}/fragments"])


def test_fuse_bitexact(golden_fuse):
    ids = [int(j) for j in golden_fuse["block_ids"]]
    blocks = [(golden_fuse.cloud(f"block{j}"), j) for j in ids]
    fused = O.fuse(list(reversed(blocks)), golden_fuse["p_min"], golden_fuse["p_max"],
                   tuple(golden_fuse["dims"]))
    ref = golden_fuse.cloud("fused")
    for f in ("positions", "opacities", "scales", "rotations", "sh"):
        assert np.array_equal(np.asarray(getattr(fused, f)), getattr(ref, f)), f


def test_select_level_edges_oracle():
    # test_lod.py:266-279 semantics through the decision routine
    ints = ((0.0, 200.0), (200.0, 400.0), (400.0, math.inf))
    from types import SimpleNamespace
    cam = SimpleNamespace(rotation_w2c=np.eye(3), translation_w2c=np.zeros(3),
                          camera_center=np.zeros(3), fx=55.0, fy=55.0, cx=32.0, cy=24.0,
                          width=64, height=48)
    for d, want in ((100.0, 2), (250.0, 1), (10_000.0, 0), (200.0, 1), (400.0, 0)):
        lo = np.array([[-1.0, -1.0, d]])
        hi = np.array([[1.0, 1.0, d + 10]])
        empty = SimpleNamespace(positions=np.zeros((1, 3)), count=1)
        lod = SimpleNamespace(levels=((empty,), (empty,), (empty,)), bounds_min=lo, bounds_max=hi,
                              distance_intervals=ints)
        dec = O.decide_visibility(lod, cam)
        assert dec[0][1]
        dd = dec[0][3]
        expect = [2 - i for i, (a, b) in enumerate(ints) if a <= dd < b][0]
        assert dec[0][2] == expect


def test_primitive_golden_vs_oracle():
    """tests/golden/primitive.npz (the reference's project_gaussian,
    render.py:191-214) against the oracle's projection of the same single
    Gaussians: geometry bit-exact, culled cases absent."""
    from pathlib import Path
    from types import SimpleNamespace
    z = np.load(Path(__file__).resolve().parent / "golden" / "primitive.npz")

    class _Cam(SimpleNamespace):
        pass
    for i in range(len(z["culled"])):
        row = z["cam"][i]
        R = row[6:15].reshape(3, 3)
        t = row[15:18]
        cam = _Cam(width=int(row[0]), height=int(row[1]), fx=row[2], fy=row[3], cx=row[4], cy=row[5],
                   rotation_w2c=R, translation_w2c=t, camera_center=-(R.T @ t))
        cloud = SimpleNamespace(positions=z["pos"][i][None], opacities=np.array([z["op"][i]]),
                                scales=z["scale"][i][None], rotations=z["rot"][i][None], sh=z["sh"][i][None])
        st = O.DefaultSettings()
        st.sh_degree = int(z["degree"][i])
        p = O.project_cloud(cloud, cam, st)
        if z["culled"][i]:
            assert p["count"] == 0, i
            continue
        assert p["count"] == 1, i
        assert np.array_equal(p["means"][0], z["mean2d"][i]), i
        a, b, c = p["covs"][0]
        assert np.array_equal(np.array([[a, b], [b, c]]), z["cov2d"][i]), i
        assert p["depths"][0] == z["depth"][i], i

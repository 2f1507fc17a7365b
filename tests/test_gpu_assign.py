"""Training-data assignment on the GPU (partition.assign / assign_b1 /
assign_b2 / enlarge_bounds over cs_render exclusion masks, cs_ssim and
cs_bounds_contain) vs the reference's golden vectors and the CPU oracle
(needs a B200).

Bar: entries, provenance, enlarged bounds and enlargement counts identical;
the contribution l_ssim within 2e-5 of the reference's (the device renders
accumulate colour in float32; SSIM itself is float64 and agrees
with scipy's to ~1e-15 on identical images); the masked render equals the
render of cloud.take(~mask) bit for bit."""

from types import SimpleNamespace

import numpy as np
import pytest
import torch

from conftest import assign_inputs
from oracle import oracle as O

pytestmark = pytest.mark.gpu

L_TOL = 2e-5


@pytest.fixture(scope="module")
def P():
    from paper_2404_01133_b200 import partition
    return partition


def test_golden_assign(P, golden_assign):
    g = golden_assign
    cloud, views, grid, st = assign_inputs(g)
    res, l = P.assign(views, grid, cloud, float(g["epsilon"]), settings=st,
                      assignment_scale=float(g["scale"]), enlarge_min_count=int(g["min_count"]),
                      return_l_ssim=True)
    fin = np.isfinite(g["l_ssim"])
    assert np.array_equal(np.isfinite(l), fin)
    np.testing.assert_allclose(l[fin], g["l_ssim"][fin], atol=L_TOL, rtol=0)
    assert np.array_equal(res.entries, g["entries"])
    assert np.array_equal(res.provenance, g["provenance"])
    assert np.array_equal(res.bounds_min_used, g["bounds_min_used"])
    assert np.array_equal(res.bounds_max_used, g["bounds_max_used"])
    assert res.unassignable == ()
    assert res.n_poses == len(views) and res.n_blocks == grid.n_blocks


def test_masked_render_equals_rest_cloud(P, golden_assign):
    import paper_2404_01133_b200 as cs
    g = golden_assign
    cloud, views, grid, st = assign_inputs(g)
    cam = P._scaled_camera(cs.CameraView(**{k: getattr(views[3], k) for k in (
        "width", "height", "fx", "fy", "cx", "cy")}, rotation_w2c=views[3].rotation_w2c,
        translation_w2c=views[3].translation_w2c), 1.0)
    r = P._Renderer(cloud, st)
    for j in (0, 6, 19):
        mask = P._mask_for(grid, j, None)
        a = r(cam, mask).cpu().numpy()
        keep = np.nonzero(np.asarray(grid.membership) != j)[0]
        rest = SimpleNamespace(positions=cloud.positions[keep], opacities=cloud.opacities[keep],
                               scales=cloud.scales[keep], rotations=cloud.rotations[keep],
                               sh=cloud.sh[keep], count=keep.size)
        b = P._Renderer(rest, st)(cam).cpu().numpy()
        assert np.array_equal(a, b), j


def test_ssim_kernel_vs_oracle(P):
    rng = np.random.default_rng(4)
    for (h, w) in ((11, 11), (37, 53), (135, 240)):
        a = rng.uniform(0, 1, (h, w, 3)).astype(np.float32)
        b = np.clip(a + rng.normal(0, 0.05, a.shape), 0, 1).astype(np.float32)
        got = P._l_ssim_host_images(a, b)
        want = 1.0 - O.ssim(a.astype(np.float64), b.astype(np.float64))
        assert abs(got - want) < 1e-12, (h, w, got, want)
        assert abs(P._l_ssim_host_images(a, a)) < 1e-14
    with pytest.raises(ValueError):
        P._l_ssim_host_images(np.zeros((10, 20, 3), np.float32), np.zeros((10, 20, 3), np.float32))


def test_enlarge_and_b2_vs_oracle(P, golden_assign):
    g = golden_assign
    cloud, views, grid, st = assign_inputs(g)
    for j in range(grid.n_blocks):
        lo, hi = P.enlarge_bounds(j, grid, 900)
        olo, ohi = O.enlarge_bounds(j, grid.bounds_min, grid.bounds_max, grid.contracted, 900)
        assert np.array_equal(lo, olo) and np.array_equal(hi, ohi), j
    centers = O.contract_normalized(np.stack([v.camera_center for v in views]), grid.map.p_min,
                                    grid.map.p_max)
    for j in range(grid.n_blocks):
        want = O.bounds_contain(centers, grid.bounds_min[j], grid.bounds_max[j])
        got = [P.assign_b2(v, j, grid) for v in views]
        assert got == list(want), j
    with pytest.warns(UserWarning):
        lo, hi = P.enlarge_bounds(0, grid, 10 ** 9)
    assert (lo == -2.0).all() and (hi == 2.0).all()


def test_assign_b1_and_renderer_hook(P, golden_assign):
    import paper_2404_01133_b200 as cs
    from paper_2404_01133_b200.core import GaussianCloud
    g = golden_assign
    cloud, views, grid, st = assign_inputs(g)
    eps = float(g["epsilon"])
    scaled = [P._scaled_camera(cs.CameraView(width=v.width, height=v.height, fx=v.fx, fy=v.fy, cx=v.cx,
                                             cy=v.cy, rotation_w2c=v.rotation_w2c,
                                             translation_w2c=v.translation_w2c), float(g["scale"]))
              for v in views]
    for (i, j) in ((0, 1), (2, 9), (5, 22)):
        want = bool(g["l_ssim"][i, j] > eps)
        assert P.assign_b1(scaled[i], j, cloud, grid, eps) == want
    hc = GaussianCloud(*(np.asarray(a, dtype=np.float64) for a in (
        cloud.positions, cloud.opacities, cloud.scales, cloud.rotations, cloud.sh)))
    rs = cs.RenderSettings()
    res = P.assign(views[:4], grid, hc, eps, assignment_scale=float(g["scale"]),
                   enlarge_min_count=int(g["min_count"]),
                   renderer=lambda c, cam: cs.rasterize(c, cam, rs))
    dev = P.assign(views[:4], grid, hc, eps, assignment_scale=float(g["scale"]),
                   enlarge_min_count=int(g["min_count"]))
    assert np.array_equal(res.entries, dev.entries)
    assert np.array_equal(res.provenance, dev.provenance)
    with pytest.raises(ValueError):
        P.assign(views, grid, hc, 1.5)


def test_failed_pose_is_unassignable(P, golden_assign):
    g = golden_assign
    cloud, views, grid, st = assign_inputs(g)
    bad = SimpleNamespace(**{k: getattr(views[0], k) for k in (
        "rotation_w2c", "translation_w2c", "camera_center", "fx", "fy", "cx", "cy", "height")}, width=0)
    res = P.assign([views[1], bad], grid, cloud, float(g["epsilon"]), settings=st,
                   assignment_scale=float(g["scale"]), enlarge_min_count=int(g["min_count"]))
    assert [u[0] for u in res.unassignable] == [1]
    assert not res.entries[1].any()

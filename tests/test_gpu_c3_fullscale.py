"""Full-scale parity on the headline configuration (BASELINE.json configs[2], C3).

The bench's own scene -- the 23M-Gaussian synthetic city, 6x6 blocks, three
detail levels built on the device, intervals 0/200/400 m, 1920x1080 orbit
flythrough at 150/300/500 m (bench.build_scene / bench.flythrough) -- against
the C oracle on identical inputs (the level clouds copied to the host):

* two frames per altitude, all of them frames the bench times with its
  default strided schedule (``bench.timed_frames``), including the 150 m
  orbit: every block decision of ``decide_visibility`` (lod.py:330-348:
  visible, level, distance, screen box) bit-exact, the assembled count
  (lod.py:360-401), the depth order (``source``, render.py:176-177), the full
  sorted tile list and CSR offsets (render.py:217-249) bit-exact, accepted
  fragments equal and the image within 1e-4;
* one frame with every visible block forced to the finest level
  (cmd_bench's ``finest`` mode, cli.py:250-258);
* one no-LoD frame of the whole 23M cloud (cmd_bench's ``full`` mode, the
  paper's ablation PAPER.md:276-280) from a low orbit inside the city: > 10^8
  tile pairs, which exercises the heavy-chunk emission and the large pair
  buffers.

Bar (north star): visible set, LoD levels and sorted tile keys bit-exact;
images within max-abs 1e-4; fragment counts equal.
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu
IMG_TOL = 1e-4
LOD_FRAMES = (0, 9, 21, 30, 45, 57)   # 150 m: 0, 9; 300 m: 21, 30; 500 m: 45, 57


@pytest.fixture(scope="module")
def c3():
    import bench
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    scene, center, radius, alts, wh, _, raw = bench.build_scene("c3", 0, dev, keep_raw=True)
    cams = bench.flythrough(center, radius, alts, wh, 20)
    assert set(LOD_FRAMES) <= set(bench.timed_frames(len(cams), 20))
    hs = bench.host_scene(scene)
    yield scene, hs, cams, raw
    del scene, raw
    torch.cuda.empty_cache()


def _check_frame(cloud_dev, cloud_host, cam, count_expected=None, min_pairs=0):
    """GPU (compatibility tier) vs oracle on one assembled / full cloud."""
    import paper_2404_01133_b200 as cs
    from paper_2404_01133_b200.render import bin_tiles_last, project_cloud
    st = cs.RenderSettings()
    p = project_cloud(cloud_dev, cam, st)
    rp = O.project_cloud(cloud_host, cam, st, nthreads=0)
    assert p["count"] == rp["count"] > 0
    assert p["skipped_singular"] == rp["skipped_singular"]
    for f in ("source", "depths", "means", "conics", "radii"):
        assert np.array_equal(p[f], rp[f]), f
    del p
    img, stats = cs.rasterize_stats(cloud_dev, cam, st)
    assert stats.visible_splats == rp["count"]
    tid, off = bin_tiles_last(cam, st.tile_size)
    rtid, roff, _, _ = O.bin_tiles(rp, cam, st.tile_size)
    assert tid.shape == rtid.shape and tid.shape[0] >= min_pairs, (tid.shape, rtid.shape)
    assert np.array_equal(off, roff)
    assert np.array_equal(tid, rtid)
    del tid
    rimg, frags = O.blend_tiles(rtid, roff, rp, cam, st)
    assert stats.blended_fragments == int(frags.sum())
    err = float(np.abs(img.pixels - np.clip(rimg, 0.0, 1.0)).max())
    assert err <= IMG_TOL, err
    return dict(visible=rp["count"], pairs=int(rtid.shape[0]), fragments=int(frags.sum()), err=err)


@pytest.mark.parametrize("fi", LOD_FRAMES)
def test_c3_lod_frame_bit_exact(c3, fi):
    import paper_2404_01133_b200 as cs
    scene, hs, cams, _ = c3
    cam = cams[fi]
    dec = cs.decide_visibility(scene, cam)
    odec = O.decide_visibility(hs, cam)
    assert len(dec) == len(odec) == 36
    for d, o in zip(dec, odec):
        assert (d.block, d.visible, d.level, d.distance, d.screen_box) == o, (d, o)
    assert sum(d.visible for d in dec) > 0
    a = cs.assemble_render_set(scene, cam)
    ocloud, _ = O.assemble(hs, cam)
    assert a.cloud.count == ocloud.count > 1_000_000
    _check_frame(a.cloud, ocloud, cam)


def test_c3_finest_mode_frame(c3):
    import paper_2404_01133_b200 as cs
    scene, hs, cams, _ = c3
    cam = cams[30]
    finest = scene.n_levels - 1
    a = cs.assemble_render_set(scene, cam, force_level=finest)
    ocloud, odec = O.assemble(hs, cam, force_level=finest)
    assert a.cloud.count == ocloud.count
    assert [(d.visible, d.level) for d in a.decisions] == [(o[1], o[2]) for o in odec]
    _check_frame(a.cloud, ocloud, cam)


def test_c3_full_cloud_frame_over_1e8_pairs(c3):
    """No LoD: the whole 23M-Gaussian cloud from a low orbit inside the city
    (the flythrough's 150 m frames give ~3e7 pairs without LoD; lower, nearer
    views reach the 1e8-2e8 pairs of SURVEY.md Appendix C).  The view with the
    most pairs among a few low-altitude candidates is checked."""
    from types import SimpleNamespace
    import paper_2404_01133_b200 as cs
    from paper_2404_01133_b200 import device
    from paper_2404_01133_b200.synth import orbit_cameras
    scene, hs, cams, raw = c3
    pos, op, sc, q, sh, _, _ = raw
    full = device.DeviceCloud.from_torch(pos, op, sc, q, sh)
    lo = pos.double().min(dim=0).values.cpu().numpy()
    hi = pos.double().max(dim=0).values.cpu().numpy()
    center = 0.5 * (lo + hi)
    cands = []
    for alt, rad in ((60.0, 150.0), (40.0, 250.0), (30.0, 100.0), (80.0, 300.0)):
        cands += orbit_cameras(center, rad, alt, 3, 1920, 1080)
    pairs = []
    for cam in cands:
        _, st = cs.rasterize_stats(full, cam)
        from paper_2404_01133_b200.render import bin_tiles_last
        pairs.append(int(bin_tiles_last(cam, 16)[0].shape[0]))
    best = int(np.argmax(pairs))
    print("candidate pairs (M):", [round(p / 1e6, 1) for p in pairs])
    host = SimpleNamespace(positions=pos.cpu().numpy(), opacities=op.cpu().numpy(),
                           scales=sc.cpu().numpy(), rotations=q.cpu().numpy(), sh=sh.cpu().numpy(),
                           count=int(pos.shape[0]))
    r = _check_frame(full, host, cands[best], min_pairs=100_000_000)
    print("full-cloud frame:", r)

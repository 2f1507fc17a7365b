"""Failure paths are loud, and kept state cannot be confused (needs a B200).

* A tile-pair buffer overflow in an ASYNCHRONOUS frame (device tier, frame
  graphs) is raised by the context's next call (MemoryError); after it the
  buffers are grown and the frame renders identically to a synchronous one.
* A training forward that overflowed makes its backward raise instead of
  returning the gradients of an incomplete frame.
* Per-forward state handles: two training forwards before one backward (a
  multi-view loss) give exactly the gradients of the two separate
  forward/backward pairs, and a render in between changes nothing.
* An AssembledSet keeps the camera it was assembled for: rendering it from a
  second camera draws the first camera's LoD set (lod.py:360-401 returns a
  concrete cloud): the same splats, depth order and decisions bit for bit as
  rendering that set materialised (colours to 1e-6: per-level SH widths vs
  the zero-padded concatenation).

Each overflow test runs on a fresh thread, i.e. a fresh context whose pair
buffer has never been sized.
"""

import ctypes
import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _on_fresh_context(fn):
    box = {}

    def run():
        try:
            box["r"] = fn()
        except BaseException as e:  # noqa: BLE001 - re-raised on the test thread
            box["e"] = e
    t = threading.Thread(target=run)
    t.start()
    t.join()
    if "e" in box:
        raise box["e"]
    return box.get("r")


def _pair_heavy_scene(n=3000, W=1920, H=1080, seed=0):
    """Few Gaussians, each covering most of a 1080p frame: >> 8 pairs per splat."""
    rng = np.random.default_rng(seed)
    z = rng.uniform(3.0, 6.0, n)
    pos = np.stack([rng.uniform(-1, 1, n) * z * 0.3, rng.uniform(-1, 1, n) * z * 0.2, z], 1)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    from types import SimpleNamespace
    f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)
    cloud = SimpleNamespace(positions=f32(pos), opacities=f32(rng.uniform(0.01, 0.05, n)),
                            scales=f32(rng.uniform(0.6, 1.2, (n, 3))), rotations=f32(q),
                            sh=f32(rng.normal(0, 0.2, (n, 3, 16))), count=n)
    cam = SimpleNamespace(rotation_w2c=np.eye(3), translation_w2c=np.zeros(3), camera_center=np.zeros(3),
                          fx=0.8 * W, fy=0.8 * W, cx=W / 2.0, cy=H / 2.0, width=W, height=H)
    return cloud, cam


def test_async_overflow_is_raised_then_recovers():
    import paper_2404_01133_b200 as cs
    from paper_2404_01133_b200.render import check, render

    cloud, cam = _pair_heavy_scene()
    st = cs.RenderSettings()

    def body():
        img0 = render(cloud, cam, st)          # fresh context: pair buffer 1M < needed
        torch.cuda.synchronize()
        with pytest.raises(MemoryError, match="overflowed"):
            render(cloud, cam, st)             # the next call reports it
        img1 = render(cloud, cam, st).clone()  # grown: complete now
        check()                                # and nothing pending
        ref, stats = cs.rasterize_stats(cloud, cam, st)
        assert stats.visible_splats == cloud.count
        assert torch.equal(img1.cpu(), torch.from_numpy(ref.pixels.astype(np.float32)))
        assert not torch.equal(img0.cpu(), img1.cpu())   # the overflowed frame was incomplete
        return True
    assert _on_fresh_context(body)


def test_async_overflow_reported_by_check():
    import paper_2404_01133_b200 as cs
    from paper_2404_01133_b200.render import check, render
    cloud, cam = _pair_heavy_scene(seed=1)

    def body():
        render(cloud, cam, cs.RenderSettings())
        with pytest.raises(MemoryError):
            check()
        check()   # reported once
        return True
    assert _on_fresh_context(body)


def test_overflowed_training_forward_fails_backward():
    from paper_2404_01133_b200 import _lib, device
    from paper_2404_01133_b200.render import RenderSettings
    from paper_2404_01133_b200.train import TrainState
    cloud, cam = _pair_heavy_scene(seed=2)

    def body():
        dev = torch.device("cuda", 0)
        dc = device.DeviceCloud.from_arrays(cloud.positions, cloud.opacities, cloud.scales, cloud.rotations,
                                            cloud.sh)
        src = _lib.CsSource()
        src.kind = _lib.CS_SRC_CLOUD
        src.force_level = -1
        src.cloud = dc.desc()
        ccam, cset = device.camera_struct(cam), device.settings_struct(RenderSettings())
        out = torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device=dev)
        h = device.context(0)
        lib = _lib.load()
        st = ctypes.c_void_p()
        _lib.check(lib.cs_render_train(h, ctypes.byref(src), ctypes.byref(ccam), ctypes.byref(cset),
                                       out.data_ptr(), 0, ctypes.byref(st), device.stream_handle(dev)))
        state = TrainState(st)
        k = dc.count
        g = [torch.empty(s, dtype=torch.float32, device=dev) for s in ((k, 3), (k, 3), (k, 4), (k,), (k, 48))]
        grads = _lib.CsGrads(*(t.data_ptr() for t in g))
        dl = torch.ones_like(out)
        rc = lib.cs_render_backward(h, state.handle, dl.data_ptr(), ctypes.byref(grads),
                                    device.stream_handle(dev))
        assert rc == _lib.CS_ENOMEM, rc
        assert b"overflowed" in lib.cs_last_error()
        state.release()
        # grown: the same step now goes through
        st2 = ctypes.c_void_p()
        _lib.check(lib.cs_render_train(h, ctypes.byref(src), ctypes.byref(ccam), ctypes.byref(cset),
                                       out.data_ptr(), 0, ctypes.byref(st2), device.stream_handle(dev)))
        state2 = TrainState(st2)
        _lib.check(lib.cs_render_backward(h, state2.handle, dl.data_ptr(), ctypes.byref(grads),
                                          device.stream_handle(dev)))
        state2.release()
        return True
    assert _on_fresh_context(body)


def test_two_forwards_before_backward():
    """Multi-view loss: both forwards' states stay intact until the backward."""
    from paper_2404_01133_b200.render import render
    from paper_2404_01133_b200.train import rasterize_train
    from tests_helpers import small_scene
    cloud, cam_a, st = small_scene(5, k=40, width=64, height=48)
    cam_b = type(cam_a)(**{**vars(cam_a), "cx": cam_a.cx + 6.0, "cy": cam_a.cy - 3.0})
    t = lambda a: torch.tensor(np.asarray(a, dtype=np.float32), device="cuda", requires_grad=True)
    rng = np.random.default_rng(3)
    wa = torch.tensor(rng.normal(size=(48, 64, 3)), dtype=torch.float32, device="cuda")
    wb = torch.tensor(rng.normal(size=(48, 64, 3)), dtype=torch.float32, device="cuda")

    def grads(views):
        params = [t(cloud.positions), t(cloud.scales), t(cloud.rotations), t(cloud.opacities), t(cloud.sh)]
        loss = 0
        for cam, w in views:
            loss = loss + (rasterize_train(*params, cam, st) * w).sum()
        # an unrelated render between the forwards and the backward
        render(cloud, cam_b, st)
        loss.backward()
        return [p.grad.clone() for p in params]

    ga = grads([(cam_a, wa)])
    gb = grads([(cam_b, wb)])
    gab = grads([(cam_a, wa), (cam_b, wb)])
    for x, y, z in zip(ga, gb, gab):
        torch.testing.assert_close(z, x + y, rtol=1e-5, atol=1e-6)
    assert any(float((x - y).abs().max()) > 1e-4 for x, y in zip(ga, gb))   # the views differ


def test_assembled_set_keeps_its_camera(golden_city):
    import paper_2404_01133_b200 as cs
    from paper_2404_01133_b200.render import project_cloud
    lod = golden_city.lod()
    names = golden_city.cases()
    st = cs.RenderSettings()
    checked = 0
    for na, nb in zip(names, names[1:]):
        cam_a, cam_b = golden_city.camera(na), golden_city.camera(nb)
        a = cs.assemble_render_set(lod, cam_a)
        b = cs.assemble_render_set(lod, cam_b)
        if a.cloud.count == 0 or a.cloud.count == b.cloud.count:
            continue
        if cs.rasterize_stats(a.cloud, cam_b, st)[1].visible_splats == 0:
            continue
        img, stats = cs.rasterize_stats(a.cloud, cam_b, st)
        fixed = a.cloud.to_cloud()              # the concrete cloud the reference returns
        assert fixed.count == a.cloud.count
        rimg, rstats = cs.rasterize_stats(fixed, cam_b, st)
        assert stats.visible_splats == rstats.visible_splats
        assert stats.blended_fragments == rstats.blended_fragments
        # decision data bit-exact; colours may differ in the float32 last bit (the
        # LoD path evaluates each level at its own SH width, the concatenated
        # cloud at the zero-padded widest one: SURVEY.md section 7 H5)
        p = project_cloud(a.cloud, cam_b, st)
        q = project_cloud(fixed, cam_b, st)
        for f in ("source", "depths", "means", "conics", "radii", "opacities"):
            assert np.array_equal(p[f], q[f]), f
        assert p["count"] == q["count"]
        if p["count"]:
            assert np.abs(p["colors"] - q["colors"]).max() <= 1e-6
        assert np.abs(img.pixels - rimg.pixels).max() <= 1e-6
        # the re-selection for cam_b would have drawn a different set
        wrong, _ = cs.rasterize_stats(b.cloud, cam_b, st)
        assert stats.visible_splats != _.visible_splats or not np.array_equal(wrong.pixels, img.pixels)
        # and the device tier draws the same set
        dimg = cs.render(a.cloud, cam_b, st)
        assert np.abs(dimg.cpu().numpy() - rimg.pixels).max() <= 1e-6
        checked += 1
    assert checked >= 3

"""RenderService drop-in (service.py:114-238) against
the reference's own RenderService on the bundle scene (tests/golden/
service.npz, made by make_golden.make_service): metadata, validation and
LoD updates on the CPU; frames (decoded PNG pixels and the stats payload)
on the GPU."""

import io
import json
import math

import numpy as np
import pytest

from conftest import GOLDEN


@pytest.fixture(scope="module")
def service():
    from paper_2404_01133_b200 import bundle
    from paper_2404_01133_b200.service import RenderService
    return RenderService(bundle.load_lod(GOLDEN / "bundle"), max_dim=256)


def _body(g, k):
    return json.loads(str(g[f"req{k}/body"]))


def test_metadata_matches_reference(service, golden_service):
    assert service.scene_info() == json.loads(str(golden_service["scene_info"]))
    assert service.block_geometry() == json.loads(str(golden_service["blocks"]))


def test_camera_validation_names_field(golden_service):
    from paper_2404_01133_b200.service import BadRequest, camera_from_json
    body = _body(golden_service, 0)["camera"]
    assert camera_from_json(body).width == body["width"]
    cases = [("fx", None, "camera.fx"), ("rotation", [[1, 0], [0, 1]], "camera.rotation"),
             ("translation", "x", "camera.translation"), ("width", 64.5, "camera.width"),
             ("cy", float("nan"), "camera.cy"), ("rotation", (2.0 * np.eye(3)).tolist(), "camera")]
    for key, val, field in cases:
        b = dict(body)
        if val is None:
            del b[key]
        else:
            b[key] = val
        with pytest.raises(BadRequest) as e:
            camera_from_json(b)
        assert e.value.field == field, (key, e.value.field)
    with pytest.raises(BadRequest):
        camera_from_json([1, 2])


def test_request_guards(service, golden_service):
    from paper_2404_01133_b200.service import BadRequest, Oversized
    with pytest.raises(BadRequest):
        service.render("not a dict")
    body = _body(golden_service, 0)
    body["camera"]["width"] = 4096
    with pytest.raises(Oversized):
        service.render(body)
    body = _body(golden_service, 0)
    body["lod"] = {"intervals": [[0, 250], [200, 400], [400, None]]}
    with pytest.raises(BadRequest) as e:
        service.render(body)
    assert e.value.field == "lod.intervals"


def test_update_lod(service):
    from paper_2404_01133_b200.service import BadRequest
    before = service.snapshot()
    try:
        ack = service.update_lod({"intervals": [[0, 150], [150, 300], [300, None]]})
        assert ack == {"ok": True, "intervals": [[0.0, 150.0], [150.0, 300.0], [300.0, None]],
                       "enabled": True}
        assert service.scene_info()["intervals"][0] == [0.0, 150.0]
        for bad in ([[0, 100], [100, None]], [[1, 5], [5, 10], [10, None]], [[0, 5], [5, 10], [10, 20]],
                    [[0, 5], [4, 10], [10, None]], "x"):
            with pytest.raises(BadRequest):
                service.update_lod({"intervals": bad})
        assert service.update_lod({"enabled": False})["enabled"] is False
    finally:
        service.update_lod({"intervals": [[a, b if math.isfinite(b) else None] for a, b in before[0]],
                            "enabled": before[1]})
    assert service.snapshot() == before


@pytest.mark.gpu
def test_frames_match_reference(service, golden_service):
    from PIL import Image as PilImage
    g = golden_service
    assert service.last_stats() is None or isinstance(service.last_stats(), dict)
    for k in range(int(g["n"])):
        png, stats = service.render(_body(g, k))
        px = np.asarray(PilImage.open(io.BytesIO(png)).convert("RGB"))
        want = g[f"req{k}/pixels"]
        assert px.shape == want.shape
        diff = np.abs(px.astype(np.int16) - want.astype(np.int16))
        # images agree to ~1e-6 before quantisation: a channel may round the
        # other way only when 255 x sits on a .5 boundary
        assert diff.max() <= 1 and (diff > 0).mean() <= 1e-3, (k, diff.max(), (diff > 0).sum())
        ref = json.loads(str(g[f"req{k}/stats"]))
        got = {key: v for key, v in stats.items() if key not in ("render_ms", "fps_estimate")}
        assert got == ref, k
        assert stats["render_ms"] > 0 and stats["fps_estimate"] == pytest.approx(1000.0 / stats["render_ms"])
        assert service.last_stats() == stats
    # identical requests, identical bytes; overrides do not persist
    a, _ = service.render(_body(g, 2))
    b, _ = service.render(_body(g, 2))
    assert a == b
    assert service.snapshot()[0] == service.scene.distance_intervals


def test_camera_center_matches_reference_bits():
    """CameraView.camera_center equals the reference's (pinned-BLAS) -R^T t
    bit for bit for every camera stored in the golden fixtures."""
    import glob
    from paper_2404_01133_b200.core import CameraView
    n = 0
    for f in glob.glob(str(GOLDEN / "*.npz")):
        z = np.load(f)
        for k in z.files:
            if k.endswith("/center"):
                p = k[:-len("/center")]
                fx, fy, cx, cy = (float(v) for v in z[p + "/intr"])
                w, h = (int(v) for v in z[p + "/size"])
                cam = CameraView(w, h, fx, fy, cx, cy, z[p + "/R"], z[p + "/t"])
                assert np.array_equal(cam.camera_center, z[k]), (f, p)
                n += 1
    assert n > 50

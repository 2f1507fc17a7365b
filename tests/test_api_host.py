"""Host-side API semantics (validation, error mapping) -- CPU only."""

import math

import numpy as np
import pytest

import paper_2404_01133_b200 as cs
from paper_2404_01133_b200 import _lib
from paper_2404_01133_b200.core import CameraView, Gaussian, GaussianCloud, Image


def test_settings_validation():
    # render.py:46-59, test_render.py:48-62
    for kw in (dict(tile_size=4), dict(alpha_floor=0.0), dict(transmittance_floor=1.0),
               dict(background=(0.0, 0.0)), dict(background=(0.0, 0.0, 1.5)), dict(near_plane=0.0),
               dict(sh_degree=4)):
        with pytest.raises(ValueError):
            cs.RenderSettings(**kw)
    s = cs.RenderSettings()
    assert s.support_sigmas == pytest.approx(math.sqrt(2.0 * math.log(255.0)))
    assert cs.RenderSettings(alpha_floor=0.1).support_sigmas < s.support_sigmas


def test_cloud_validation():
    good = dict(positions=np.zeros((2, 3)), opacities=[0.5, 0.5], scales=np.ones((2, 3)),
                rotations=np.tile([1.0, 0, 0, 0], (2, 1)), sh=np.zeros((2, 3, 16)))
    c = GaussianCloud(**good)
    assert c.count == 2 and c.sh_degree == 3
    assert not c.positions.flags.writeable
    for k, v in (("opacities", [1.5, 0.5]), ("scales", -np.ones((2, 3))),
                 ("rotations", np.tile([2.0, 0, 0, 0], (2, 1))), ("sh", np.zeros((2, 3, 5)))):
        with pytest.raises(ValueError):
            GaussianCloud(**{**good, k: v})
    cat = GaussianCloud.concat([c, c.with_sh_degree(1)])
    assert cat.count == 4 and cat.sh.shape == (4, 3, 16)
    assert GaussianCloud.empty().count == 0


def test_camera_and_image_validation():
    cam = CameraView(64, 48, 55.0, 55.0, 32.0, 24.0, np.eye(3), np.array([1.0, 2.0, 3.0]))
    np.testing.assert_array_equal(cam.camera_center, [-1.0, -2.0, -3.0])
    with pytest.raises(ValueError):
        CameraView(64, 48, 55.0, 55.0, 32.0, 24.0, 2 * np.eye(3), np.zeros(3))
    with pytest.raises(ValueError):
        CameraView(0, 48, 55.0, 55.0, 32.0, 24.0, np.eye(3), np.zeros(3))
    with pytest.raises(ValueError):
        Image(np.full((2, 2, 3), 1.5))
    with pytest.raises(ValueError):
        Gaussian(np.zeros(3), 0.5, np.ones(3), np.array([1.0, 1.0, 0, 0]), np.zeros((3, 16)))


def test_lodscene_validation():
    c = GaussianCloud.empty()
    with pytest.raises(ValueError):
        cs.LodScene(levels=(), bounds_min=np.zeros((0, 3)), bounds_max=np.zeros((0, 3)),
                    distance_intervals=(), sh_degrees=(), n_mad=4.0, full=c)
    with pytest.raises(ValueError):
        cs.LodScene(levels=((c,), (c,)), bounds_min=np.zeros((1, 3)), bounds_max=np.zeros((1, 3)),
                    distance_intervals=((0, 1),), sh_degrees=(1, 2), n_mad=4.0, full=c)
    s = cs.LodScene(levels=((c,), (c,)), bounds_min=np.zeros((1, 3)), bounds_max=np.ones((1, 3)),
                    distance_intervals=((0, 1), (1, math.inf)), sh_degrees=(1, 2), n_mad=4.0, full=c)
    assert s.n_levels == 2 and s.finest == 1 and not s.occupied(0)


def test_error_mapping():
    with pytest.raises(ValueError):
        _lib.check(_lib.CS_EINVAL)
    with pytest.raises(ValueError):
        _lib.check(_lib.CS_ERANGE)
    with pytest.raises(MemoryError):
        _lib.check(_lib.CS_ENOMEM)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.CS_ECUDA)


def test_struct_layouts_match_header():
    import ctypes
    assert ctypes.sizeof(_lib.CsCamera) == 8 * 19 + 8
    assert ctypes.sizeof(_lib.CsCloud) == 4 * 8 + 8 + 16
    assert ctypes.sizeof(_lib.CsFrameStats) == 5 * 8 + 8 + 8 * 8
    assert ctypes.sizeof(_lib.CsDecision) == 5 * 8 + 8

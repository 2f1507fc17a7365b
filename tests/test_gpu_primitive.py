"""render.project_gaussian (render.py:191-214)
against the reference's own outputs (tests/golden/primitive.npz, made by
tests/golden/make_golden_primitive.py running the reference): 192 Gaussians
under 12 cameras, SH degrees 0-3, 33 of them culled (None).  Geometry
(mean2d, cov2d, depth, opacity, support radius) bit-exact; colour (float64 SH
on the host, core.sh_to_colors) within 1e-12."""

from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden" / "primitive.npz"


def _camera(row):
    from paper_2404_01133_b200.core import CameraView
    return CameraView(width=int(row[0]), height=int(row[1]), fx=row[2], fy=row[3], cx=row[4], cy=row[5],
                      rotation_w2c=row[6:15].reshape(3, 3), translation_w2c=row[15:18])


def test_project_gaussian_matches_reference():
    from paper_2404_01133_b200.render import RenderSettings, project_gaussian
    z = np.load(GOLDEN)
    n = len(z["culled"])
    assert n == 192 and int(z["culled"].sum()) == 33
    for i in range(n):
        g = SimpleNamespace(position=z["pos"][i], opacity=float(z["op"][i]), scale=z["scale"][i],
                            rotation=z["rot"][i], sh=z["sh"][i])
        p = project_gaussian(g, _camera(z["cam"][i]), RenderSettings(sh_degree=int(z["degree"][i])),
                             source_index=int(z["source_index"][i]))
        if z["culled"][i]:
            assert p is None, i
            continue
        assert p is not None, i
        assert np.array_equal(p.mean2d, z["mean2d"][i]), i
        assert np.array_equal(p.cov2d, z["cov2d"][i]), i
        assert p.depth == z["depth"][i] and p.opacity == z["opacity"][i], i
        assert p.radius == z["radius"][i], i
        assert p.source_index == int(z["source_index"][i])
        assert np.abs(np.asarray(p.color) - z["color"][i]).max() <= 1e-12, i

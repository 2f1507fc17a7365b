"""Golden vectors for render.project_gaussian (render.py:191-214), produced by
running the REFERENCE itself (this container only: /root/reference is absent
on the GPU box):

    python tests/golden/make_golden_primitive.py   -> tests/golden/primitive.npz

Seeded Gaussians from the reference's own cloud_in_view (tests/conftest.py:
37-54: some behind the camera or off-image, so some project to None) under
random_camera / identity_camera, SH degrees 0-3; per case the SplatPrimitive
fields or a culled flag.  OPENBLAS_CORETYPE=Sandybridge as make_golden.py.
"""

import os
import sys

if os.environ.get("OPENBLAS_CORETYPE") != "Sandybridge":
    os.environ["OPENBLAS_CORETYPE"] = "Sandybridge"
    os.execv(sys.executable, [sys.executable] + sys.argv)

from pathlib import Path  # noqa: E402

import numpy as np  # noqa: E402

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

from citysplat.core import Gaussian  # noqa: E402
from citysplat.render import RenderSettings, project_gaussian  # noqa: E402
from conftest import cloud_in_view, identity_camera, random_camera  # noqa: E402


def main():
    rng = np.random.default_rng(2404)
    out = {k: [] for k in ("cam", "pos", "op", "scale", "rot", "sh", "degree", "culled", "mean2d",
                           "cov2d", "depth", "color", "opacity", "radius", "source_index")}
    n = 0
    for c in range(12):
        cam = identity_camera() if c == 0 else random_camera(rng)
        degree = c % 4
        cloud = cloud_in_view(rng, cam, 16)
        st = RenderSettings(sh_degree=degree)
        for i in range(len(cloud)):
            g = Gaussian(position=cloud.positions[i], opacity=float(cloud.opacities[i]),
                         scale=cloud.scales[i], rotation=cloud.rotations[i], sh=cloud.sh[i])
            p = project_gaussian(g, cam, st, source_index=n)
            out["cam"].append(np.concatenate([[cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy],
                                              cam.rotation_w2c.ravel(), cam.translation_w2c]))
            out["pos"].append(g.position); out["op"].append(g.opacity); out["scale"].append(g.scale)
            out["rot"].append(g.rotation); out["sh"].append(np.asarray(g.sh, dtype=np.float64))
            out["degree"].append(degree); out["source_index"].append(n)
            out["culled"].append(p is None)
            out["mean2d"].append(np.zeros(2) if p is None else p.mean2d)
            out["cov2d"].append(np.zeros((2, 2)) if p is None else p.cov2d)
            out["depth"].append(0.0 if p is None else p.depth)
            out["color"].append(np.zeros(3) if p is None else p.color)
            out["opacity"].append(0.0 if p is None else p.opacity)
            out["radius"].append(0.0 if p is None else p.radius)
            n += 1
    arrs = {k: np.asarray(v) for k, v in out.items()}
    dst = Path(__file__).resolve().parent / "primitive.npz"
    np.savez_compressed(dst, **arrs)
    print(dst, n, "cases,", int(arrs["culled"].sum()), "culled")


if __name__ == "__main__":
    main()

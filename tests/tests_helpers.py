"""Small seeded scenes for gradient tests (cloud_in_view-style, tests/conftest.py:37-54
of the reference)."""

from types import SimpleNamespace

import numpy as np


def random_unit_quats(rng, n):
    q = rng.normal(size=(n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def small_scene(seed, k=16, width=32, height=24):
    rng = np.random.default_rng(seed)
    f = 0.9 * width
    cam = SimpleNamespace(rotation_w2c=np.eye(3), translation_w2c=np.zeros(3), camera_center=np.zeros(3),
                          fx=f, fy=f, cx=width / 2.0 + 0.3, cy=height / 2.0 - 0.2, width=width, height=height)
    z = rng.uniform(2.0, 8.0, k)
    u = rng.uniform(0.1 * width, 0.9 * width, k)
    v = rng.uniform(0.1 * height, 0.9 * height, k)
    pos = np.stack([(u - cam.cx) / cam.fx * z, (v - cam.cy) / cam.fy * z, z], axis=1)
    cloud = SimpleNamespace(positions=pos, opacities=rng.uniform(0.2, 0.9, k),
                            scales=rng.uniform(0.05, 0.4, (k, 3)), rotations=random_unit_quats(rng, k),
                            sh=rng.normal(0.0, 0.3, (k, 3, 16)), count=k)
    st = SimpleNamespace(background=(0.2, 0.3, 0.1), sh_degree=3, tile_size=16, alpha_floor=1.0 / 255.0,
                         transmittance_floor=1e-4, near_plane=0.2)
    return cloud, cam, st

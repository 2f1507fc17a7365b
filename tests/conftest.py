"""Shared fixtures: golden-vector loading and the gpu marker.

Tests marked ``gpu`` need a B200 (run with ``-m gpu``); everything else runs
on CPU.  The oracle (oracle/) is the parity checker only.
"""

import os
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


class Golden:
    """Lazy view of one golden .npz with '/'-separated keys."""

    def __init__(self, name):
        self.z = np.load(GOLDEN / name, allow_pickle=False)

    def __getitem__(self, k):
        return self.z[k]

    def has(self, k):
        return k in self.z.files

    def cases(self):
        return [str(c) for c in self.z["cases"]]

    def cloud(self, prefix):
        g = lambda k: self.z[f"{prefix}/{k}"]
        return SimpleNamespace(positions=g("positions"), opacities=g("opacities"),
                               scales=g("scales"), rotations=g("rotations"), sh=g("sh"),
                               count=int(g("positions").shape[0]))

    def camera(self, prefix):
        g = lambda k: self.z[f"{prefix}/{k}"]
        fx, fy, cx, cy = (float(v) for v in g("intr"))
        w, h = (int(v) for v in g("size"))
        return SimpleNamespace(rotation_w2c=g("R"), translation_w2c=g("t"), camera_center=g("center"),
                               fx=fx, fy=fy, cx=cx, cy=cy, width=w, height=h)

    def settings(self, prefix):
        g = lambda k: self.z[f"{prefix}/{k}"]
        return SimpleNamespace(background=tuple(float(v) for v in g("bg")),
                               sh_degree=int(g("sh_degree")), tile_size=int(g("tile_size")),
                               alpha_floor=float(g("alpha_floor")),
                               transmittance_floor=float(g("t_floor")), near_plane=float(g("near")))

    def lod(self):
        L, J = int(self.z["n_levels"]), int(self.z["n_blocks"])
        levels = tuple(tuple(self.cloud(f"level{l}/block{j}") for j in range(J)) for l in range(L))
        return SimpleNamespace(levels=levels, bounds_min=self.z["bounds_min"],
                               bounds_max=self.z["bounds_max"],
                               distance_intervals=tuple(map(tuple, self.z["intervals"])),
                               sh_degrees=tuple(int(d) for d in self.z["sh_degrees"]),
                               n_levels=L, n_blocks=J)


@pytest.fixture(scope="session")
def golden_render():
    return Golden("render.npz")


@pytest.fixture(scope="session")
def golden_city():
    return Golden("city.npz")


@pytest.fixture(scope="session")
def golden_fuse():
    return Golden("fuse.npz")


@pytest.fixture(scope="session")
def golden_lodgen():
    return Golden("lodgen.npz")


def lodgen_inputs(g):
    """(cloud, cameras, membership, n_blocks) of tests/golden/lodgen.npz."""
    k = int(g["positions"].shape[0])
    rng = np.random.default_rng(1)
    cloud = SimpleNamespace(positions=g["positions"], opacities=g["opacities"], scales=g["scales"],
                            rotations=g["rotations"],
                            sh=rng.normal(0.0, 0.2, (k, 3, 16)).astype(np.float32), count=k)
    cams = [g.camera(f"cam{i:02d}") for i in range(int(g["n_cams"]))]
    return cloud, cams, g["membership"], int(g["n_blocks"])


@pytest.fixture(scope="session")
def golden_assign():
    return Golden("assign.npz")


def assign_inputs(g):
    """(cloud, views, grid, settings) of tests/golden/assign.npz (duck-typed)."""
    cloud = SimpleNamespace(positions=g["positions"], opacities=g["opacities"], scales=g["scales"],
                            rotations=g["rotations"], sh=g["sh"], count=int(g["positions"].shape[0]))
    views = [g.camera(f"pose{i:02d}") for i in range(int(g["n_poses"]))]
    grid = SimpleNamespace(map=SimpleNamespace(p_min=g["p_min"], p_max=g["p_max"]),
                           dims=tuple(int(d) for d in g["dims"]), bounds_min=g["bounds_min"],
                           bounds_max=g["bounds_max"], membership=g["membership"], counts=g["counts"],
                           contracted=g["contracted"], n_blocks=int(g["bounds_min"].shape[0]))
    settings = SimpleNamespace(background=(0.0, 0.0, 0.0), sh_degree=3, tile_size=16,
                               alpha_floor=1.0 / 255.0, transmittance_floor=1e-4, near_plane=0.2)
    return cloud, views, grid, settings


@pytest.fixture(scope="session")
def golden_bundle():
    return Golden("bundle.npz")


@pytest.fixture(scope="session")
def golden_service():
    return Golden("service.npz")

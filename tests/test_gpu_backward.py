"""Backward (K10/K11) vs the float64 autograd oracle; training step sanity (needs a B200).

Tolerance (BASELINE.json north star): gradients within max-abs 1e-4 or
relative 1e-3 of the oracle, element-wise.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ABS, REL = 1e-4, 1e-3


def _q32(cloud):
    from types import SimpleNamespace
    f = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)
    return SimpleNamespace(positions=f(cloud.positions), scales=f(cloud.scales), rotations=f(cloud.rotations),
                           opacities=f(cloud.opacities), sh=f(cloud.sh), count=cloud.count)


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_backward_matches_oracle(seed):
    from oracle import grad_oracle as G
    from paper_2404_01133_b200.train import rasterize_train
    from tests_helpers import small_scene
    cloud, cam, st = small_scene(seed, k=24)
    cloud = _q32(cloud)
    rng = np.random.default_rng(7 + seed)
    dl = rng.normal(size=(cam.height, cam.width, 3))
    ref_img, ref_grads = G.gradients(cloud, cam, st, dl)
    t = lambda a: torch.tensor(np.asarray(a), dtype=torch.float32, device="cuda", requires_grad=True)
    params = [t(cloud.positions), t(cloud.scales), t(cloud.rotations), t(cloud.opacities), t(cloud.sh)]
    img = rasterize_train(*params, cam, st)
    assert np.abs(img.detach().cpu().numpy() - ref_img).max() <= 1e-4
    (img * torch.tensor(dl, dtype=torch.float32, device="cuda")).sum().backward()
    for name, p, ref in zip(("positions", "scales", "rotations", "opacities", "sh"), params, ref_grads):
        got = p.grad.cpu().numpy().astype(np.float64)
        err = np.abs(got - ref)
        bad = err > np.maximum(ABS, REL * np.abs(ref))
        assert not bad.any(), (name, float(err.max()), float(np.abs(ref).max()), int(bad.sum()))


def test_training_step_reduces_loss():
    from paper_2404_01133_b200.render import RenderSettings, render
    from paper_2404_01133_b200.synth import city_cameras, generate_city
    from paper_2404_01133_b200.train import BlockTrainer
    c = generate_city(seed=4, extent=40.0, n_buildings=6, n_gaussians=20_000)
    cams = city_cameras(8, 40.0, 160, 120, seed=4)
    gt = [render(c, cam).clone() for cam in cams]
    rng = np.random.default_rng(0)
    dev = torch.device("cuda")
    T = lambda a: torch.tensor(np.asarray(a), dtype=torch.float32, device=dev)
    pos = T(c.positions + rng.normal(0, 0.05, c.positions.shape))
    tr = BlockTrainer(pos, T(c.scales), T(c.rotations), T(c.opacities), T(c.sh), lr=1e-3)
    first = [float(tr.step(cam, g)) for cam, g in zip(cams, gt)]
    for _ in range(20):
        for cam, g in zip(cams, gt):
            tr.step(cam, g)
    last = [float(tr.step(cam, g)) for cam, g in zip(cams, gt)]
    assert np.mean(last) < 0.8 * np.mean(first), (np.mean(first), np.mean(last))

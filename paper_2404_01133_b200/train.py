"""Per-block training on the B200 (the paper's divide-and-conquer fine-tuning,
PAPER.md:52).

* ``RasterizeFn`` -- torch.autograd.Function around the C ABI: forward =
  cs_render(KEEP_STATE) of one cloud, backward = cs_render_backward
  (K10 blend backward + K11 projection backward).  Gradients are w.r.t. the
  *activated* parameters the renderer consumes (position, scale, raw
  quaternion, opacity in [0, 1], SH).
* ``BlockTrainer`` -- raw parameters with the checkpoint activations of the
  reference's PLY convention (ply.py:108-123: sigmoid opacity, exp scale,
  normalised quaternion), loss = (1 - lambda) L1 + lambda (1 - SSIM) with
  lambda = 0.2 and the valid-region 11x11 Gaussian-window SSIM (sigma 1.5) of
  metrics.py:70-125, Adam with the manifest LR multipliers (0.4 position,
  0.8 scale; partition.py:45-50).
* Multi-GPU: blocks are independent units (no gradient exchange); ranks take
  blocks by LPT on block sizes; after training the fused cloud is gathered with
  fusion.fuse_all_gather.
"""

from __future__ import annotations

import ctypes
import math
from typing import List, Sequence

import numpy as np
import torch
import torch.nn.functional as F

from . import _lib, device
from ._lib import CsGrads, CsSource, check

LOSS_LAMBDA = 0.2          # metrics.py:121-125 / config.py:106
POSITION_LR_SCALE = 0.4    # partition.py:47
SCALE_LR_SCALE = 0.8       # partition.py:48


class RasterizeFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, positions, scales, rotations, opacities, sh, cam, settings):
        dc = device.DeviceCloud.from_torch(positions.detach(), opacities.detach(), scales.detach(),
                                           rotations.detach(), sh.detach())
        dev = positions.device
        H, W = int(cam.height), int(cam.width)
        out = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
        src = CsSource()
        src.kind = _lib.CS_SRC_CLOUD
        src.force_level = -1
        src.cloud = dc.desc()
        ccam = device.camera_struct(cam)
        cset = device.settings_struct(settings)
        h = device.context(dev.index)  # backward may run on autograd's device thread: reuse h
        check(_lib.load().cs_render(h, ctypes.byref(src), ctypes.byref(ccam),
                                    ctypes.byref(cset), out.data_ptr(), _lib.CS_RENDER_KEEP_STATE, None,
                                    device.stream_handle(dev)), "cs_render")
        ctx.keep = (dc, src, ccam, cset, h)
        ctx.sh_shape = sh.shape
        return out

    @staticmethod
    def backward(ctx, grad_out):
        dc, src, ccam, cset, h = ctx.keep
        dev = grad_out.device
        k = dc.count
        g = grad_out.contiguous().float()
        gp = torch.empty((k, 3), dtype=torch.float32, device=dev)
        gs = torch.empty((k, 3), dtype=torch.float32, device=dev)
        gq = torch.empty((k, 4), dtype=torch.float32, device=dev)
        go = torch.empty((k,), dtype=torch.float32, device=dev)
        gsh = torch.empty(ctx.sh_shape, dtype=torch.float32, device=dev)
        grads = CsGrads(gp.data_ptr(), gs.data_ptr(), gq.data_ptr(), go.data_ptr(), gsh.data_ptr())
        check(_lib.load().cs_render_backward(h, ctypes.byref(src), ctypes.byref(ccam),
                                             ctypes.byref(cset), g.data_ptr(), ctypes.byref(grads),
                                             device.stream_handle(dev)), "cs_render_backward")
        return gp, gs, gq, go, gsh, None, None


def rasterize_train(positions, scales, rotations, opacities, sh, cam, settings):
    """Differentiable render of one cloud -> (H, W, 3) float32 image in [0, 1]."""
    return RasterizeFn.apply(positions, scales, rotations, opacities, sh, cam, settings)


def _gauss_window(size=11, sigma=1.5, device=None):
    x = torch.arange(size, dtype=torch.float32, device=device) - (size - 1) / 2.0
    g = torch.exp(-(x * x) / (2 * sigma * sigma))
    return g / g.sum()


def ssim(img: torch.Tensor, ref: torch.Tensor) -> torch.Tensor:
    """Mean SSIM over the valid region of an 11x11 Gaussian window (sigma 1.5),
    per channel, constants C1 = 0.01^2, C2 = 0.03^2 (metrics.py:70-95)."""
    x = img.permute(2, 0, 1)[:, None]
    y = ref.permute(2, 0, 1)[:, None]
    g = _gauss_window(device=img.device)
    kx = g.view(1, 1, 1, -1)
    ky = g.view(1, 1, -1, 1)
    blur = lambda t: F.conv2d(F.conv2d(t, kx), ky)
    mx, my = blur(x), blur(y)
    sxx = blur(x * x) - mx * mx
    syy = blur(y * y) - my * my
    sxy = blur(x * y) - mx * my
    c1, c2 = 0.01 ** 2, 0.03 ** 2
    s = ((2 * mx * my + c1) * (2 * sxy + c2)) / ((mx * mx + my * my + c1) * (sxx + syy + c2))
    return s.mean()


def training_loss(img: torch.Tensor, ref: torch.Tensor, lam: float = LOSS_LAMBDA) -> torch.Tensor:
    """(1 - lambda) L1 + lambda (1 - SSIM) (metrics.py:121-125)."""
    return (1.0 - lam) * (img - ref).abs().mean() + lam * (1.0 - ssim(img, ref))


class BlockTrainer:
    """Adam on the raw parameters of one block (PLY activations, ply.py:108-123)."""

    def __init__(self, positions, scales, rotations, opacities, sh, lr=1.6e-4, settings=None):
        from .render import RenderSettings
        eps = 1e-6
        self.settings = settings or RenderSettings()
        f = lambda t: torch.nn.Parameter(t.detach().float().contiguous().clone())
        self.pos = f(positions)
        self.log_scale = f(torch.log(scales.clamp_min(1e-8)))
        self.quat = f(rotations)
        o = opacities.clamp(eps, 1 - eps)
        self.logit_op = f(torch.log(o / (1 - o)))
        self.sh = f(sh)
        self.opt = torch.optim.Adam([
            {"params": [self.pos], "lr": lr * POSITION_LR_SCALE},
            {"params": [self.log_scale], "lr": 5e-3 * SCALE_LR_SCALE},
            {"params": [self.quat], "lr": 1e-3},
            {"params": [self.logit_op], "lr": 5e-2},
            {"params": [self.sh], "lr": 2.5e-3},
        ], eps=1e-15)

    def activated(self):
        q = self.quat / self.quat.norm(dim=1, keepdim=True)
        return (self.pos, torch.exp(self.log_scale), q, torch.sigmoid(self.logit_op), self.sh)

    def step(self, cam, target: torch.Tensor) -> torch.Tensor:
        self.opt.zero_grad(set_to_none=True)
        img = rasterize_train(*self.activated(), cam, self.settings)
        loss = training_loss(img, target)
        loss.backward()
        self.opt.step()
        return loss.detach()


def lpt_assign(sizes: Sequence[int], n_ranks: int) -> List[int]:
    """Longest-processing-time block -> rank assignment."""
    owner = [0] * len(sizes)
    load = [0] * n_ranks
    for j in sorted(range(len(sizes)), key=lambda j: (-sizes[j], j)):
        r = min(range(n_ranks), key=lambda r: (load[r], r))
        owner[j] = r
        load[r] += sizes[j]
    return owner

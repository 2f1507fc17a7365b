"""Drop-in for citysplat.metrics (metrics.py:1-140) on the device.

* ``ssim`` / ``l_ssim`` (metrics.py:70-101): K20 ``cs_ssim`` -- the reference's
  11x11 Gaussian window (sigma 1.5), valid region, C1 = 0.01^2, C2 = 0.03^2,
  float64 statistics from float32 pixels (the rendered images are float32);
  agrees with the reference's scipy SSIM to ~1e-8;
* ``psnr``, ``l1`` (metrics.py:104-118), ``training_loss`` (metrics.py:121-125),
  ``MetricReport`` / ``metric_report``: float64 reductions on the device.

Inputs: ``Image`` objects, host (H, W, 3) arrays or CUDA tensors; the
reference's errors (ValueError on a wrong shape, a size mismatch or images
smaller than 11x11).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import device
from .partition import _W2D, _ssim_into

__all__ = ["MetricReport", "ssim", "l_ssim", "psnr", "l1", "training_loss", "metric_report"]

_WINDOW = 11


@dataclass(frozen=True)
class MetricReport:
    """metrics.MetricReport: per-image quality summary."""

    ssim: float
    psnr: float
    l1: float
    loss: float


def _tensor(a) -> torch.Tensor:
    px = getattr(a, "pixels", a)
    t = px if isinstance(px, torch.Tensor) else torch.as_tensor(np.asarray(px, dtype=np.float64))
    if t.ndim != 3 or t.shape[2] != 3:
        raise ValueError(f"expected an (H, W, 3) image, got {tuple(t.shape)}")
    return t.to(device.default_device())


def _pair(a, b):
    ta, tb = _tensor(a), _tensor(b)
    if ta.shape != tb.shape:
        raise ValueError(f"image dimensions differ: {tuple(ta.shape)} vs {tuple(tb.shape)}")
    return ta, tb


def ssim(a, b) -> float:
    """metrics.ssim (metrics.py:70-96)."""
    ta, tb = _pair(a, b)
    if ta.shape[0] < _WINDOW or ta.shape[1] < _WINDOW:
        raise ValueError(f"images must be at least {_WINDOW}x{_WINDOW} for ssim")
    acc = torch.zeros(4, dtype=torch.float64, device=ta.device)
    _ssim_into(ta.to(torch.float32).contiguous(), tb.to(torch.float32).contiguous(), acc)
    return float(acc[3].item())


def l_ssim(a, b) -> float:
    """metrics.l_ssim: 1 - ssim."""
    return 1.0 - ssim(a, b)


def psnr(a, b) -> float:
    """metrics.psnr: 10 log10(1 / MSE); inf for identical images."""
    ta, tb = _pair(a, b)
    mse = float(((ta.double() - tb.double()) ** 2).mean().item())
    if mse == 0.0:
        return math.inf
    return 10.0 * math.log10(1.0 / mse)


def l1(a, b) -> float:
    """metrics.l1: mean absolute error."""
    ta, tb = _pair(a, b)
    return float((ta.double() - tb.double()).abs().mean().item())


def training_loss(render, gt, lam: float = 0.2) -> float:
    """metrics.training_loss: (1 - lam) * L1 + lam * (1 - SSIM)."""
    if not 0.0 <= lam <= 1.0:
        raise ValueError("lam must be in [0, 1]")
    return (1.0 - lam) * l1(render, gt) + lam * l_ssim(render, gt)


def metric_report(render, gt, lam: float = 0.2) -> MetricReport:
    """metrics.metric_report (metrics.py:128-132)."""
    s = ssim(render, gt)
    e1 = l1(render, gt)
    return MetricReport(ssim=s, psnr=psnr(render, gt), l1=e1, loss=(1.0 - lam) * e1 + lam * (1.0 - s))

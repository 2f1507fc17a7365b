"""metrics drop-in (ssim / l_ssim / psnr / l1 / training_loss / metric_report)
vs the oracle's restatement of metrics.py (scipy SSIM) on random images
(needs a B200): SSIM within 1e-7 (float32 pixels), the rest exact to 1e-12."""

import math

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_metrics_vs_oracle():
    from paper_2404_01133_b200 import metrics as M
    rng = np.random.default_rng(3)
    a = rng.uniform(0, 1, (67, 91, 3)).astype(np.float32).astype(np.float64)
    b = np.clip(a + rng.normal(0, 0.03, a.shape), 0, 1).astype(np.float32).astype(np.float64)
    assert abs(M.ssim(a, b) - O.ssim(a, b)) < 1e-7
    assert abs(M.l_ssim(a, b) - (1.0 - O.ssim(a, b))) < 1e-7
    assert abs(M.psnr(a, b) - 10.0 * math.log10(1.0 / np.mean((a - b) ** 2))) < 1e-9
    assert abs(M.l1(a, b) - np.mean(np.abs(a - b))) < 1e-12
    assert M.psnr(a, a) == math.inf
    lam = 0.2
    want = (1 - lam) * np.mean(np.abs(a - b)) + lam * (1 - O.ssim(a, b))
    assert abs(M.training_loss(a, b, lam) - want) < 1e-7
    r = M.metric_report(a, b)
    assert abs(r.loss - want) < 1e-7 and abs(r.ssim - O.ssim(a, b)) < 1e-7


def test_metrics_errors():
    from paper_2404_01133_b200 import metrics as M
    with pytest.raises(ValueError):
        M.ssim(np.zeros((10, 30, 3)), np.zeros((10, 30, 3)))
    with pytest.raises(ValueError):
        M.l1(np.zeros((12, 12, 3)), np.zeros((12, 13, 3)))
    with pytest.raises(ValueError):
        M.psnr(np.zeros((12, 12)), np.zeros((12, 12)))
    with pytest.raises(ValueError):
        M.training_loss(np.zeros((12, 12, 3)), np.zeros((12, 12, 3)), lam=1.5)

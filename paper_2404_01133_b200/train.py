"""Per-block training on the B200 (the paper's divide-and-conquer fine-tuning,
PAPER.md:52).

* ``RasterizeFn`` -- torch.autograd.Function around the C ABI: forward =
  cs_render_train of one cloud (a kept-state handle per forward, so several
  forwards -- a multi-view loss -- or other renders may run before the
  backward), backward = cs_render_backward on that handle (K10 blend backward
  + K11 projection backward); a forward whose pair buffer overflowed raises
  MemoryError in the backward instead of differentiating an incomplete frame.  Gradients are w.r.t. the
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


class TrainState:
    """A cs_render_train state handle (its frame workspace stays reserved for
    the backward until the handle is released or collected)."""

    def __init__(self, handle: ctypes.c_void_p):
        self.handle = handle

    def release(self):
        if self.handle is not None and self.handle.value:
            _lib.load().cs_state_release(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


_sized = {}  # device index -> (largest cloud, largest image) a training forward was sized for


def render_train(h, src, ccam, cset, out: torch.Tensor, count: int, dev) -> TrainState:
    """cs_render_train; a forward of a larger cloud or a larger image than any
    before on this device runs synchronously, so the pair buffers are sized by
    the frame itself (pairs grow with both).  A later asynchronous forward that
    still overflows (a much nearer view) fails loudly in its backward."""
    pixels = int(ccam.width) * int(ccam.height)
    k0, p0 = _sized.get(dev.index, (-1, -1))
    flags = 0 if (k0 >= count and p0 >= pixels) else _lib.CS_RENDER_SYNC
    st = ctypes.c_void_p()
    check(_lib.load().cs_render_train(h, ctypes.byref(src), ctypes.byref(ccam), ctypes.byref(cset),
                                      out.data_ptr(), flags, ctypes.byref(st), device.stream_handle(dev)),
          "cs_render_train")
    _sized[dev.index] = (max(k0, count), max(p0, pixels))
    return TrainState(st)


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
        state = render_train(h, src, ccam, cset, out, dc.count, dev)
        ctx.keep = (dc, state, h)
        ctx.sh_shape = sh.shape
        return out

    @staticmethod
    def backward(ctx, grad_out):
        dc, state, h = ctx.keep
        dev = grad_out.device
        k = dc.count
        g = grad_out.contiguous().float()
        gp = torch.empty((k, 3), dtype=torch.float32, device=dev)
        gs = torch.empty((k, 3), dtype=torch.float32, device=dev)
        gq = torch.empty((k, 4), dtype=torch.float32, device=dev)
        go = torch.empty((k,), dtype=torch.float32, device=dev)
        gsh = torch.empty(ctx.sh_shape, dtype=torch.float32, device=dev)
        grads = CsGrads(gp.data_ptr(), gs.data_ptr(), gq.data_ptr(), go.data_ptr(), gsh.data_ptr())
        check(_lib.load().cs_render_backward(h, state.handle, g.data_ptr(), ctypes.byref(grads),
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
        ], eps=1e-15, fused=self.pos.is_cuda)

    def activated(self):
        q = self.quat / self.quat.norm(dim=1, keepdim=True)
        return (self.pos, torch.exp(self.log_scale), q, torch.sigmoid(self.logit_op), self.sh)

    def step(self, cam, target: torch.Tensor, events=None) -> torch.Tensor:
        """One iteration; `events` (5 CUDA events) brackets forward, loss,
        backward and the optimizer step for per-phase timing."""
        rec = (lambda i: events[i].record()) if events is not None else (lambda i: None)
        self.opt.zero_grad(set_to_none=True)
        rec(0)
        img = rasterize_train(*self.activated(), cam, self.settings)
        rec(1)
        loss = training_loss(img, target)
        rec(2)
        loss.backward()
        rec(3)
        self.opt.step()
        rec(4)
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


class DeviceBlockTrainer:
    """The block iteration on the C ABI end to end (no autograd graph):

        cs_render_train -> cs_training_loss (K13) -> cs_render_backward
        (K10/K11) -> cs_block_adam (K14: activation chain + Adam + the
        activated quads of the next forward)

    Same loss, activations, learning rates and Adam semantics as
    ``BlockTrainer`` (its torch restatement, used as the reference in tests).
    Raw parameters: geom (K, 11) = [xyz, log scale, raw quaternion wxyz,
    logit opacity] and sh (K, 3C); the sh array doubles as the render's SH
    row table, so C must be 4 or 16 (3C a multiple of 4).
    """

    def __init__(self, positions, scales, rotations, opacities, sh, lr=1.6e-4, settings=None,
                 betas=(0.9, 0.999), eps=1e-15):
        from .render import RenderSettings
        self.settings = settings or RenderSettings()
        dev = positions.device
        k = int(positions.shape[0])
        C = int(sh.shape[2])
        if C not in (4, 16):
            raise ValueError("DeviceBlockTrainer needs 4 or 16 SH coefficients (row stride 3C % 4 == 0)")
        self.K, self.C, self.dev = k, C, dev
        f = lambda t: t.detach().to(device=dev, dtype=torch.float32)
        o = f(opacities).reshape(k).clamp(1e-6, 1 - 1e-6)
        self.geom = torch.cat([f(positions).reshape(k, 3), torch.log(f(scales).clamp_min(1e-8)).reshape(k, 3),
                               f(rotations).reshape(k, 4), torch.log(o / (1 - o)).reshape(k, 1)],
                              dim=1).contiguous()
        self.sh = f(sh).reshape(k, 3 * C).contiguous()
        self.geom_m = torch.zeros_like(self.geom)
        self.geom_v = torch.zeros_like(self.geom)
        self.sh_m = torch.zeros_like(self.sh)
        self.sh_v = torch.zeros_like(self.sh)
        self.quads = torch.empty((3, k, 4), dtype=torch.float32, device=dev)
        self.g_pos = torch.empty((k, 3), dtype=torch.float32, device=dev)
        self.g_scale = torch.empty((k, 3), dtype=torch.float32, device=dev)
        self.g_rot = torch.empty((k, 4), dtype=torch.float32, device=dev)
        self.g_op = torch.empty((k,), dtype=torch.float32, device=dev)
        self.g_sh = torch.empty((k, 3 * C), dtype=torch.float32, device=dev)
        self.loss = torch.zeros(1, dtype=torch.float64, device=dev)
        self.hp = _lib.CsAdamHparams(lr * POSITION_LR_SCALE, 5e-3 * SCALE_LR_SCALE, 1e-3, 5e-2, 2.5e-3,
                                     betas[0], betas[1], eps, 0, 0)
        self.grads = CsGrads(self.g_pos.data_ptr(), self.g_scale.data_ptr(), self.g_rot.data_ptr(),
                             self.g_op.data_ptr(), self.g_sh.data_ptr())
        self.src = CsSource()
        self.src.kind = _lib.CS_SRC_CLOUD
        self.src.force_level = -1
        self.src.cloud = _lib.CsCloud(self.quads[0].data_ptr(), self.quads[1].data_ptr(),
                                      self.quads[2].data_ptr(), self.sh.data_ptr(), k, C, 3 * C, 0, 0)
        self.cset = device.settings_struct(self.settings)
        self._bufs = {}
        self.lib = _lib.load()
        self.h = device.context(dev.index)
        check(self.lib.cs_block_activate(self.h, k, self.geom.data_ptr(), self.quads[0].data_ptr(),
                                         self.quads[1].data_ptr(), self.quads[2].data_ptr(),
                                         device.stream_handle(dev)), "cs_block_activate")

    @property
    def step_count(self) -> int:
        return int(self.hp.step)

    def activated(self):
        """(positions, scales, rotations, opacities, sh) as the renderer sees them."""
        q = self.quads
        return (q[0, :, :3], q[1, :, :3], q[2], q[0, :, 3], self.sh.reshape(self.K, 3, self.C))

    def _images(self, H: int, W: int):
        b = self._bufs.get((H, W))
        if b is None:
            b = self._bufs[(H, W)] = (torch.empty((H, W, 3), dtype=torch.float32, device=self.dev),
                                      torch.empty((H, W, 3), dtype=torch.float32, device=self.dev))
        return b

    def step(self, cam, target: torch.Tensor, events=None) -> torch.Tensor:
        rec = (lambda i: events[i].record()) if events is not None else (lambda i: None)
        lib, h = self.lib, self.h
        s = device.stream_handle(self.dev)
        H, W = int(cam.height), int(cam.width)
        img, dimg = self._images(H, W)
        ccam = device.camera_struct(cam)
        for attempt in range(2):
            rec(0)
            state = render_train(h, self.src, ccam, self.cset, img, self.K, self.dev)
            rec(1)
            check(lib.cs_training_loss(h, img.data_ptr(), target.data_ptr(), H, W, LOSS_LAMBDA,
                                       self.loss.data_ptr(), dimg.data_ptr(), s), "cs_training_loss")
            rec(2)
            try:
                check(lib.cs_render_backward(h, state.handle, dimg.data_ptr(), ctypes.byref(self.grads), s),
                      "cs_render_backward")
                break
            except MemoryError:
                # the forward overflowed its pair buffer (nothing was differentiated
                # and the buffers have grown): the step is repeated once
                if attempt:
                    raise
            finally:
                state.release()
        rec(3)
        self.hp.step += 1
        check(lib.cs_block_adam(h, self.K, self.C, self.geom.data_ptr(), self.geom_m.data_ptr(),
                                self.geom_v.data_ptr(), self.sh.data_ptr(), self.sh_m.data_ptr(),
                                self.sh_v.data_ptr(), ctypes.byref(self.grads), ctypes.byref(self.hp),
                                self.quads[0].data_ptr(), self.quads[1].data_ptr(), self.quads[2].data_ptr(),
                                s), "cs_block_adam")
        rec(4)
        return self.loss

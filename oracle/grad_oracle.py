"""Float64 autograd oracle for the backward pass (TEST INFRASTRUCTURE ONLY).

The reference has no backward, so gradient parity is anchored
on a restatement of the reference *forward* in float64 torch, differentiated
by autograd:

* projection: render.py:118-172 + core.py:67-172 (quat_to_rotmat polynomial,
  R diag(s^2) R^T, W Sigma W^T, J V J^T + 0.3 I, conic, SH colour with clip);
* blend: _kernels.py:17-76 over the depth-sorted splats, with the discrete
  per-pixel decisions (which fragments are accepted, where the pixel stops)
  taken from the float64 forward -- skipped and dropped fragments carry no
  gradient, alpha = min(0.99, o exp(power)) is clamped, the image is clipped
  to [0, 1] (render.py:273).

tests/test_grad_oracle.py checks this oracle's forward against the golden
vectors and its gradients against central finite differences of the C
oracle's rasterize (itself bit-pinned to the reference).  Only small scenes
(dense per-pixel x per-splat tensors).
"""

from __future__ import annotations

import numpy as np
import torch

from . import oracle as O

SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
SH_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
         0.5462742152960396)
SH_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
         -0.4570457994644658, 1.445305721320277, -0.5900435899266435)


def _basis(d, degree):
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    out = [torch.full_like(x, SH_C0)]
    if degree >= 1:
        out += [-SH_C1 * y, SH_C1 * z, -SH_C1 * x]
    if degree >= 2:
        xx, yy, zz, xy, yz, xz = x * x, y * y, z * z, x * y, y * z, x * z
        out += [SH_C2[0] * xy, SH_C2[1] * yz, SH_C2[2] * (2 * zz - xx - yy), SH_C2[3] * xz,
                SH_C2[4] * (xx - yy)]
        if degree >= 3:
            out += [SH_C3[0] * y * (3 * xx - yy), SH_C3[1] * xy * z, SH_C3[2] * y * (4 * zz - xx - yy),
                    SH_C3[3] * z * (2 * zz - 3 * xx - 3 * yy), SH_C3[4] * x * (4 * zz - xx - yy),
                    SH_C3[5] * z * (xx - yy), SH_C3[6] * x * (xx - 3 * yy)]
    return torch.stack(out, dim=1)


def project_torch(pos, scl, quat, opac, sh, cam, sh_degree, src):
    """Differentiable projection of the rows `src` (visible set, depth order)."""
    R = torch.tensor(np.asarray(cam.rotation_w2c, dtype=np.float64))
    T = torch.tensor(np.asarray(cam.translation_w2c, dtype=np.float64))
    C = torch.tensor(np.asarray(cam.camera_center, dtype=np.float64))
    p, s, q, o, f = pos[src], scl[src], quat[src], opac[src], sh[src]
    t = p @ R.T + T
    tx, ty, z = t[:, 0], t[:, 1], t[:, 2]
    mx = cam.fx * tx / z + cam.cx
    my = cam.fy * ty / z + cam.cy
    w, x, y, qz = q.unbind(1)
    r = torch.stack([1 - 2 * (y * y + qz * qz), 2 * (x * y - w * qz), 2 * (x * qz + w * y),
                     2 * (x * y + w * qz), 1 - 2 * (x * x + qz * qz), 2 * (y * qz - w * x),
                     2 * (x * qz - w * y), 2 * (y * qz + w * x), 1 - 2 * (x * x + y * y)], 1).view(-1, 3, 3)
    M = r * s[:, None, :]
    Sig = M @ M.transpose(1, 2)
    V = R @ Sig @ R.T
    zero = torch.zeros_like(z)
    J = torch.stack([torch.stack([cam.fx / z, zero, -cam.fx * tx / (z * z)], 1),
                     torch.stack([zero, cam.fy / z, -cam.fy * ty / (z * z)], 1)], 1)
    cov = J @ V @ J.transpose(1, 2)
    a = cov[:, 0, 0] + 0.3
    b = cov[:, 0, 1]
    c = cov[:, 1, 1] + 0.3
    det = a * c - b * b
    conic = torch.stack([c / det, -b / det, a / det], 1)
    width = f.shape[2]
    deg = min(sh_degree, {1: 0, 4: 1, 9: 2, 16: 3}[width])
    v = p - C
    d = v / torch.linalg.norm(v, dim=1, keepdim=True)
    Y = _basis(d, deg)
    n = Y.shape[1]
    col = torch.clamp(0.5 + torch.einsum("kcn,kn->kc", f[:, :, :n], Y), 0.0, 1.0)
    return torch.stack([mx, my], 1), conic, o, col


def blend_decisions(proj: dict, cam, settings):
    """Per (pixel, splat) accepted mask from the float64 forward (numpy; exactly
    the loop of _kernels.py:46-72 without tiling -- tiling never changes the
    accepted set because binning uses the alpha-floor support)."""
    H, W = int(cam.height), int(cam.width)
    m = proj["count"]
    acc = np.zeros((H * W, m), dtype=bool)
    means, conics, opac = proj["means"], proj["conics"], proj["opacities"]
    for py in range(H):
        for px in range(W):
            sx, sy = px + 0.5, py + 0.5
            T = 1.0
            for k in range(m):
                dx, dy = sx - means[k, 0], sy - means[k, 1]
                power = -0.5 * (conics[k, 0] * dx * dx + conics[k, 2] * dy * dy) - conics[k, 1] * dx * dy
                alpha = min(0.99, opac[k] * np.exp(power))
                if alpha < settings.alpha_floor:
                    continue
                nt = T * (1.0 - alpha)
                if nt < settings.transmittance_floor:
                    break
                acc[py * W + px, k] = True
                T = nt
    return acc


def render_torch(cloud, cam, settings, params=None):
    """(image, params) with image differentiable w.r.t. params =
    (positions, scales, rotations, opacities, sh) float64 leaf tensors."""
    if params is None:
        params = tuple(torch.tensor(np.asarray(a, dtype=np.float64), requires_grad=True)
                       for a in (cloud.positions, cloud.scales, cloud.rotations, cloud.opacities, cloud.sh))
    pos, scl, quat, opac, sh = params
    proj = O.project_cloud(cloud, cam, settings)
    src = torch.tensor(proj["source"], dtype=torch.long)
    accepted = torch.tensor(blend_decisions(proj, cam, settings))
    H, W = int(cam.height), int(cam.width)
    bg = torch.tensor(settings.background, dtype=torch.float64)
    if proj["count"] == 0:
        return bg.expand(H, W, 3).clone(), params
    mean, conic, o, col = project_torch(pos, scl, quat, opac, sh, cam, int(settings.sh_degree), src)
    ys, xs = torch.meshgrid(torch.arange(H, dtype=torch.float64), torch.arange(W, dtype=torch.float64),
                            indexing="ij")
    px = (xs.reshape(-1) + 0.5)[:, None]
    py = (ys.reshape(-1) + 0.5)[:, None]
    dx = px - mean[None, :, 0]
    dy = py - mean[None, :, 1]
    power = -0.5 * (conic[None, :, 0] * dx * dx + conic[None, :, 2] * dy * dy) - conic[None, :, 1] * dx * dy
    alpha = torch.clamp(o[None, :] * torch.exp(power), max=0.99)
    alpha = torch.where(accepted, alpha, torch.zeros_like(alpha))
    one_minus = 1.0 - alpha
    T = torch.cumprod(torch.cat([torch.ones_like(one_minus[:, :1]), one_minus], 1), 1)
    Tk, Tend = T[:, :-1], T[:, -1]
    img = (Tk * alpha) @ col + Tend[:, None] * bg[None, :]
    return torch.clamp(img, 0.0, 1.0).reshape(H, W, 3), params


def gradients(cloud, cam, settings, dl_dimg: np.ndarray):
    img, params = render_torch(cloud, cam, settings)
    (img * torch.tensor(dl_dimg, dtype=torch.float64)).sum().backward()
    return img.detach().numpy(), [p.grad.numpy() if p.grad is not None else np.zeros(p.shape)
                                  for p in params]


# ---------------------------------------------------------------------------
# Sparse form for training-scale scenes (thousands to tens of thousands of
# Gaussians, up to 1080p): the same float64 autograd restatement, but only the
# ACCEPTED fragments enter the graph.  The C oracle (bit-pinned to the
# reference) supplies the projection, the tile lists and every pixel's
# accepted fragments in blend order (oracle.blend_fragments); per chunk of
# pixels the transmittance is a cumulative product over a [pixels, max
# fragments] matrix of (1 - alpha) -- exactly the dense form above, whose
# non-accepted entries are 1 -- and the chunk's loss is back-propagated on its
# own (retaining only the shared projection graph), so memory is bounded by the
# chunk.


def gradients_sparse(cloud, cam, settings, dl_dimg: np.ndarray, chunk_pixels: int = 1 << 16,
                     nthreads: int = 0):
    """(image, [d positions, d scales, d rotations, d opacities, d sh]) of
    sum(image * dl_dimg), float64, for the rasterize of `cloud`."""
    params = tuple(torch.tensor(np.asarray(a, dtype=np.float64), requires_grad=True)
                   for a in (cloud.positions, cloud.scales, cloud.rotations, cloud.opacities, cloud.sh))
    pos, scl, quat, opac, sh = params
    H, W = int(cam.height), int(cam.width)
    proj = O.project_cloud(cloud, cam, settings, nthreads=nthreads)
    bg = torch.tensor(settings.background, dtype=torch.float64)
    dl = torch.tensor(np.asarray(dl_dimg, dtype=np.float64).reshape(H * W, 3))
    img = np.empty((H * W, 3))
    if proj["count"] == 0:
        img[:] = np.clip(np.asarray(settings.background, dtype=np.float64), 0.0, 1.0)
        return img.reshape(H, W, 3), [np.zeros(p.shape) for p in params]
    tid, toff, _, _ = O.bin_tiles(proj, cam, int(settings.tile_size))
    poff, psplat = O.blend_fragments(tid, toff, proj, cam, settings, nthreads=nthreads)
    src = torch.tensor(proj["source"], dtype=torch.long)
    mean, conic, o, col = project_torch(pos, scl, quat, opac, sh, cam, int(settings.sh_degree), src)
    # the shared projection graph: accumulate d(loss)/d(projected) over the
    # chunks, then one backward through the projection
    leaves = [t.detach().requires_grad_(True) for t in (mean, conic, o, col)]
    acc = [torch.zeros_like(t) for t in leaves]
    counts = np.diff(poff)
    for p0 in range(0, H * W, chunk_pixels):
        p1 = min(H * W, p0 + chunk_pixels)
        n = counts[p0:p1]
        f0, f1 = int(poff[p0]), int(poff[p1])
        fmax = int(n.max()) if n.size else 0
        pix = torch.tensor(np.repeat(np.arange(p1 - p0), n), dtype=torch.long)
        slot = torch.tensor(np.arange(f1 - f0) - np.repeat(poff[p0:p1] - f0, n), dtype=torch.long)
        spl = torch.tensor(psplat[f0:f1], dtype=torch.long)
        m_, c_, o_, col_ = leaves
        gpix = torch.arange(p0, p1, dtype=torch.long)
        px = (gpix % W).to(torch.float64) + 0.5
        py = (gpix // W).to(torch.float64) + 0.5
        dx = px[pix] - m_[spl, 0]
        dy = py[pix] - m_[spl, 1]
        power = -0.5 * (c_[spl, 0] * dx * dx + c_[spl, 2] * dy * dy) - c_[spl, 1] * dx * dy
        alpha = torch.clamp(o_[spl] * torch.exp(power), max=0.99)
        A = torch.ones((p1 - p0, fmax + 1), dtype=torch.float64)
        A = A.index_put((pix, slot + 1), 1.0 - alpha)
        T = torch.cumprod(A, dim=1)                 # T[:, k] = transmittance before slot k
        Tk = T[pix, slot]
        Tend = T[:, -1]
        rgb = torch.zeros((p1 - p0, 3), dtype=torch.float64).index_add(0, pix, (Tk * alpha)[:, None] * col_[spl])
        out = torch.clamp(rgb + Tend[:, None] * bg[None, :], 0.0, 1.0)
        img[p0:p1] = out.detach().numpy()
        loss = (out * dl[p0:p1]).sum()
        g = torch.autograd.grad(loss, leaves, allow_unused=True)
        for a, gi in zip(acc, g):
            if gi is not None:
                a += gi
    torch.autograd.backward([mean, conic, o, col], acc)
    return img.reshape(H, W, 3), [p.grad.numpy() if p.grad is not None else np.zeros(p.shape) for p in params]

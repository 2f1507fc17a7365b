// cs_train.cu -- K13/K14: the rest of a block-training iteration on the
// device, so one iteration is
//   cs_render(KEEP_STATE) -> cs_training_loss -> cs_render_backward -> cs_block_adam
// with no autograd graph and no host round trip.
//
// K13 training loss (metrics.py:70-125): (1 - lam) * L1 + lam * (1 - SSIM),
// SSIM = mean over channels of the mean over the valid region of the 11x11
// Gaussian-window (sigma 1.5) statistics, C1 = 0.01^2, C2 = 0.03^2.  Two
// tiled kernels:
//   k_ssim_stats: per valid window q the five separable sums (mu_x, mu_y,
//     E[xx], E[yy], E[xy]) -> S(q) (summed for the loss) and the partials
//     A = dS/dmu_x, B = dS/dE[xx], C = dS/dE[xy] (written as maps);
//   k_ssim_grad: dL/dx(p) = (1-lam)/(3HW) sign(x-y)
//                         - lam/(3 Nv) sum_k w(k) [A + 2 x(p) B + y(p) C](p - k)
//     (the adjoint correlation of the three maps), plus the L1 sum.
// Both stage an input tile with its 10-pixel halo in shared memory and run
// the 11-tap window as a horizontal then a vertical pass.
//
// K14 Adam + activations (ply.py:108-123 conventions, torch.optim.Adam
// semantics): per Gaussian the gradient w.r.t. the activated parameters
// (cs_render_backward) is chained through exp(scale), sigmoid(opacity) and
// the quaternion normalisation, Adam updates the raw parameters, and the
// activated 16-byte quads the next forward reads are written in the same
// pass.  SH coefficients are updated elementwise in place; the SH parameter
// array is itself the render's SH row table (3C floats per row).
#include <math.h>

#include <algorithm>

#include "cs_internal.cuh"

namespace cs {

constexpr int kWin = 11;
constexpr int kHalo = kWin - 1;
#ifndef CS_SSIM_TX
#define CS_SSIM_TX 16
#endif
#ifndef CS_SSIM_TY
#define CS_SSIM_TY 32
#endif
constexpr int kTX = CS_SSIM_TX, kTY = CS_SSIM_TY;  // output tile of both loss kernels
constexpr int kRX = kTX + kHalo, kRY = kTY + kHalo;  // 42 x 26 region
constexpr int kLossThreads = 256;
constexpr float kC1 = 0.01f * 0.01f, kC2 = 0.03f * 0.03f;

__constant__ float c_win[kWin];

struct LossDims {
  int H, W, Hv, Wv;
  float k_l1;    // (1 - lam) / (3 H W)
  float k_ssim;  // -lam / (3 Hv Wv)
};

// maps layout: [ch][3][Hv][Wv]  (A, B, C)
__global__ void __launch_bounds__(kLossThreads)
k_ssim_stats(const float* __restrict__ img, const float* __restrict__ ref, LossDims d,
             float* __restrict__ maps, double* __restrict__ acc) {
  __shared__ float sx[kRY][kRX * 3];
  __shared__ float sy[kRY][kRX * 3];
  __shared__ float hs[5][kRY][kTX];
  __shared__ double s_red[kLossThreads / 32];
  const int ox = blockIdx.x * kTX, oy = blockIdx.y * kTY;
  // stage the 3-channel region (rows contiguous in HWC: coalesced)
  for (int i = threadIdx.x; i < kRY * kRX * 3; i += kLossThreads) {
    const int r = i / (kRX * 3), cc = i - r * (kRX * 3);
    const int gy = oy + r, gx = ox + cc / 3;
    float vx = 0.f, vy = 0.f;
    if (gy < d.H && gx < d.W) {
      const size_t o = ((size_t)gy * d.W + gx) * 3 + (cc % 3);
      vx = __ldg(img + o);
      vy = __ldg(ref + o);
    }
    sx[r][cc] = vx;
    sy[r][cc] = vy;
  }
  __syncthreads();
  double ssum = 0.0;
  for (int ch = 0; ch < 3; ++ch) {
    // horizontal pass: 26 rows x 32 output columns
    for (int i = threadIdx.x; i < kRY * kTX; i += kLossThreads) {
      const int r = i / kTX, c = i - r * kTX;
      float mx = 0.f, my = 0.f, xx = 0.f, yy = 0.f, xy = 0.f;
#pragma unroll
      for (int k = 0; k < kWin; ++k) {
        const float w = c_win[k];
        const float a = sx[r][(c + k) * 3 + ch], b = sy[r][(c + k) * 3 + ch];
        mx += w * a; my += w * b;
        xx += w * a * a; yy += w * b * b; xy += w * a * b;
      }
      hs[0][r][c] = mx; hs[1][r][c] = my; hs[2][r][c] = xx; hs[3][r][c] = yy; hs[4][r][c] = xy;
    }
    __syncthreads();
    // vertical pass + per-window SSIM and partials
    for (int i = threadIdx.x; i < kTY * kTX; i += kLossThreads) {
      const int r = i / kTX, c = i - r * kTX;
      const int qy = oy + r, qx = ox + c;
      if (qy >= d.Hv || qx >= d.Wv) continue;
      float mx = 0.f, my = 0.f, xx = 0.f, yy = 0.f, xy = 0.f;
#pragma unroll
      for (int k = 0; k < kWin; ++k) {
        const float w = c_win[k];
        mx += w * hs[0][r + k][c]; my += w * hs[1][r + k][c];
        xx += w * hs[2][r + k][c]; yy += w * hs[3][r + k][c]; xy += w * hs[4][r + k][c];
      }
      const float vx = xx - mx * mx, vy = yy - my * my, cv = xy - mx * my;
      const float n1 = 2.f * mx * my + kC1, n2 = 2.f * cv + kC2;
      const float d1 = mx * mx + my * my + kC1, d2 = vx + vy + kC2;
      const float den = d1 * d2;
      const float S = n1 * n2 / den;
      ssum += (double)S;
      // dS/dmu_x with E[xx], E[xy] held fixed (var_x, cov depend on mu_x)
      const float A = (2.f * my * n2 - 2.f * my * n1) / den - S * (2.f * mx / d1 - 2.f * mx / d2);
      const float B = -S / d2;            // dS/dE[xx]
      const float C = 2.f * n1 / den;     // dS/dE[xy]
      const size_t plane = (size_t)d.Hv * d.Wv;
      const size_t o = (size_t)qy * d.Wv + qx;
      float* m = maps + (size_t)ch * 3 * plane;
      m[o] = A;
      m[plane + o] = B;
      m[2 * plane + o] = C;
    }
    __syncthreads();
  }
  ssum = warp_sum(ssum);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = ssum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kLossThreads / 32; ++w) t += s_red[w];
    atomicAdd(acc + 1, t);
  }
}

__global__ void __launch_bounds__(kLossThreads)
k_ssim_grad(const float* __restrict__ img, const float* __restrict__ ref,
            const float* __restrict__ maps, LossDims d, float* __restrict__ grad,
            double* __restrict__ acc) {
  __shared__ float sm[3][kRY][kRX];     // A, B, C region of one channel
  __shared__ float hs[3][kRY][kTX];
  __shared__ float so[kTY][kTX * 3];    // gradient tile, HWC
  __shared__ double s_red[kLossThreads / 32];
  const int ox = blockIdx.x * kTX, oy = blockIdx.y * kTY;
  const size_t plane = (size_t)d.Hv * d.Wv;
  double l1 = 0.0;
  for (int ch = 0; ch < 3; ++ch) {
    const float* m = maps + (size_t)ch * 3 * plane;
    // windows q = p - k, k in [0, 10]: rows oy-10 .. oy+15, cols ox-10 .. ox+31
    for (int i = threadIdx.x; i < 3 * kRY * kRX; i += kLossThreads) {
      const int mi = i / (kRY * kRX), rem = i - mi * (kRY * kRX);
      const int r = rem / kRX, c = rem - r * kRX;
      const int qy = oy - kHalo + r, qx = ox - kHalo + c;
      float v = 0.f;
      if (qy >= 0 && qy < d.Hv && qx >= 0 && qx < d.Wv) v = __ldg(m + mi * plane + (size_t)qy * d.Wv + qx);
      sm[mi][r][c] = v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 3 * kRY * kTX; i += kLossThreads) {
      const int mi = i / (kRY * kTX), rem = i - mi * (kRY * kTX);
      const int r = rem / kTX, c = rem - r * kTX;
      float s = 0.f;
#pragma unroll
      for (int k = 0; k < kWin; ++k) s += c_win[k] * sm[mi][r][c + kHalo - k];
      hs[mi][r][c] = s;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kTY * kTX; i += kLossThreads) {
      const int r = i / kTX, c = i - r * kTX;
      const int py = oy + r, px = ox + c;
      if (py >= d.H || px >= d.W) continue;
      float a = 0.f, b = 0.f, cc = 0.f;
#pragma unroll
      for (int k = 0; k < kWin; ++k) {
        const float w = c_win[k];
        a += w * hs[0][r + kHalo - k][c];
        b += w * hs[1][r + kHalo - k][c];
        cc += w * hs[2][r + kHalo - k][c];
      }
      const size_t o = ((size_t)py * d.W + px) * 3 + ch;
      const float x = __ldg(img + o), y = __ldg(ref + o);
      const float diff = x - y;
      l1 += (double)fabsf(diff);
      const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
      so[r][c * 3 + ch] = d.k_l1 * sgn + d.k_ssim * (a + 2.f * x * b + y * cc);
    }
    __syncthreads();
  }
  // coalesced HWC write of the tile
  for (int i = threadIdx.x; i < kTY * kTX * 3; i += kLossThreads) {
    const int r = i / (kTX * 3), cc = i - r * (kTX * 3);
    const int py = oy + r, px = ox + cc / 3;
    if (py < d.H && px < d.W) grad[((size_t)py * d.W + px) * 3 + (cc % 3)] = so[r][cc];
  }
  l1 = warp_sum(l1);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = l1;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kLossThreads / 32; ++w) t += s_red[w];
    atomicAdd(acc, t);
  }
}

__global__ void k_loss_finalize(const double* acc, LossDims d, double lam, double* loss) {
  const double l1 = acc[0] / (3.0 * d.H * d.W);
  const double s = acc[1] / (3.0 * (double)d.Hv * d.Wv);
  loss[0] = (1.0 - lam) * l1 + lam * (1.0 - s);
}

static void set_window() {
  static bool done = false;  // the window is a constant of the op (metrics.py:60-64)
  if (done) return;
  double g[kWin], sum = 0.0;
  for (int k = 0; k < kWin; ++k) {
    const double x = k - kWin / 2;
    g[k] = exp(-(x * x) / (2.0 * 1.5 * 1.5));
    sum += g[k];
  }
  float gf[kWin];
  for (int k = 0; k < kWin; ++k) gf[k] = (float)(g[k] / sum);
  cudaMemcpyToSymbol(c_win, gf, sizeof(gf));
  done = true;
}

void launch_training_loss(const float* img, const float* ref, int H, int W, double lam,
                          float* maps, double* acc, double* loss, float* grad, cudaStream_t s) {
  set_window();
  LossDims d;
  d.H = H; d.W = W; d.Hv = H - kHalo; d.Wv = W - kHalo;
  d.k_l1 = (float)((1.0 - lam) / (3.0 * H * W));
  d.k_ssim = (float)(-lam / (3.0 * (double)d.Hv * d.Wv));
  cudaMemsetAsync(acc, 0, 2 * sizeof(double), s);
  dim3 g1((d.Wv + kTX - 1) / kTX, (d.Hv + kTY - 1) / kTY);
  k_ssim_stats<<<g1, kLossThreads, 0, s>>>(img, ref, d, maps, acc);
  dim3 g2((W + kTX - 1) / kTX, (H + kTY - 1) / kTY);
  k_ssim_grad<<<g2, kLossThreads, 0, s>>>(img, ref, maps, d, grad, acc);
  k_loss_finalize<<<1, 1, 0, s>>>(acc, d, lam, loss);
}

// ---------------------------------------------------------------------------
// K14: Adam on raw block parameters + activation chain + activated quads

__device__ __forceinline__ void adam1(float& p, float& m, float& v, float g, float lr,
                                      const cs_adam_hparams& h, float bc1, float bc2s) {
  m = h.beta1 * m + (1.f - h.beta1) * g;
  v = h.beta2 * v + (1.f - h.beta2) * g * g;
  const float denom = sqrtf(v) / bc2s + h.eps;
  p -= (lr / bc1) * (m / denom);
}

// One warp per 32 consecutive Gaussians: their (K, 11) rows of parameters and
// both moments are contiguous, so they are staged through shared memory with
// coalesced float4 copies (odd row pitch 11: conflict-free per-lane access),
// updated per lane, and written back the same way.
constexpr int kAdamThreads = 256;

__global__ void __launch_bounds__(kAdamThreads)
k_adam_geom(int64_t K, float* __restrict__ geom, float* __restrict__ gm,
            float* __restrict__ gv, cs_grads g, cs_adam_hparams h, float bc1,
            float bc2s, float4* __restrict__ pos_op, float4* __restrict__ scale,
            float4* __restrict__ quat) {
  __shared__ __align__(16) float s_buf[kAdamThreads / 32][3][32 * 11];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* arrs[3] = {geom, gm, gv};
  for (int64_t base = ((int64_t)blockIdx.x * (kAdamThreads / 32) + warp) * 32; base < K;
       base += (int64_t)gridDim.x * (kAdamThreads / 32) * 32) {
    const int n_rows = (int)min((int64_t)32, K - base);
    const int nf = n_rows * 11;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float* src = arrs[a] + base * 11;
      if (n_rows == 32) {
        const float4* s4 = reinterpret_cast<const float4*>(src);
        float4* d4 = reinterpret_cast<float4*>(s_buf[warp][a]);
        for (int i = lane; i < 88; i += 32) d4[i] = s4[i];
      } else {
        for (int i = lane; i < nf; i += 32) s_buf[warp][a][i] = src[i];
      }
    }
    __syncwarp();
    const int64_t k = base + lane;
    if (lane < n_rows) {
      float* p = &s_buf[warp][0][lane * 11];
      float* m = &s_buf[warp][1][lane * 11];
      float* v = &s_buf[warp][2][lane * 11];
      float gr[11];
      // chain the activated-parameter gradients to the raw parameters
#pragma unroll
      for (int i = 0; i < 3; ++i) gr[i] = g.positions[3 * k + i];
#pragma unroll
      for (int i = 0; i < 3; ++i) gr[3 + i] = g.scales[3 * k + i] * expf(p[3 + i]);  // d exp
      {
        const float q0 = p[6], q1 = p[7], q2 = p[8], q3 = p[9];
        const float n = sqrtf(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
        const float inv = 1.f / n;
        const float u[4] = {q0 * inv, q1 * inv, q2 * inv, q3 * inv};
        const float4 gq4 = reinterpret_cast<const float4*>(g.rotations)[k];
        const float gq[4] = {gq4.x, gq4.y, gq4.z, gq4.w};
        const float dot = u[0] * gq[0] + u[1] * gq[1] + u[2] * gq[2] + u[3] * gq[3];
#pragma unroll
        for (int i = 0; i < 4; ++i) gr[6 + i] = (gq[i] - u[i] * dot) * inv;  // d (q / |q|)
      }
      {
        const float sg = 1.f / (1.f + expf(-p[10]));
        gr[10] = g.opacities[k] * sg * (1.f - sg);  // d sigmoid
      }
      const float lrs[11] = {h.lr_position, h.lr_position, h.lr_position, h.lr_scale, h.lr_scale,
                             h.lr_scale, h.lr_rotation, h.lr_rotation, h.lr_rotation,
                             h.lr_rotation, h.lr_opacity};
      float pr[11], mr[11], vr[11];
#pragma unroll
      for (int i = 0; i < 11; ++i) {
        pr[i] = p[i]; mr[i] = m[i]; vr[i] = v[i];
        adam1(pr[i], mr[i], vr[i], gr[i], lrs[i], h, bc1, bc2s);
        p[i] = pr[i]; m[i] = mr[i]; v[i] = vr[i];
      }
      // activated quads for the next forward
      const float n = sqrtf(pr[6] * pr[6] + pr[7] * pr[7] + pr[8] * pr[8] + pr[9] * pr[9]);
      pos_op[k] = make_float4(pr[0], pr[1], pr[2], 1.f / (1.f + expf(-pr[10])));
      scale[k] = make_float4(expf(pr[3]), expf(pr[4]), expf(pr[5]), 0.f);
      quat[k] = make_float4(pr[6] / n, pr[7] / n, pr[8] / n, pr[9] / n);
    }
    __syncwarp();
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float* dst = arrs[a] + base * 11;
      if (n_rows == 32) {
        float4* d4 = reinterpret_cast<float4*>(dst);
        const float4* s4 = reinterpret_cast<const float4*>(s_buf[warp][a]);
        for (int i = lane; i < 88; i += 32) d4[i] = s4[i];
      } else {
        for (int i = lane; i < nf; i += 32) dst[i] = s_buf[warp][a][i];
      }
    }
    __syncwarp();
  }
}

__global__ void k_adam_flat(int64_t n, float* __restrict__ p, float* __restrict__ m,
                            float* __restrict__ v, const float* __restrict__ g, float lr,
                            cs_adam_hparams h, float bc1, float bc2s) {
  const int64_t n4 = n / 4;
  float4* p4 = reinterpret_cast<float4*>(p);
  float4* m4 = reinterpret_cast<float4*>(m);
  float4* v4 = reinterpret_cast<float4*>(v);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 pp = p4[i], mm = m4[i], vv = v4[i];
    const float4 gg = __ldg(g4 + i);
    adam1(pp.x, mm.x, vv.x, gg.x, lr, h, bc1, bc2s);
    adam1(pp.y, mm.y, vv.y, gg.y, lr, h, bc1, bc2s);
    adam1(pp.z, mm.z, vv.z, gg.z, lr, h, bc1, bc2s);
    adam1(pp.w, mm.w, vv.w, gg.w, lr, h, bc1, bc2s);
    p4[i] = pp; m4[i] = mm; v4[i] = vv;
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    adam1(p[i], m[i], v[i], g[i], lr, h, bc1, bc2s);
}

__global__ void k_activate_geom(int64_t K, const float* __restrict__ geom, float4* __restrict__ pos_op,
                                float4* __restrict__ scale, float4* __restrict__ quat) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K;
       k += (int64_t)gridDim.x * blockDim.x) {
    const float* p = geom + 11 * k;
    const float n = sqrtf(p[6] * p[6] + p[7] * p[7] + p[8] * p[8] + p[9] * p[9]);
    pos_op[k] = make_float4(p[0], p[1], p[2], 1.f / (1.f + expf(-p[10])));
    scale[k] = make_float4(expf(p[3]), expf(p[4]), expf(p[5]), 0.f);
    quat[k] = make_float4(p[6] / n, p[7] / n, p[8] / n, p[9] / n);
  }
}

void launch_block_adam(int64_t K, int C, float* geom, float* gm, float* gv, float* sh, float* shm,
                       float* shv, const cs_grads& g, const cs_adam_hparams& h, float4* pos_op,
                       float4* scale, float4* quat, cudaStream_t s) {
  const double bc1 = 1.0 - pow((double)h.beta1, (double)h.step);
  const double bc2 = 1.0 - pow((double)h.beta2, (double)h.step);
  const float bc2s = (float)sqrt(bc2);
  if (K <= 0) return;
  const int grid = (int)std::min<int64_t>(148 * 8, (K + kAdamThreads - 1) / kAdamThreads);
  k_adam_geom<<<grid, kAdamThreads, 0, s>>>(K, geom, gm, gv, g, h, (float)bc1, bc2s, pos_op, scale,
                                            quat);
  const int64_t n = K * 3 * C;
  const int grid2 = (int)std::min<int64_t>(148 * 8, (n / 4 + 255) / 256 + 1);
  k_adam_flat<<<grid2, 256, 0, s>>>(n, sh, shm, shv, g.sh, h.lr_sh, h, (float)bc1, bc2s);
}

void launch_activate_geom(int64_t K, const float* geom, float4* pos_op, float4* scale, float4* quat,
                          cudaStream_t s) {
  if (K <= 0) return;
  const int grid = (int)std::min<int64_t>(148 * 8, (K + 255) / 256);
  k_activate_geom<<<grid, 256, 0, s>>>(K, geom, pos_op, scale, quat);
}

}  // namespace cs

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
// Both run one block per (32x32 tile, channel): the tile's 42x42 region is
// staged in shared memory and the 11-tap window runs as a horizontal then a
// vertical register-sliding pass (8 outputs per thread, each input read once).
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
constexpr int kTX = 32, kTY = 32;                   // output tile of both loss kernels
constexpr int kSeg = 8;                             // outputs per thread along a sliding pass
constexpr int kRX = kTX + kHalo, kRY = kTY + kHalo;  // 42 x 42 region
constexpr int kRP = kRX + 1;                        // odd region pitch: conflict-free rows
constexpr int kHP = kTX + 1;                        // pass-1 output pitch
constexpr int kSegsX = kTX / kSeg, kSegsY = kTY / kSeg;
constexpr int kGOff = 12;                           // grad region starts 12 columns left (aligned)
constexpr int kGChunks = (kTX + kGOff) / 4;         // 11 float4 chunks per region row
constexpr int kGP = 4 * kGChunks;                   // 44: 16-byte rows, conflict-free LDS.128
constexpr int kLossThreads = 256;
constexpr float kC1 = 0.01f * 0.01f, kC2 = 0.03f * 0.03f;

__constant__ float c_win[kWin];

struct LossDims {
  int H, W, Hv, Wv;
  int Wp;        // maps row pitch: Wv rounded up to 4 (pad columns hold zeros)
  float k_l1;    // (1 - lam) / (3 H W)
  float k_ssim;  // -lam / (3 Hv Wv)
};

// 4-byte asynchronous copy into shared memory, zero-filled when !valid (the
// staging loops issue every copy of the region before the first wait instead
// of one dependent load/store round trip per loop iteration).
__device__ __forceinline__ void cp_async4(float* smem, const float* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sa), "l"(gmem), "r"(valid ? 4 : 0)
               : "memory");
}

__device__ __forceinline__ void cp_async16z(float* smem, const float* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0)
               : "memory");
}

// One step of a register-sliding 11-tap pass: input j (of kSeg + kHalo) adds
// into every output o it falls under, tap j - o (the correlation of the
// forward statistics) or kHalo - (j - o) (the adjoint correlation of the
// gradient).  j is a compile-time index of an unrolled loop, so the tap
// selection folds away and each thread reads each input once instead of 11x.
template <int N, bool ADJ>
__device__ __forceinline__ void win_step(float (&acc)[kSeg][N], int j, const float (&v)[N]) {
#pragma unroll
  for (int o = 0; o < kSeg; ++o) {
    const int k = ADJ ? kHalo - (j - o) : j - o;
    if (j - o >= 0 && j - o < kWin) {
#pragma unroll
      for (int n = 0; n < N; ++n) acc[o][n] = fmaf(c_win[k], v[n], acc[o][n]);
    }
  }
}

// maps layout: [ch][3][Hv][Wp]  (A, B, C); columns Wv..Wp-1 are written as zeros.
// One block per 32x32 window tile, all three channels: the tile's 42 image
// rows x 42 pixels x 3 channels are staged interleaved, as they lie in HWC
// (16-byte copies when a row of 3W floats keeps 16-byte alignment, VEC), and
// each channel then runs the two sliding passes; the horizontal pass picks
// its channel out of 16-byte shared loads.
constexpr int kSX = 132;  // staged row pitch: 126 floats -> 33 float4 (odd: conflict-free LDS.128)
constexpr int kStatsSmem = (2 * kRY * kSX + 5 * kRY * kHP) * 4;

template <bool VEC>
__global__ void __launch_bounds__(kLossThreads, 3)
k_ssim_stats(const float* __restrict__ img, const float* __restrict__ ref, LossDims d,
             float* __restrict__ maps, double* __restrict__ acc) {
  extern __shared__ __align__(16) float dsm[];  // kStatsSmem bytes
  float(*sx)[kSX] = reinterpret_cast<float(*)[kSX]>(dsm);
  float(*sy)[kSX] = reinterpret_cast<float(*)[kSX]>(dsm + kRY * kSX);
  float(*hs)[kRY][kHP] = reinterpret_cast<float(*)[kRY][kHP]>(dsm + 2 * kRY * kSX);
  __shared__ double s_red[kLossThreads / 32];
  const int ox = blockIdx.x * kTX, oy = blockIdx.y * kTY;
  const int rowlen = 3 * d.W;
  if (VEC) {
    for (int i = threadIdx.x; i < kRY * 32; i += kLossThreads) {
      const int r = i >> 5, k = i & 31;
      const int gy = oy + r, f = 3 * ox + 4 * k;
      const bool in = gy < d.H && f < rowlen;
      const size_t o = in ? (size_t)gy * rowlen + f : 0;
      cp_async16z(&sx[r][4 * k], img + o, in);
      cp_async16z(&sy[r][4 * k], ref + o, in);
    }
  } else {
    for (int i = threadIdx.x; i < kRY * 128; i += kLossThreads) {
      const int r = i >> 7, k = i & 127;
      const int gy = oy + r, f = 3 * ox + k;
      const bool in = gy < d.H && f < rowlen;
      const size_t o = in ? (size_t)gy * rowlen + f : 0;
      cp_async4(&sx[r][k], img + o, in);
      cp_async4(&sy[r][k], ref + o, in);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  double ssum = 0.0;
  const size_t plane = (size_t)d.Hv * d.Wp;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
  // horizontal pass: (row, 8-column segment) per thread, segment fastest;
  // input pixel c0 + j, channel ch = float 3 (c0 + j) + ch of the staged row
  for (int i = threadIdx.x; i < kRY * kSegsX; i += kLossThreads) {
    const int r = i / kSegsX, s4 = i - r * kSegsX, c0 = s4 * kSeg;
    const float* rx = &sx[r][3 * c0];
    const float* ry = &sy[r][3 * c0];
    float a[kSeg][5] = {};
    float4 qx = make_float4(0.f, 0.f, 0.f, 0.f), qy = qx;
#pragma unroll
    for (int j = 0; j < kSeg + kHalo; ++j) {
      const int e = 3 * j + ch;
      if (j == 0 || (e >> 2) != ((e - 3) >> 2)) {  // compile-time: first use of this chunk
        qx = *reinterpret_cast<const float4*>(rx + 4 * (e >> 2));
        qy = *reinterpret_cast<const float4*>(ry + 4 * (e >> 2));
      }
      const int w = e & 3;
      const float x = w == 0 ? qx.x : w == 1 ? qx.y : w == 2 ? qx.z : qx.w;
      const float y = w == 0 ? qy.x : w == 1 ? qy.y : w == 2 ? qy.z : qy.w;
      const float v[5] = {x, y, x * x, y * y, x * y};
      win_step<5, false>(a, j, v);
    }
#pragma unroll
    for (int o = 0; o < kSeg; ++o)
#pragma unroll
      for (int n = 0; n < 5; ++n) hs[n][r][c0 + o] = a[o][n];
  }
  __syncthreads();
  float* m = maps + (size_t)ch * 3 * plane;
  // vertical pass + per-window SSIM and partials: (column, 8-row segment)
  for (int i = threadIdx.x; i < kTX * kSegsY; i += kLossThreads) {
    const int c = i % kTX, r0 = (i / kTX) * kSeg;
    float a[kSeg][5] = {};
#pragma unroll
    for (int j = 0; j < kSeg + kHalo; ++j) {
      const float v[5] = {hs[0][r0 + j][c], hs[1][r0 + j][c], hs[2][r0 + j][c], hs[3][r0 + j][c],
                          hs[4][r0 + j][c]};
      win_step<5, false>(a, j, v);
    }
    const int qx = ox + c;
    const size_t q0 = (size_t)(oy + r0) * d.Wp + qx;
#pragma unroll
    for (int o = 0; o < kSeg; ++o) {
      // the zero-filled region keeps out-of-range windows finite (d1 >= C1,
      // d2 >= C2): evaluate unconditionally, predicate the sum and the stores
      const bool row_ok = oy + r0 + o < d.Hv;
      const bool valid = row_ok && qx < d.Wv;
      const float mx = a[o][0], my = a[o][1], xx = a[o][2], yy = a[o][3], xy = a[o][4];
      const float vx = xx - mx * mx, vy = yy - my * my, cv = xy - mx * my;
      const float n1 = 2.f * mx * my + kC1, n2 = 2.f * cv + kC2;
      const float d1 = mx * mx + my * my + kC1, d2 = vx + vy + kC2;
      const float inv = 1.f / (d1 * d2);
      const float S = n1 * n2 * inv;
      ssum += valid ? (double)S : 0.0;
      // dS/dmu_x with E[xx], E[xy] held fixed (var_x, cov depend on mu_x);
      // 1/d1 = d2 inv, 1/d2 = d1 inv
      const float A = 2.f * my * (n2 - n1) * inv - S * 2.f * mx * (d2 - d1) * inv;
      const float B = -S * d1 * inv;      // dS/dE[xx]
      const float C = 2.f * n1 * inv;     // dS/dE[xy]
      if (row_ok && qx < d.Wp) {
        const size_t q = q0 + (size_t)o * d.Wp;
        m[q] = valid ? A : 0.f;
        m[plane + q] = valid ? B : 0.f;
        m[2 * plane + q] = valid ? C : 0.f;
      }
    }
  }
  __syncthreads();  // hs is rewritten by the next channel
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
  // A, B, C region of this channel: windows rows oy-10 .. oy+31, columns
  // ox-12 .. ox+31 (16-byte aligned: ox and the pitch Wp are multiples of 4)
  __shared__ __align__(16) float sm[3][kRY][kGP];
  __shared__ float hs[3][kRY][kHP];
  __shared__ double s_red[kLossThreads / 32];
  const int ch = blockIdx.z;
  const int ox = blockIdx.x * kTX, oy = blockIdx.y * kTY;
  const size_t plane = (size_t)d.Hv * d.Wp;
  const float* m = maps + (size_t)ch * 3 * plane;
  for (int i = threadIdx.x; i < 3 * kRY * kGChunks; i += kLossThreads) {
    const int row = i / kGChunks, k = i - row * kGChunks;
    const int mi = row / kRY, r = row - mi * kRY;
    const int qy = oy - kHalo + r, qx = ox - kGOff + 4 * k;
    const bool in = qy >= 0 && qy < d.Hv && qx >= 0 && qx < d.Wp;
    cp_async16z(&sm[mi][r][4 * k], m + (in ? mi * plane + (size_t)qy * d.Wp + qx : 0), in);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * kRY * kSegsX; i += kLossThreads) {
    const int mi = i / (kRY * kSegsX), rem = i - mi * (kRY * kSegsX);
    const int r = rem / kSegsX, c0 = (rem - r * kSegsX) * kSeg;
    float a[kSeg][1] = {};
    float in[kSeg + 16];  // region columns c0 .. c0+23 (taps use c0+2 .. c0+19)
#pragma unroll
    for (int t = 0; t < 6; ++t) {
      const float4 q = *reinterpret_cast<const float4*>(&sm[mi][r][c0 + 4 * t]);
      in[4 * t] = q.x; in[4 * t + 1] = q.y; in[4 * t + 2] = q.z; in[4 * t + 3] = q.w;
    }
#pragma unroll
    for (int j = 0; j < kSeg + kHalo; ++j) {
      const float v[1] = {in[kGOff - kHalo + j]};
      win_step<1, true>(a, j, v);
    }
#pragma unroll
    for (int o = 0; o < kSeg; ++o) hs[mi][r][c0 + o] = a[o][0];
  }
  __syncthreads();
  double l1 = 0.0;
  for (int i = threadIdx.x; i < kTX * kSegsY; i += kLossThreads) {
    const int c = i % kTX, r0 = (i / kTX) * kSeg;
    const int px = ox + c;
    // issue the 8 pixels' image loads before the window sums hide their latency
    float xs[kSeg], ys[kSeg];
#pragma unroll
    for (int o = 0; o < kSeg; ++o) {
      const int py = oy + r0 + o;
      const bool in = py < d.H && px < d.W;
      const size_t q = in ? ((size_t)py * d.W + px) * 3 + ch : 0;
      xs[o] = in ? __ldg(img + q) : 0.f;
      ys[o] = in ? __ldg(ref + q) : 0.f;
    }
    float a[kSeg][3] = {};
#pragma unroll
    for (int j = 0; j < kSeg + kHalo; ++j) {
      const float v[3] = {hs[0][r0 + j][c], hs[1][r0 + j][c], hs[2][r0 + j][c]};
      win_step<3, true>(a, j, v);
    }
#pragma unroll
    for (int o = 0; o < kSeg; ++o) {
      const int py = oy + r0 + o;
      if (py >= d.H || px >= d.W) continue;
      const size_t q = ((size_t)py * d.W + px) * 3 + ch;
      const float x = xs[o], y = ys[o];
      const float diff = x - y;
      l1 += (double)fabsf(diff);
      const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
      grad[q] = d.k_l1 * sgn + d.k_ssim * (a[o][0] + 2.f * x * a[o][1] + y * a[o][2]);
    }
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
  d.H = H; d.W = W; d.Hv = H - kHalo; d.Wv = W - kHalo; d.Wp = (d.Wv + 3) & ~3;
  d.k_l1 = (float)((1.0 - lam) / (3.0 * H * W));
  d.k_ssim = (float)(-lam / (3.0 * (double)d.Hv * d.Wv));
  cudaMemsetAsync(acc, 0, 2 * sizeof(double), s);
  dim3 g1((d.Wv + kTX - 1) / kTX, (d.Hv + kTY - 1) / kTY);
  // 16-byte staging needs every image row (3W floats) 16-byte aligned
  const bool vec = (W & 3) == 0 && ((reinterpret_cast<uintptr_t>(img) | reinterpret_cast<uintptr_t>(ref)) & 15) == 0;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_ssim_stats<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStatsSmem);
    cudaFuncSetAttribute(k_ssim_stats<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStatsSmem);
    attr = true;
  }
  if (vec) k_ssim_stats<true><<<g1, kLossThreads, kStatsSmem, s>>>(img, ref, d, maps, acc);
  else k_ssim_stats<false><<<g1, kLossThreads, kStatsSmem, s>>>(img, ref, d, maps, acc);
  dim3 g2((W + kTX - 1) / kTX, (H + kTY - 1) / kTY, 3);
  k_ssim_grad<<<g2, kLossThreads, 0, s>>>(img, ref, maps, d, grad, acc);
  k_loss_finalize<<<1, 1, 0, s>>>(acc, d, lam, loss);
}

// ---------------------------------------------------------------------------
// K14: Adam on raw block parameters + activation chain + activated quads

// torch.optim.Adam (bias-corrected, eps outside the root) with the root and
// the quotient as single MUFU-based approximations (relative error ~1e-7,
// far inside the trainer-vs-torch bound) instead of IEEE sqrt / division
// sequences: the SH stream was issue-bound on them.  step = lr / bc1,
// ibc2s = 1 / sqrt(bc2).
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void adam1(float& p, float& m, float& v, float g, float step,
                                      const cs_adam_hparams& h, float ibc2s) {
  m = h.beta1 * m + (1.f - h.beta1) * g;
  v = h.beta2 * v + (1.f - h.beta2) * g * g;
  const float denom = fmaf(sqrt_approx(v), ibc2s, h.eps);
  p -= step * __fdividef(m, denom);
}

// One warp per 32 consecutive Gaussians: their (K, 11) rows of parameters and
// both moments are contiguous, so they are staged through shared memory with
// coalesced float4 copies (odd row pitch 11: conflict-free per-lane access),
// updated per lane, and written back the same way.
constexpr int kAdamThreads = 256;
#ifndef CS_ADAM_GEOM_DIV
#define CS_ADAM_GEOM_DIV 3  // 1 / (fraction of the Adam CTAs on geometry rows)
#endif

__device__ __forceinline__ void adam_geom(int blk, int nblk, int64_t K, float* __restrict__ geom,
                                          float* __restrict__ gm, float* __restrict__ gv,
                                          const cs_grads& g, const cs_adam_hparams& h, float ibc1,
                                          float ibc2s, float4* __restrict__ pos_op,
                                          float4* __restrict__ scale, float4* __restrict__ quat,
                                          float (*s_buf)[3][32 * 11]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* arrs[3] = {geom, gm, gv};
  for (int64_t base = ((int64_t)blk * (kAdamThreads / 32) + warp) * 32; base < K;
       base += (int64_t)nblk * (kAdamThreads / 32) * 32) {
    const int n_rows = (int)min((int64_t)32, K - base);
    const int nf = n_rows * 11;
    // asynchronous staging: all 3 x 88 16-byte copies in flight at once
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float* src = arrs[a] + base * 11;
      if (n_rows == 32) {
#pragma unroll
        for (int i = lane; i < 88 + 32; i += 32)
          if (i < 88) cp_async16(&s_buf[warp][a][4 * i], src + 4 * i);
      } else {
        for (int i = lane; i < nf; i += 32) s_buf[warp][a][i] = src[i];
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
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
        adam1(pr[i], mr[i], vr[i], gr[i], lrs[i] * ibc1, h, ibc2s);
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

// SH moments: elementwise, two float4 groups per thread per iteration (16
// independent 16-byte loads in flight per thread)
__device__ __forceinline__ void adam_flat(int blk, int nblk, int64_t n, float* __restrict__ p,
                                          float* __restrict__ m, float* __restrict__ v,
                                          const float* __restrict__ g, float step,
                                          const cs_adam_hparams& h, float ibc2s) {
  const int64_t n4 = n / 4;
  float4* p4 = reinterpret_cast<float4*>(p);
  float4* m4 = reinterpret_cast<float4*>(m);
  float4* v4 = reinterpret_cast<float4*>(v);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const int64_t stride = (int64_t)nblk * blockDim.x;
  const int64_t t = blk * (int64_t)blockDim.x + threadIdx.x;
  auto upd = [&](float4& pp, float4& mm, float4& vv, const float4& gg) {
    adam1(pp.x, mm.x, vv.x, gg.x, step, h, ibc2s);
    adam1(pp.y, mm.y, vv.y, gg.y, step, h, ibc2s);
    adam1(pp.z, mm.z, vv.z, gg.z, step, h, ibc2s);
    adam1(pp.w, mm.w, vv.w, gg.w, step, h, ibc2s);
  };
  int64_t i = t;
  for (; i + stride < n4; i += 2 * stride) {
    const int64_t j = i + stride;
    float4 pa = p4[i], ma = m4[i], va = v4[i];
    float4 pb = p4[j], mb = m4[j], vb = v4[j];
    const float4 ga = __ldg(g4 + i), gb = __ldg(g4 + j);
    upd(pa, ma, va, ga);
    upd(pb, mb, vb, gb);
    p4[i] = pa; m4[i] = ma; v4[i] = va;
    p4[j] = pb; m4[j] = mb; v4[j] = vb;
  }
  if (i < n4) {
    float4 pa = p4[i], ma = m4[i], va = v4[i];
    upd(pa, ma, va, __ldg(g4 + i));
    p4[i] = pa; m4[i] = ma; v4[i] = va;
  }
  for (int64_t k = 4 * n4 + t; k < n; k += stride) adam1(p[k], m[k], v[k], g[k], step, h, ibc2s);
}

// One launch for both parameter groups: the first geom_blocks CTAs run the
// geometry rows, the rest the SH moments, so the latency-bound geometry
// update overlaps the bandwidth-bound SH stream instead of preceding it.
__global__ void __launch_bounds__(kAdamThreads, 4)
k_adam(int64_t K, int geom_blocks, float* __restrict__ geom, float* __restrict__ gm,
       float* __restrict__ gv, int64_t n_sh, float* __restrict__ sh, float* __restrict__ shm,
       float* __restrict__ shv, cs_grads g, cs_adam_hparams h, float ibc1, float ibc2s,
       float4* __restrict__ pos_op, float4* __restrict__ scale, float4* __restrict__ quat) {
  __shared__ __align__(16) float s_buf[kAdamThreads / 32][3][32 * 11];
  if ((int)blockIdx.x < geom_blocks)
    adam_geom(blockIdx.x, geom_blocks, K, geom, gm, gv, g, h, ibc1, ibc2s, pos_op, scale, quat, s_buf);
  else
    adam_flat(blockIdx.x - geom_blocks, gridDim.x - geom_blocks, n_sh, sh, shm, shv, g.sh, h.lr_sh * ibc1, h,
              ibc2s);
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
  const float ibc1 = (float)(1.0 / bc1), ibc2s = (float)(1.0 / sqrt(bc2));
  if (K <= 0) return;
  // one resident wave (4 CTAs/SM: 64 registers), split by traffic: the
  // geometry rows are ~1/5 of the bytes but latency-bound, so ~1/3 of the CTAs
  const int64_t n = K * 3 * C;
  const int wave = 148 * 4;
  const int gb = (int)std::max<int64_t>(1, std::min<int64_t>(wave / CS_ADAM_GEOM_DIV, (K + kAdamThreads - 1) / kAdamThreads));
  const int fb = (int)std::max<int64_t>(1, std::min<int64_t>(wave - gb, (n / 4 + kAdamThreads - 1) / kAdamThreads));
  k_adam<<<gb + fb, kAdamThreads, 0, s>>>(K, gb, geom, gm, gv, n, sh, shm, shv, g, h, ibc1, ibc2s,
                                          pos_op, scale, quat);
}

void launch_activate_geom(int64_t K, const float* geom, float4* pos_op, float4* scale, float4* quat,
                          cudaStream_t s) {
  if (K <= 0) return;
  const int grid = (int)std::min<int64_t>(148 * 8, (K + 255) / 256);
  k_activate_geom<<<grid, 256, 0, s>>>(K, geom, pos_op, scale, quat);
}

}  // namespace cs

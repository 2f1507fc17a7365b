// cs_assign.cu -- K20: SSIM of two rendered images for training-data assignment.
//
// Replaces metrics.ssim / l_ssim (metrics.py:70-101) as used by the
// contribution test of partition.assign_b1 / assign (partition.py:318-334,
// partition.py:382-386): per channel the 11x11 Gaussian-window (sigma 1.5)
// local statistics over the valid region, C1 = 0.01^2, C2 = 0.03^2,
//   num = (2 mu_x mu_y + C1)(2 cov + C2),  den = (mu_x^2 + mu_y^2 + C1)(var_x + var_y + C2)
// and the mean of num / den, averaged over the three channels.  The window
// weights are the reference's own (outer(g, g) / sum, computed by the host
// with numpy and passed in), applied as a direct 2D correlation (the window
// is symmetric, so equal to scipy's convolution) in float64 from the float32
// rendered pixels.  The reference's scipy.signal.convolve may evaluate by
// FFT, so the two agree to rounding (~1e-15 relative), not bit for bit.
#include "cs_internal.cuh"

namespace cs {

constexpr int kWin = 11;
constexpr int kSsimTile = 16;
constexpr int kSsimIn = kSsimTile + kWin - 1;  // 26

__constant__ double c_ssim_w[kWin * kWin];

// One CTA per 16x16 block of valid output positions; the 26x26 input patches
// of both images (3 channels) are staged in shared memory.  acc[c] += sum of
// num/den over the CTA's outputs (channel c).
__global__ void __launch_bounds__(kSsimTile * kSsimTile)
k_ssim(const float* __restrict__ a, const float* __restrict__ b, int H, int W,
       double* __restrict__ acc) {
  __shared__ float sa[3][kSsimIn][kSsimIn + 1];
  __shared__ float sb[3][kSsimIn][kSsimIn + 1];
  __shared__ double red[3][kSsimTile * kSsimTile / 32];
  const int ox0 = blockIdx.x * kSsimTile, oy0 = blockIdx.y * kSsimTile;
  const int tid = threadIdx.y * kSsimTile + threadIdx.x;
  for (int i = tid; i < kSsimIn * kSsimIn; i += kSsimTile * kSsimTile) {
    const int r = i / kSsimIn, c = i - r * kSsimIn;
    const int y = oy0 + r, x = ox0 + c;
    const bool in = y < H && x < W;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      sa[ch][r][c] = in ? a[((int64_t)y * W + x) * 3 + ch] : 0.f;
      sb[ch][r][c] = in ? b[((int64_t)y * W + x) * 3 + ch] : 0.f;
    }
  }
  __syncthreads();
  const int Ho = H - kWin + 1, Wo = W - kWin + 1;
  const int ox = ox0 + threadIdx.x, oy = oy0 + threadIdx.y;
  const bool valid = ox < Wo && oy < Ho;
  double val[3] = {0.0, 0.0, 0.0};
  if (valid) {
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      double mx = 0.0, my = 0.0, exx = 0.0, eyy = 0.0, exy = 0.0;
      for (int u = 0; u < kWin; ++u)
#pragma unroll
        for (int v = 0; v < kWin; ++v) {
          const double w = c_ssim_w[u * kWin + v];
          const double x = (double)sa[ch][threadIdx.y + u][threadIdx.x + v];
          const double y = (double)sb[ch][threadIdx.y + u][threadIdx.x + v];
          mx += w * x;
          my += w * y;
          exx += w * (x * x);
          eyy += w * (y * y);
          exy += w * (x * y);
        }
      const double var_x = exx - mx * mx, var_y = eyy - my * my, cov = exy - mx * my;
      const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
      const double num = (2.0 * mx * my + C1) * (2.0 * cov + C2);
      const double den = (mx * mx + my * my + C1) * (var_x + var_y + C2);
      val[ch] = num / den;
    }
  }
  const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    const double s = warp_sum(val[ch]);
    if (lane == 0) red[ch][warp] = s;
  }
  __syncthreads();
  if (tid < 3) {
    double s = 0.0;
    for (int w = 0; w < kSsimTile * kSsimTile / 32; ++w) s += red[tid][w];
    atomicAdd(&acc[tid], s);
  }
}

// acc[3] = mean over channels of acc[c] / (Ho * Wo)   (np.mean of each map, then of the 3)
__global__ void k_ssim_finish(double* acc, int64_t n_valid) {
  acc[3] = ((acc[0] / (double)n_valid + acc[1] / (double)n_valid) + acc[2] / (double)n_valid) / 3.0;
}

cudaError_t ssim_run(const float* a, const float* b, int H, int W, const double* window,
                     double* acc4, cudaStream_t s) {
  cudaError_t e;
  if ((e = cudaMemcpyToSymbolAsync(c_ssim_w, window, sizeof(double) * kWin * kWin, 0,
                                   cudaMemcpyHostToDevice, s)))
    return e;
  if ((e = cudaMemsetAsync(acc4, 0, sizeof(double) * 4, s))) return e;
  const int Ho = H - kWin + 1, Wo = W - kWin + 1;
  dim3 grid((Wo + kSsimTile - 1) / kSsimTile, (Ho + kSsimTile - 1) / kSsimTile);
  k_ssim<<<grid, dim3(kSsimTile, kSsimTile), 0, s>>>(a, b, H, W, acc4);
  k_ssim_finish<<<1, 1, 0, s>>>(acc4, (int64_t)Ho * Wo);
  return cudaGetLastError();
}

}  // namespace cs

namespace cs {

// FP64 peak microbenchmark (the blend's roofline denominator is
// measured on the box): every thread runs 8 independent DFMA chains.
__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = (double)(threadIdx.x + i) * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

cudaError_t fp64_peak_run(double* tflops, cudaStream_t s) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&out), sizeof(double), s);
  if (e) return e;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, iters = 4096;
  k_dfma_peak<<<blocks, 256, 0, s>>>(out, 64, 1.0000001, 1e-12);  // warm-up
  cudaEventRecord(e0, s);
  k_dfma_peak<<<blocks, 256, 0, s>>>(out, iters, 1.0000001, 1e-12);
  cudaEventRecord(e1, s);
  e = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *tflops = 2.0 * 8.0 * iters * (double)blocks * 256.0 / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(out, s);
  return e ? e : cudaGetLastError();
}

}  // namespace cs

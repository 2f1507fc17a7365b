// cs_depth.cu -- K4b: exact depth order from a 32-bit radix sort.
//
// The reference orders visible splats by np.argsort(depths, kind="stable")
// (render.py:176-177): float64 depth, ties by assembled index.  K4 sorts only
// a 32-bit monotone coarsening of the float64 depth (the top bits of
// bits(z) - bits(near), cs_project.cu: 4 radix passes over 8-byte (key, id)
// pairs instead of 8 over 12-byte ones).  Splats with equal 32-bit keys
// form runs that are contiguous after the sort and already in ascending id
// order (the sort is stable); this kernel re-sorts every run by (float64
// depth bits, id), which restores the reference order exactly.
//   * runs of <= 8 (nearly all; 1-ulp float32 buckets at city scale hold a
//     few splats at most): one thread, insertion sort in registers;
//   * longer runs (e.g. many splats at exactly equal depth): queued and
//     sorted by one CTA each -- bitonic in shared memory up to 2048
//     entries, beyond that a merge of sorted 2048-blocks through a global
//     scratch buffer (ranks by binary search; (depth, id) keys are distinct).
#include "cs_internal.cuh"

namespace cs {

constexpr int kShortRun = 8;
constexpr int kSmemSort = 2048;

struct RunCtl {
  uint32_t n_long;   // long runs queued
  uint32_t ticket;   // CTA work ticket over the long runs
  uint32_t pad[2];
};

__device__ __forceinline__ bool key_less(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

// One run of equal 32-bit keys starting at rank r (r + 1 < M, k32[r + 1] ==
// k32[r]): short runs are re-sorted in registers, long ones queued.
__device__ __forceinline__ void fix_run(const uint32_t* __restrict__ k32, uint32_t* __restrict__ order,
                                        const uint64_t* __restrict__ k64, int64_t M, int64_t r,
                                        RunCtl* __restrict__ ctl, uint32_t* __restrict__ long_runs,
                                        uint32_t long_cap) {
  const uint32_t k = k32[r];
  int L = 2;
  while (L <= kShortRun && r + L < M && k32[r + L] == k) ++L;
  if (L > kShortRun) {  // long_cap >= M / (kShortRun + 1) + 1: the queue cannot overflow
    const uint32_t slot = atomicAdd(&ctl->n_long, 1u);
    if (slot < long_cap) long_runs[slot] = (uint32_t)r;
    return;
  }
  uint32_t id[kShortRun];
  uint64_t key[kShortRun];
#pragma unroll
  for (int j = 0; j < kShortRun; ++j) {
    if (j < L) {
      id[j] = order[r + j];
      key[j] = k64[id[j]];
    }
  }
  // insertion sort (ids arrive ascending, so equal depths keep their order)
#pragma unroll
  for (int j = 1; j < kShortRun; ++j) {
    if (j >= L) break;
#pragma unroll
    for (int m = j; m > 0; --m) {
      if (key_less(key[m], id[m], key[m - 1], id[m - 1])) {
        const uint64_t tk = key[m]; key[m] = key[m - 1]; key[m - 1] = tk;
        const uint32_t ti = id[m]; id[m] = id[m - 1]; id[m - 1] = ti;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kShortRun; ++j)
    if (j < L) order[r + j] = id[j];
}

// Run starts, four ranks per thread (one 16-byte key load plus the two
// neighbours): the scan is a streaming read, the rare runs branch off.
__global__ void k_fix_short_runs(const uint32_t* __restrict__ k32, uint32_t* __restrict__ order,
                                 const uint64_t* __restrict__ k64, const DevStats* __restrict__ stats,
                                 RunCtl* __restrict__ ctl, uint32_t* __restrict__ long_runs,
                                 uint32_t long_cap) {
  const int64_t M = stats->visible;
  const int64_t groups = (M + 3) / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gi < groups; gi += stride) {
    const int64_t r0 = 4 * gi;
    uint32_t k[6];  // k[0] = rank r0 - 1, k[1..4] = r0..r0+3, k[5] = r0 + 4
    if (r0 + 4 <= M) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(k32) + gi);
      k[1] = v.x; k[2] = v.y; k[3] = v.z; k[4] = v.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) k[1 + j] = r0 + j < M ? __ldg(k32 + r0 + j) : 0xfffffffeu - j;
    }
    k[0] = r0 > 0 ? __ldg(k32 + r0 - 1) : ~k[1];
    k[5] = r0 + 4 < M ? __ldg(k32 + r0 + 4) : ~k[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t r = r0 + j;
      // the start of a run: equal to the next key, different from the previous
      if (r + 1 < M && k[j + 2] == k[j + 1] && k[j] != k[j + 1])
        fix_run(k32, order, k64, M, r, ctl, long_runs, long_cap);
    }
  }
}

// bitonic sort of n (power of two) (key, id) pairs in shared memory
__device__ void bitonic_smem(uint64_t* sk, uint32_t* si, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < n / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const bool gt = key_less(sk[hi], si[hi], sk[lo], si[lo]);
        if (gt == up) {
          const uint64_t tk = sk[lo]; sk[lo] = sk[hi]; sk[hi] = tk;
          const uint32_t ti = si[lo]; si[lo] = si[hi]; si[hi] = ti;
        }
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256)
k_fix_long_runs(const uint32_t* __restrict__ k32, uint32_t* __restrict__ order,
                const uint64_t* __restrict__ k64, const DevStats* __restrict__ stats,
                RunCtl* __restrict__ ctl, const uint32_t* __restrict__ long_runs, uint32_t long_cap,
                uint32_t* __restrict__ scratch /* M ids */) {
  __shared__ uint64_t sk[kSmemSort];
  __shared__ uint32_t si[kSmemSort];
  __shared__ uint32_t s_run;
  __shared__ int s_len;
  const int64_t M = stats->visible;
  const uint32_t n_long = min(ctl->n_long, long_cap);
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_run = atomicAdd(&ctl->ticket, 1u);
    __syncthreads();
    if (s_run >= n_long) return;
    const int64_t r0 = long_runs[s_run];
    const uint32_t k = k32[r0];
    // run length: first index >= r0 whose key differs
    if (threadIdx.x == 0) s_len = 0x7fffffff;
    __syncthreads();
    for (int64_t base = r0; ; base += blockDim.x) {
      const int64_t r = base + threadIdx.x;
      if (r < M && k32[r] != k) atomicMin(&s_len, (int)(r - r0));
      if (r >= M) atomicMin(&s_len, (int)(M - r0));
      __syncthreads();
      const bool found = s_len != 0x7fffffff;
      __syncthreads();
      if (found) break;
    }
    const int L = s_len;
    if (L <= kSmemSort) {
      int n = 1;
      while (n < L) n <<= 1;
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        if (j < L) {
          si[j] = order[r0 + j];
          sk[j] = k64[si[j]];
        } else {
          sk[j] = ~0ull;
          si[j] = 0xffffffffu;
        }
      }
      bitonic_smem(sk, si, n);
      for (int j = threadIdx.x; j < L; j += blockDim.x) order[r0 + j] = si[j];
      continue;
    }
    // L > 2048: sort 2048-blocks in place, then merge block pairs through scratch
    for (int b0 = 0; b0 < L; b0 += kSmemSort) {
      const int nb = min(kSmemSort, L - b0);
      int n = 1;
      while (n < nb) n <<= 1;
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        if (j < nb) {
          si[j] = order[r0 + b0 + j];
          sk[j] = k64[si[j]];
        } else {
          sk[j] = ~0ull;
          si[j] = 0xffffffffu;
        }
      }
      bitonic_smem(sk, si, n);
      for (int j = threadIdx.x; j < nb; j += blockDim.x) order[r0 + b0 + j] = si[j];
      __syncthreads();
    }
    uint32_t* src = order + r0;
    uint32_t* dst = scratch + r0;  // runs are disjoint: each CTA merges in its own window
    for (int w = kSmemSort; w < L; w <<= 1) {
      for (int j = threadIdx.x; j < L; j += blockDim.x) {
        const int blk = j / (2 * w), off = j - blk * 2 * w;
        const int a0 = blk * 2 * w, a1 = min(a0 + w, L), b1 = min(a0 + 2 * w, L);
        const uint32_t id = src[j];
        const uint64_t kk = k64[id];
        // elements of the partner block that precede this one (keys are distinct)
        int lo, hi;
        if (off < w) { lo = a1; hi = b1; } else { lo = a0; hi = a1; }
        const int p0 = lo;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          const uint32_t im = src[mid];
          if (key_less(k64[im], im, kk, id)) lo = mid + 1; else hi = mid;
        }
        const int before = lo - p0;
        const int own = off < w ? off : off - w;
        dst[a0 + own + before] = id;
      }
      __syncthreads();
      uint32_t* t = src; src = dst; dst = t;
    }
    if (src != order + r0)
      for (int j = threadIdx.x; j < L; j += blockDim.x) order[r0 + j] = src[j];
  }
}

void launch_fix_depth_runs(const uint32_t* k32_sorted, uint32_t* order, const uint64_t* k64,
                           const DevStats* stats, int64_t capacity, void* ctl_mem,
                           uint32_t* long_runs, uint32_t long_cap, uint32_t* scratch,
                           cudaStream_t s) {
  RunCtl* ctl = reinterpret_cast<RunCtl*>(ctl_mem);
  cudaMemsetAsync(ctl, 0, sizeof(RunCtl), s);
#ifndef CS_FIX_GRID_MULT
#define CS_FIX_GRID_MULT 8
#endif
  const int grid = (int)std::min<int64_t>(148 * CS_FIX_GRID_MULT, (capacity + 255) / 256 + 1);
  k_fix_short_runs<<<grid, 256, 0, s>>>(k32_sorted, order, k64, stats, ctl, long_runs, long_cap);
  k_fix_long_runs<<<148, 256, 0, s>>>(k32_sorted, order, k64, stats, ctl, long_runs, long_cap,
                                      scratch);
}

size_t fix_ctl_bytes() { return sizeof(RunCtl); }
int64_t fix_long_cap(int64_t capacity) { return capacity / (kShortRun + 1) + 1; }

}  // namespace cs

// cs_lodgen.cu -- K15-K19: offline LoD generation.
//
// Replaces the builder half of citysplat.lod:
//   significance_scores (lod.py:54-101)  K15 k_significance (cs_project.cu: it shares
//                                        the projection's float64 covariance chain),
//                                        K16 volume percentile + k_scores
//   _priority (lod.py:114-116)           stable descending order: 64-bit radix sort of
//                                        the complemented score bits (cs_sort.cu)
//   build_lod level rows (lod.py:222-234) K17 rank scatter + stable block grouping +
//                                        per-level stream compaction
//   mad_bounds (lod.py:130-147)          K18 per-block order statistics through two
//                                        stable sorts (value, then block) per axis
//   GaussianCloud.take +                 K19 row gather into level clouds with the SH
//   with_sh_degree (core.py)             bands above the level's degree dropped
//
// Decision quantities (hit counts, volumes, percentile, ranking, kept rows,
// medians, bounds) are float64 / integer in numpy's op order; the score's
// clamped ** 0.1 uses CUDA's pow (<= 2 ulp from glibc's), which leaves the
// ranking -- and so every kept set -- unchanged unless two distinct scores lie
// within a few ulp (checked against the reference's own outputs in
// tests/golden/lodgen.npz).
#include <cmath>
#include <vector>

#include "cs_internal.cuh"

namespace cs {

void launch_significance(const cs_cloud& cl, const cs_camera* cams, int n_cams,
                         const cs_settings& st, int32_t* hits, uint64_t* vol_keys, uint32_t* vals,
                         cudaStream_t s);

template <typename K>
int radix_sort(K* k0, uint32_t* v0, K* k1, uint32_t* v1, const int64_t* n_dev, int64_t capacity,
               int begin_bit, int end_bit, uint32_t* hist, uint32_t* status, uint32_t* tickets,
               cudaStream_t s, bool hist_ready = false, bool identity_vals = false);

static inline unsigned grid_for(int64_t n, int threads, int cap = 148 * 16) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, cap));
}

// numpy.percentile(..., method="linear") lerp (numpy _lerp): a + (b - a) t, or
// b - (b - a)(1 - t) when t >= 0.5.
__global__ void k_percentile(const uint64_t* __restrict__ sorted, int64_t prev, int64_t next,
                             double gamma, double* __restrict__ out) {
  const double a = __longlong_as_double((long long)sorted[prev]);
  const double b = __longlong_as_double((long long)sorted[next]);
  const double d = dsub(b, a);
  *out = gamma >= 0.5 ? dsub(b, dmul(d, dsub(1.0, gamma))) : dadd(a, dmul(d, gamma));
}

// hits * opacities * minimum(volume, cap) ** 0.1  (lod.py:97-100)
__global__ void k_scores(const cs_cloud cl, const int32_t* __restrict__ hits,
                         const double* __restrict__ cap_p, double* __restrict__ scores) {
  const double cap = *cap_p;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < cl.count;
       k += (int64_t)gridDim.x * blockDim.x) {
    const Geom g = load_geom(cl, k);
    const double vol = dmul(dmul(g.sx, g.sy), g.sz);
    const double cl_v = vol < cap ? vol : cap;  // np.minimum (no NaN here)
    scores[k] = dmul(dmul((double)hits[k], g.op), pow(cl_v, 0.1));
  }
}

// descending score, ties -> lower index: key = ~bits(score) (scores >= 0)
__global__ void k_priority_keys(int64_t n, const double* __restrict__ scores,
                                uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    double v = scores[k];
    if (v == 0.0) v = 0.0;  // -0.0 == 0.0 for argsort(-scores)
    keys[k] = ~(uint64_t)__double_as_longlong(v);
    vals[k] = (uint32_t)k;
  }
}

__global__ void k_rank_scatter(int64_t n, const uint32_t* __restrict__ order,
                               uint32_t* __restrict__ rank) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    rank[order[p]] = (uint32_t)p;
}

__global__ void k_iota_keys(int64_t n, const int32_t* __restrict__ src, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ vals) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    keys[k] = (uint32_t)src[k];
    vals[k] = (uint32_t)k;
  }
}

// ---- stable stream compaction of rows[q] with rank[rows[q]] < keep --------
constexpr int kCompThreads = 256, kCompItems = 8, kCompChunk = kCompThreads * kCompItems;

__global__ void __launch_bounds__(kCompThreads)
k_keep_count(int64_t n, const uint32_t* __restrict__ rows, const uint32_t* __restrict__ rank,
             uint32_t keep, uint32_t* __restrict__ chunk_count) {
  __shared__ uint32_t scratch[kCompThreads / 32 + 1];
  const int64_t base = (int64_t)blockIdx.x * kCompChunk + (int64_t)threadIdx.x * kCompItems;
  uint32_t c = 0;
#pragma unroll
  for (int i = 0; i < kCompItems; ++i)
    if (base + i < n && rank[rows[base + i]] < keep) ++c;
  uint32_t total;
  block_excl_scan<uint32_t>(c, scratch, total);
  if (threadIdx.x == 0) chunk_count[blockIdx.x] = total;
}

// exclusive scan of the chunk counts in place (one CTA)
__global__ void k_scan_counts(int64_t n, uint32_t* __restrict__ v) {
  __shared__ uint32_t scratch[1024 / 32 + 1];
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t b = threadIdx.x * per, e = min(n, b + per);
  uint32_t s = 0;
  for (int64_t i = b; i < e; ++i) s += v[i];
  uint32_t total;
  uint32_t run = block_excl_scan<uint32_t>(s, scratch, total);
  for (int64_t i = b; i < e; ++i) {
    const uint32_t x = v[i];
    v[i] = run;
    run += x;
  }
}

__global__ void __launch_bounds__(kCompThreads)
k_keep_compact(int64_t n, const uint32_t* __restrict__ rows, const uint32_t* __restrict__ rank,
               uint32_t keep, const uint32_t* __restrict__ chunk_off,
               const int32_t* __restrict__ membership, int n_blocks, int32_t* __restrict__ out,
               int64_t* __restrict__ counts) {
  __shared__ uint32_t scratch[kCompThreads / 32 + 1];
  extern __shared__ uint32_t s_hist[];  // n_blocks
  for (int j = threadIdx.x; j < n_blocks; j += blockDim.x) s_hist[j] = 0;
  const int64_t base = (int64_t)blockIdx.x * kCompChunk + (int64_t)threadIdx.x * kCompItems;
  uint32_t flags = 0, c = 0;
#pragma unroll
  for (int i = 0; i < kCompItems; ++i)
    if (base + i < n && rank[rows[base + i]] < keep) {
      flags |= 1u << i;
      ++c;
    }
  uint32_t total;
  uint32_t pos = chunk_off[blockIdx.x] + block_excl_scan<uint32_t>(c, scratch, total);
#pragma unroll
  for (int i = 0; i < kCompItems; ++i)
    if (flags & (1u << i)) {
      const uint32_t r = rows[base + i];
      out[pos++] = (int32_t)r;
      atomicAdd(&s_hist[membership[r]], 1u);
    }
  __syncthreads();
  for (int j = threadIdx.x; j < n_blocks; j += blockDim.x)
    if (s_hist[j]) atomicAdd(reinterpret_cast<unsigned long long*>(&counts[j]), (unsigned long long)s_hist[j]);
}

// ---- mad_bounds ------------------------------------------------------------

__device__ __forceinline__ double pos_axis(const cs_cloud& c, int64_t k, int axis) {
  if (c.fp64) return reinterpret_cast<const double*>(c.pos_op)[4 * k + axis];
  return (double)reinterpret_cast<const float*>(c.pos_op)[4 * k + axis];
}

// IEEE bits -> unsigned order of the value
__device__ __forceinline__ uint64_t ordered_bits(double v) {
  if (v == 0.0) v = 0.0;
  const uint64_t u = (uint64_t)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | (1ull << 63));
}

// mode 0: key = value of axis; mode 1: key = |value - med[block]| (lod.py:142)
__global__ void k_axis_keys(const cs_cloud cl, int axis, int mode, const int32_t* __restrict__ mem,
                            const double* __restrict__ med, uint64_t* __restrict__ keys,
                            uint32_t* __restrict__ vals) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < cl.count;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double p = pos_axis(cl, k, axis);
    const double v = mode == 0 ? p : fabs(dsub(p, med[mem[k]]));
    keys[k] = ordered_bits(v);
    vals[k] = (uint32_t)k;
  }
}

__global__ void k_block_of_rows(int64_t n, const uint32_t* __restrict__ rows,
                                const int32_t* __restrict__ mem, uint32_t* __restrict__ keys,
                                uint32_t* __restrict__ vals) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = rows[q];
    keys[q] = (uint32_t)mem[r];
    vals[q] = r;
  }
}

__device__ __forceinline__ double sorted_val(const cs_cloud& cl, const uint32_t* rows, int64_t q,
                                             int axis, int mode, const int32_t* mem,
                                             const double* med) {
  const int64_t r = rows[q];
  const double p = pos_axis(cl, r, axis);
  return mode == 0 ? p : fabs(dsub(p, med[mem[r]]));
}

// np.median of the block's sorted values (mean of the two middle ones for an
// even count: np.mean -> (a + b) / 2).  mode 0 also records min / max.
__global__ void k_block_median(const cs_cloud cl, int axis, int mode, const uint32_t* __restrict__ rows,
                               const int64_t* __restrict__ off, const int64_t* __restrict__ cnt,
                               int n_blocks, const int32_t* __restrict__ mem,
                               double* __restrict__ med_io, double* __restrict__ mad,
                               double* __restrict__ lo, double* __restrict__ hi) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_blocks) return;
  const int64_t n = cnt[j], o = off[j];
  if (n == 0) {
    if (mode == 0) { med_io[j] = 0.0; lo[j] = 0.0; hi[j] = 0.0; }
    else mad[j] = 0.0;
    return;
  }
  double m;
  if (n & 1) {
    m = sorted_val(cl, rows, o + n / 2, axis, mode, mem, med_io);
  } else {
    const double a = sorted_val(cl, rows, o + n / 2 - 1, axis, mode, mem, med_io);
    const double b = sorted_val(cl, rows, o + n / 2, axis, mode, mem, med_io);
    m = ddiv(dadd(a, b), 2.0);
  }
  if (mode == 0) {
    lo[j] = sorted_val(cl, rows, o, axis, 0, mem, med_io);
    hi[j] = sorted_val(cl, rows, o + n - 1, axis, 0, mem, med_io);
    med_io[j] = m;
  } else {
    mad[j] = m;
  }
}

// lod.py:143-146
__global__ void k_mad_clip(int n_blocks, int axis, double n_mad, const int64_t* __restrict__ cnt,
                           const double* __restrict__ med, const double* __restrict__ mad,
                           const double* __restrict__ lo, const double* __restrict__ hi,
                           double* __restrict__ bmin, double* __restrict__ bmax) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_blocks) return;
  double l = lo[j], h = hi[j];
  if (cnt[j] > 0 && mad[j] > 0.0 && isfinite(n_mad)) {
    const double ml = dsub(med[j], dmul(n_mad, mad[j]));
    const double mh = dadd(med[j], dmul(n_mad, mad[j]));
    l = ml > l ? ml : l;  // max(lo, med - n_mad*mad)
    h = mh < h ? mh : h;  // min(hi, med + n_mad*mad)
  }
  bmin[3 * j + axis] = l;
  bmax[3 * j + axis] = h;
}

__global__ void k_block_hist(int64_t n, const int32_t* __restrict__ mem, int n_blocks,
                             int64_t* __restrict__ cnt) {
  extern __shared__ uint32_t s_hist[];
  for (int j = threadIdx.x; j < n_blocks; j += blockDim.x) s_hist[j] = 0;
  __syncthreads();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&s_hist[mem[k]], 1u);
  __syncthreads();
  for (int j = threadIdx.x; j < n_blocks; j += blockDim.x)
    if (s_hist[j]) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[j]), (unsigned long long)s_hist[j]);
}

// ---- row gather (GaussianCloud.take + with_sh_degree) -----------------------

__global__ void k_gather_quads(int64_t n, const int32_t* __restrict__ rows, const cs_cloud src,
                               cs_cloud dst) {
  const int q = src.fp64 ? 2 : 1;  // 16-byte units per quad
  const int64_t total = n * 3 * q;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (3 * q);
    const int w = (int)(i - r * 3 * q);
    const int arr = w / q, part = w - arr * q;
    const int64_t s = rows[r];
    const float4* sp = reinterpret_cast<const float4*>(arr == 0 ? src.pos_op : arr == 1 ? src.scale : src.quat);
    float4* dp = reinterpret_cast<float4*>(const_cast<void*>(arr == 0 ? dst.pos_op : arr == 1 ? dst.scale : dst.quat));
    dp[r * q + part] = __ldg(sp + s * q + part);
  }
}

__global__ void k_gather_sh(int64_t n, const int32_t* __restrict__ rows, const cs_cloud src,
                            cs_cloud dst) {
  const int Cs = src.sh_coeffs, Cd = dst.sh_coeffs, ds = dst.sh_stride;
  const int64_t total = n * ds;
  float* out = const_cast<float*>(dst.sh);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ds;
    const int e = (int)(i - r * ds);
    float v = 0.f;
    if (e < 3 * Cd) {
      const int ch = e / Cd, m = e - ch * Cd;
      if (m < Cs) v = __ldg(src.sh + (int64_t)rows[r] * src.sh_stride + ch * Cs + m);
    }
    out[i] = v;
  }
}

// ---- host orchestration -------------------------------------------------------

template <typename T>
static cudaError_t dalloc(T** p, size_t n, cudaStream_t s) {
  return cudaMallocAsync(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T), s);
}

size_t radix_status_words(int64_t capacity, int key_bytes);

struct SortWs {
  uint32_t *hist = nullptr, *status = nullptr, *tickets = nullptr;
  int64_t* n_dev = nullptr;
  cudaError_t init(int64_t n, cudaStream_t s) {
    cudaError_t e;
    if ((e = dalloc(&hist, 256 * 8, s))) return e;
    if ((e = dalloc(&status, std::max(radix_status_words(n, 8), radix_status_words(n, 4)), s))) return e;
    if ((e = dalloc(&tickets, 16, s))) return e;
    if ((e = dalloc(&n_dev, 1, s))) return e;
    return cudaMemcpyAsync(n_dev, &n, sizeof(int64_t), cudaMemcpyHostToDevice, s);
  }
  void free(cudaStream_t s) {
    cudaFreeAsync(hist, s); cudaFreeAsync(status, s); cudaFreeAsync(tickets, s); cudaFreeAsync(n_dev, s);
  }
};

static int bits_needed(int64_t n) {
  int b = 1;
  while ((1ll << b) < n) ++b;
  return b;
}

// numpy's linear-method indices for q = 0.9 (numpy _quantile / _get_indexes)
static void percentile_indices(int64_t n, double q, int64_t& prev, int64_t& next, double& gamma) {
  const double vi = (double)(n - 1) * q;
  double p = std::floor(vi);
  gamma = vi - p;
  prev = (int64_t)p;
  next = prev + 1;
  if (vi >= (double)(n - 1)) prev = next = n - 1;
  if (vi < 0.0) prev = next = 0;
}

cudaError_t significance_run(const cs_cloud& cl, const cs_camera* cams_host, int n_cams,
                             const cs_settings& st, double* scores, int32_t* hits_out,
                             cudaStream_t s) {
  const int64_t K = cl.count;
  if (K == 0) return cudaSuccess;
  cs_camera* cams = nullptr;
  int32_t* hits = hits_out;
  uint64_t *k0 = nullptr, *k1 = nullptr;
  uint32_t *v0 = nullptr, *v1 = nullptr;
  double* cap = nullptr;
  SortWs ws;
  cudaError_t e;
  if ((e = dalloc(&cams, n_cams, s))) return e;
  if (!hits_out && (e = dalloc(&hits, K, s))) return e;
  if ((e = dalloc(&k0, K, s)) || (e = dalloc(&k1, K, s)) || (e = dalloc(&v0, K, s)) ||
      (e = dalloc(&v1, K, s)) || (e = dalloc(&cap, 1, s)) || (e = ws.init(K, s)))
    return e;
  if (n_cams > 0 &&
      (e = cudaMemcpyAsync(cams, cams_host, sizeof(cs_camera) * n_cams, cudaMemcpyHostToDevice, s)))
    return e;
  launch_significance(cl, cams, n_cams, st, hits, k0, v0, s);
  const int which = radix_sort<uint64_t>(k0, v0, k1, v1, ws.n_dev, K, 0, 64, ws.hist, ws.status,
                                         ws.tickets, s);
  int64_t prev, next;
  double gamma;
  percentile_indices(K, 90.0 / 100.0, prev, next, gamma);  // VOLUME_PERCENTILE, lod.py:44
  k_percentile<<<1, 1, 0, s>>>(which ? k1 : k0, prev, next, gamma, cap);
  k_scores<<<grid_for(K, 256), 256, 0, s>>>(cl, hits, cap, scores);
  e = cudaGetLastError();
  cudaFreeAsync(cams, s);
  if (!hits_out) cudaFreeAsync(hits, s);
  cudaFreeAsync(k0, s); cudaFreeAsync(k1, s); cudaFreeAsync(v0, s); cudaFreeAsync(v1, s);
  cudaFreeAsync(cap, s);
  ws.free(s);
  return e;
}

cudaError_t priority_run(int64_t K, const double* scores, int32_t* order, cudaStream_t s) {
  if (K == 0) return cudaSuccess;
  uint64_t *k0 = nullptr, *k1 = nullptr;
  uint32_t *v0 = nullptr, *v1 = nullptr;
  SortWs ws;
  cudaError_t e;
  if ((e = dalloc(&k0, K, s)) || (e = dalloc(&k1, K, s)) || (e = dalloc(&v0, K, s)) ||
      (e = dalloc(&v1, K, s)) || (e = ws.init(K, s)))
    return e;
  k_priority_keys<<<grid_for(K, 256), 256, 0, s>>>(K, scores, k0, v0);
  const int which = radix_sort<uint64_t>(k0, v0, k1, v1, ws.n_dev, K, 0, 64, ws.hist, ws.status,
                                         ws.tickets, s);
  e = cudaMemcpyAsync(order, which ? v1 : v0, sizeof(uint32_t) * K, cudaMemcpyDeviceToDevice, s);
  cudaFreeAsync(k0, s); cudaFreeAsync(k1, s); cudaFreeAsync(v0, s); cudaFreeAsync(v1, s);
  ws.free(s);
  return e;
}

cudaError_t lod_rows_run(int64_t K, const int32_t* order, const int32_t* membership, int n_blocks,
                         const int64_t* keep, int n_levels, int32_t* rows_out, int64_t* counts_dev,
                         cudaStream_t s) {
  if (K == 0) return cudaSuccess;
  uint32_t *rank = nullptr, *k0 = nullptr, *k1 = nullptr, *v0 = nullptr, *v1 = nullptr;
  uint32_t* chunk = nullptr;
  SortWs ws;
  cudaError_t e;
  const int64_t chunks = (K + kCompChunk - 1) / kCompChunk;
  if ((e = dalloc(&rank, K, s)) || (e = dalloc(&k0, K, s)) || (e = dalloc(&k1, K, s)) ||
      (e = dalloc(&v0, K, s)) || (e = dalloc(&v1, K, s)) || (e = dalloc(&chunk, chunks, s)) ||
      (e = ws.init(K, s)))
    return e;
  k_rank_scatter<<<grid_for(K, 256), 256, 0, s>>>(K, reinterpret_cast<const uint32_t*>(order), rank);
  // rows grouped by block, ascending index inside each block (stable sort on the block id)
  k_iota_keys<<<grid_for(K, 256), 256, 0, s>>>(K, membership, k0, v0);
  const int which = radix_sort<uint32_t>(k0, v0, k1, v1, ws.n_dev, K, 0, bits_needed(n_blocks),
                                         ws.hist, ws.status, ws.tickets, s);
  const uint32_t* rbb = which ? v1 : v0;
  cudaMemsetAsync(counts_dev, 0, sizeof(int64_t) * n_levels * n_blocks, s);
  for (int L = 0; L < n_levels; ++L) {
    k_keep_count<<<(unsigned)chunks, kCompThreads, 0, s>>>(K, rbb, rank, (uint32_t)keep[L], chunk);
    k_scan_counts<<<1, 1024, 0, s>>>(chunks, chunk);
    k_keep_compact<<<(unsigned)chunks, kCompThreads, sizeof(uint32_t) * n_blocks, s>>>(
        K, rbb, rank, (uint32_t)keep[L], chunk, membership, n_blocks, rows_out + L * K,
        counts_dev + (int64_t)L * n_blocks);
  }
  e = cudaGetLastError();
  cudaFreeAsync(rank, s); cudaFreeAsync(k0, s); cudaFreeAsync(k1, s); cudaFreeAsync(v0, s);
  cudaFreeAsync(v1, s); cudaFreeAsync(chunk, s);
  ws.free(s);
  return e;
}

cudaError_t mad_bounds_run(const cs_cloud& cl, const int32_t* membership, int n_blocks,
                           double n_mad, double* bmin_dev, double* bmax_dev, int64_t* cnt_host,
                           cudaStream_t s) {
  const int64_t K = cl.count;
  uint64_t *k0 = nullptr, *k1 = nullptr;
  uint32_t *v0 = nullptr, *v1 = nullptr, *b0 = nullptr, *b1 = nullptr;
  int64_t *cnt = nullptr, *off = nullptr;
  double *med = nullptr, *mad = nullptr, *lo = nullptr, *hi = nullptr;
  SortWs ws;
  cudaError_t e;
  if ((e = dalloc(&k0, K, s)) || (e = dalloc(&k1, K, s)) || (e = dalloc(&v0, K, s)) ||
      (e = dalloc(&v1, K, s)) || (e = dalloc(&b0, K, s)) || (e = dalloc(&b1, K, s)) ||
      (e = dalloc(&cnt, n_blocks, s)) || (e = dalloc(&off, n_blocks, s)) ||
      (e = dalloc(&med, n_blocks, s)) || (e = dalloc(&mad, n_blocks, s)) ||
      (e = dalloc(&lo, n_blocks, s)) || (e = dalloc(&hi, n_blocks, s)) || (e = ws.init(K, s)))
    return e;
  cudaMemsetAsync(cnt, 0, sizeof(int64_t) * n_blocks, s);
  k_block_hist<<<grid_for(K, 256, 148 * 4), 256, sizeof(uint32_t) * n_blocks, s>>>(K, membership,
                                                                                n_blocks, cnt);
  if ((e = cudaMemcpyAsync(cnt_host, cnt, sizeof(int64_t) * n_blocks, cudaMemcpyDeviceToHost, s)))
    return e;
  if ((e = cudaStreamSynchronize(s))) return e;
  std::vector<int64_t> h_off(n_blocks);
  int64_t acc = 0;
  for (int j = 0; j < n_blocks; ++j) { h_off[j] = acc; acc += cnt_host[j]; }
  cudaMemcpyAsync(off, h_off.data(), sizeof(int64_t) * n_blocks, cudaMemcpyHostToDevice, s);
  const int bb = bits_needed(n_blocks);
  const unsigned jb = (unsigned)((n_blocks + 127) / 128);
  for (int axis = 0; axis < 3; ++axis) {
    for (int mode = 0; mode < 2; ++mode) {
      // stable sort by value (64-bit ordered key), then stable by block:
      // per block, rows in ascending value order
      k_axis_keys<<<grid_for(K, 256), 256, 0, s>>>(cl, axis, mode, membership, med, k0, v0);
      const int w1 = radix_sort<uint64_t>(k0, v0, k1, v1, ws.n_dev, K, 0, 64, ws.hist, ws.status,
                                          ws.tickets, s);
      k_block_of_rows<<<grid_for(K, 256), 256, 0, s>>>(K, w1 ? v1 : v0, membership, b0, b1);
      // b0 = block keys, b1 = rows; sort into (k-buffers reused as u32 scratch)
      uint32_t* sk = reinterpret_cast<uint32_t*>(k0);
      uint32_t* sv = reinterpret_cast<uint32_t*>(k1);
      const int w2 = radix_sort<uint32_t>(b0, b1, sk, sv, ws.n_dev, K, 0, bb, ws.hist, ws.status,
                                          ws.tickets, s);
      const uint32_t* rows = w2 ? sv : b1;
      k_block_median<<<jb, 128, 0, s>>>(cl, axis, mode, rows, off, cnt, n_blocks, membership, med,
                                        mad, lo, hi);
    }
    k_mad_clip<<<jb, 128, 0, s>>>(n_blocks, axis, n_mad, cnt, med, mad, lo, hi, bmin_dev, bmax_dev);
  }
  e = cudaGetLastError();
  cudaFreeAsync(k0, s); cudaFreeAsync(k1, s); cudaFreeAsync(v0, s); cudaFreeAsync(v1, s);
  cudaFreeAsync(b0, s); cudaFreeAsync(b1, s); cudaFreeAsync(cnt, s); cudaFreeAsync(off, s);
  cudaFreeAsync(med, s); cudaFreeAsync(mad, s); cudaFreeAsync(lo, s); cudaFreeAsync(hi, s);
  ws.free(s);
  return e;
}

void launch_gather_cloud(const cs_cloud& src, const int32_t* rows, int64_t n, const cs_cloud& dst,
                         cudaStream_t s) {
  if (n <= 0) return;
  const int q = src.fp64 ? 2 : 1;
  k_gather_quads<<<grid_for(n * 3 * q, 256), 256, 0, s>>>(n, rows, src, dst);
  k_gather_sh<<<grid_for(n * dst.sh_stride, 256), 256, 0, s>>>(n, rows, src, dst);
}

}  // namespace cs

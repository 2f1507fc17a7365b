// cs_fuse.cu -- K12: fusion membership filter.
//
// Replaces the keep mask of partition.fuse (partition.py:570-587):
// normalize_position (partition.py:110-114) -> contract (partition.py:117-126)
// -> block_of_points with lower-inclusive bins over [-2, 2] (partition.py:155-169).
// Float64 in numpy op order; the kept rows are compacted stably (ascending)
// with a decoupled look-back so the fused cloud is byte-identical to the CPU
// fuse() when pieces are concatenated in ascending block order.
#include "cs_internal.cuh"

namespace cs {

struct FuseMap {
  double pmin[3], pmax[3];
  int nx, ny, nz;
};

// contract(normalize_position(p)) (partition.py:110-126), numpy op order
__device__ __forceinline__ void contract_point(double x, double y, double z, const FuseMap& m,
                                               double c[3]) {
  double p[3] = {x, y, z};
  double ph[3];
#pragma unroll
  for (int a = 0; a < 3; ++a)  // 2.0 * (p - p_min) / (p_max - p_min) - 1.0
    ph[a] = dsub(ddiv(dmul(2.0, dsub(p[a], m.pmin[a])), dsub(m.pmax[a], m.pmin[a])), 1.0);
  const double mx = fmax(fmax(fabs(ph[0]), fabs(ph[1])), fabs(ph[2]));
  const double safe = fmax(mx, 1.0);
#pragma unroll
  for (int a = 0; a < 3; ++a)  // identity inside the unit cube, (2 - 1/m) * p / m outside
    c[a] = mx <= 1.0 ? ph[a] : ddiv(dmul(dsub(2.0, ddiv(1.0, safe)), ph[a]), safe);
}

__device__ __forceinline__ int block_of(double x, double y, double z, const FuseMap& m) {
  double c[3];
  contract_point(x, y, z, m, c);
  const int dims[3] = {m.nx, m.ny, m.nz};
  int64_t ib[3];
#pragma unroll
  for (int a = 0; a < 3; ++a)  // _bin: floor((c + 2) / 4 * n), astype(int64), clip
    ib[a] = clip_i64(np_to_i64(floor(dmul(ddiv(dadd(c[a], 2.0), 4.0), (double)dims[a]))), 0,
                     dims[a] - 1);
  if (m.nz <= 1) ib[2] = 0;
  return (int)(ib[0] + (int64_t)m.nx * (ib[1] + (int64_t)m.ny * ib[2]));
}

__device__ __forceinline__ void load_xyz(const void* pos, int f32, int64_t k, double& x, double& y,
                                         double& z, int stride = 3) {
  if (f32) {
    const float* p = reinterpret_cast<const float*>(pos) + stride * k;
    x = p[0]; y = p[1]; z = p[2];
  } else {
    const double* p = reinterpret_cast<const double*>(pos) + stride * k;
    x = p[0]; y = p[1]; z = p[2];
  }
}

// bounds_contain(contract(normalize_position(p)), lo, hi) (partition.py:172-181):
// lower-inclusive, upper-exclusive, an upper bound on the cube surface (== 2)
// inclusive.  mask (optional) per point; count of contained points.
__global__ void k_bounds_contain(int64_t n, const void* pos, int f32, int stride, FuseMap m,
                                 double lo0, double lo1, double lo2, double hi0, double hi1,
                                 double hi2, uint8_t* mask, unsigned long long* count) {
  const double lo[3] = {lo0, lo1, lo2}, hi[3] = {hi0, hi1, hi2};
  unsigned long long local = 0;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += gstride) {
    double x, y, z, c[3];
    load_xyz(pos, f32, k, x, y, z, stride);
    if (m.nx) {
      contract_point(x, y, z, m, c);
    } else {  // points already contracted
      c[0] = x; c[1] = y; c[2] = z;
    }
    bool in = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) in = in && c[a] >= lo[a] && (hi[a] == 2.0 ? c[a] <= hi[a] : c[a] < hi[a]);
    if (mask) mask[k] = in ? 1 : 0;
    local += in ? 1ull : 0ull;
  }
  local = warp_sum(local);
  if (lane_id() == 0 && local) atomicAdd(count, local);
}

__global__ void k_block_of_points(int64_t n, const void* pos, int f32, FuseMap m, int32_t* out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += stride) {
    double x, y, z;
    load_xyz(pos, f32, k, x, y, z);
    out[k] = block_of(x, y, z, m);
  }
}

constexpr int kFuseThreads = 256;
__global__ void __launch_bounds__(kFuseThreads)
k_fuse_filter(int64_t n, const void* pos, int f32, FuseMap m, int block, uint64_t* status,
              uint32_t* ticket, int64_t* kept, int64_t* kept_count) {
  __shared__ int64_t s_chunk;
  __shared__ uint32_t s_scan[kFuseThreads / 32 + 1];
  __shared__ uint64_t s_prefix;
  if (threadIdx.x == 0) s_chunk = atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t chunk = s_chunk;
  const int64_t base = chunk * kFuseThreads;
  if (base >= n) return;
  const int64_t k = base + threadIdx.x;
  bool keep = false;
  if (k < n) {
    double x, y, z;
    load_xyz(pos, f32, k, x, y, z);
    keep = block_of(x, y, z, m) == block;
  }
  uint32_t total;
  const uint32_t excl = block_excl_scan<uint32_t>(keep ? 1u : 0u, s_scan, total);
  if (threadIdx.x < 32) {
    const uint64_t pre = lookback_exclusive(status, chunk, total);
    if (threadIdx.x == 0) {
      s_prefix = pre;
      if (base + kFuseThreads >= n) *kept_count = (int64_t)(pre + total);
    }
  }
  __syncthreads();
  if (keep) kept[s_prefix + excl] = k;
}

void launch_block_of_points(int64_t n, const void* pos, int f32, const double* pmin,
                            const double* pmax, int nx, int ny, int nz, int32_t* out,
                            cudaStream_t s) {
  FuseMap m;
  for (int a = 0; a < 3; ++a) { m.pmin[a] = pmin[a]; m.pmax[a] = pmax[a]; }
  m.nx = nx; m.ny = ny; m.nz = nz;
  if (n > 0) k_block_of_points<<<148 * 8, 256, 0, s>>>(n, pos, f32, m, out);
}

void launch_bounds_contain(int64_t n, const void* pos, int f32, int stride, const double* pmin,
                           const double* pmax, const double* lo, const double* hi, uint8_t* mask,
                           unsigned long long* count, cudaStream_t s) {
  FuseMap m;
  for (int a = 0; a < 3; ++a) { m.pmin[a] = pmin ? pmin[a] : 0.0; m.pmax[a] = pmax ? pmax[a] : 1.0; }
  m.nx = m.ny = m.nz = pmin ? 1 : 0;  // 0: the points are contracted already
  cudaMemsetAsync(count, 0, sizeof(unsigned long long), s);
  if (n > 0)
    k_bounds_contain<<<148 * 8, 256, 0, s>>>(n, pos, f32, stride, m, lo[0], lo[1], lo[2], hi[0], hi[1],
                                             hi[2], mask, count);
}

void launch_fuse_filter(int64_t n, const void* pos, int f32, const double* pmin, const double* pmax,
                        int nx, int ny, int nz, int block, uint64_t* status, uint32_t* ticket,
                        int64_t* kept, int64_t* kept_count, cudaStream_t s) {
  FuseMap m;
  for (int a = 0; a < 3; ++a) { m.pmin[a] = pmin[a]; m.pmax[a] = pmax[a]; }
  m.nx = nx; m.ny = ny; m.nz = nz;
  cudaMemsetAsync(kept_count, 0, sizeof(int64_t), s);
  const int64_t chunks = (n + kFuseThreads - 1) / kFuseThreads;
  if (chunks > 0)
    k_fuse_filter<<<(unsigned)chunks, kFuseThreads, 0, s>>>(n, pos, f32, m, block, status, ticket,
                                                           kept, kept_count);
}

}  // namespace cs

// cs_lod.cu -- K1/K2: block-wise LoD selection and render-set assembly.
//
// Replaces lod.decide_visibility (lod.py:330-348) with block_visible
// (lod.py:267-295), _screen_box (lod.py:298-308) and select_level
// (lod.py:311-321), and assemble_render_set (lod.py:360-401).  Assembly does
// not copy Gaussians: it emits a segment table (level, block, count, start) in
// ascending block order (lod.py:373-377) which the projection kernel walks, so
// the assembled index of every Gaussian equals its position in the
// reference's concatenated cloud (the depth-sort tie-break, render.py:176-177).
//
// Decision math is float64 in numpy order (no FMA), bit-identical to the
// reference; see SURVEY.md Appendix B.
#include "cs_internal.cuh"

namespace cs {


__device__ __forceinline__ double wc(const cs_camera& cam, int row, double x, double y, double z) {
  const double* R = cam.R + 3 * row;
  return dadd(dadd(dadd(dmul(x, R[0]), dmul(y, R[1])), dmul(z, R[2])), cam.t[row]);
}

__device__ __forceinline__ double norm3(double dx, double dy, double dz) {
  return __dsqrt_rn(dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz)));
}

// block_visible (lod.py:267-295) + _screen_box (lod.py:298-308).
__device__ void block_decision(const double* lo, const double* hi, const cs_camera& cam,
                               bool& visible, double& distance, double box[4]) {
  const double* C = cam.center;
  bool inside = true;
#pragma unroll
  for (int a = 0; a < 3; ++a)
    if (!(C[a] >= lo[a] && C[a] <= hi[a])) inside = false;
  double u[8], v[8];
  bool any_behind = false, all_behind = true;
  double dist = __longlong_as_double(0x7ff0000000000000ll);  // +inf
#pragma unroll
  for (int ci = 0; ci < 8; ++ci) {  // corner order x-major, then y, then z (lod.py:282-283)
    const double x = (ci & 4) ? hi[0] : lo[0];
    const double y = (ci & 2) ? hi[1] : lo[1];
    const double z = (ci & 1) ? hi[2] : lo[2];
    const double t0 = wc(cam, 0, x, y, z), t1 = wc(cam, 1, x, y, z), t2 = wc(cam, 2, x, y, z);
    if (t2 <= 0.0) any_behind = true; else all_behind = false;
    u[ci] = dadd(ddiv(dmul(cam.fx, t0), t2), cam.cx);
    v[ci] = dadd(ddiv(dmul(cam.fy, t1), t2), cam.cy);
    const double d = norm3(dsub(x, C[0]), dsub(y, C[1]), dsub(z, C[2]));
    dist = d < dist ? d : dist;
  }
  double umin = u[0], umax = u[0], vmin = v[0], vmax = v[0];
#pragma unroll
  for (int ci = 1; ci < 8; ++ci) {
    umin = fmin(umin, u[ci]); umax = fmax(umax, u[ci]);
    vmin = fmin(vmin, v[ci]); vmax = fmax(vmax, v[ci]);
  }
  if (inside) {
    visible = true;
    distance = 0.0;
  } else {
    distance = dist;
    if (all_behind) visible = false;
    else if (any_behind) visible = true;
    else visible = umax >= 0.0 && umin <= (double)cam.width && vmax >= 0.0 &&
                   vmin <= (double)cam.height;
  }
  if (any_behind) {
    box[0] = 0.0; box[1] = 0.0; box[2] = (double)cam.width; box[3] = (double)cam.height;
  } else {
    box[0] = umin; box[1] = vmin; box[2] = umax; box[3] = vmax;
  }
}

// select_level (lod.py:311-321): first interval with lo <= d < hi -> n-1-i.
__device__ __forceinline__ int select_level_dev(double d, const double* iv, int n) {
  for (int i = 0; i < n; ++i)
    if (iv[2 * i] <= d && d < iv[2 * i + 1]) return n - 1 - i;
  return -1;
}

// One CTA: the block decisions, 256 blocks at a time, and the ascending-block
// segment table from two block scans (pieces kept, rows) -- no serial walk
// over the decisions (that walk, one thread re-reading every decision and
// piece count, was most of this kernel's 21 us).
__global__ void __launch_bounds__(256) k_lod_select(LodTables T, cs_camera cam, int force_level,
                                                    cs_decision* __restrict__ dec, Seg* __restrict__ segs,
                                                    DevStats* __restrict__ stats) {
  __shared__ unsigned int s_scan_n[9];
  __shared__ unsigned long long s_scan_c[9];
  const int J = T.n_blocks;
  unsigned int n_base = 0;
  unsigned long long start_base = 0;
  for (int j0 = 0; j0 < J; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    unsigned int keep = 0;
    unsigned long long cnt = 0;
    int ci = 0;
    if (j < J) {
      cs_decision d;
      d.level = -1;
      d.visible = 0;
      d.has_box = 0;
      d.pad[0] = d.pad[1] = 0;
      d.box[0] = d.box[1] = d.box[2] = d.box[3] = 0.0;
      if (!T.occupied[j]) {  // lod.py:334-336
        d.distance = __longlong_as_double(0x7ff0000000000000ll);
      } else {
        bool vis;
        double dist, box[4];
        block_decision(T.bmin + 3 * j, T.bmax + 3 * j, cam, vis, dist, box);
        d.distance = dist;
        if (vis) {
          d.visible = 1;
          d.has_box = 1;
          for (int a = 0; a < 4; ++a) d.box[a] = box[a];
          if (force_level >= 0) {
            d.level = force_level;  // lod.py:342-345
          } else {
            d.level = select_level_dev(dist, T.intervals, T.n_levels);
            if (d.level < 0) atomicOr(&stats->status, 2);  // ValueError in select_level
          }
        }
      }
      dec[j] = d;
      if (d.visible && d.level >= 0 && d.level < T.n_levels) {
        ci = d.level * J + j;
        cnt = (unsigned long long)T.clouds[ci].count;
        keep = cnt > 0 ? 1u : 0u;  // empty pieces dropped (lod.py:375-377)
      }
    }
    unsigned int n_tot;
    unsigned long long c_tot;
    const unsigned int pos = block_excl_scan<unsigned int>(keep, s_scan_n, n_tot);
    const unsigned long long off = block_excl_scan<unsigned long long>(keep ? cnt : 0ull, s_scan_c, c_tot);
    if (keep) {  // ascending block order = concatenation order (lod.py:373-377)
      Seg& sg = segs[n_base + pos];
      sg.start = (int64_t)(start_base + off);
      sg.count = (int64_t)cnt;
      sg.cloud = ci;
      sg.pad = 0;
    }
    n_base += n_tot;
    start_base += c_tot;
  }
  if (threadIdx.x == 0) {
    stats->n_segs = (int)n_base;
    stats->assembled = (int64_t)start_base;
  }
}

// Pointwise ablation (lod.py:378-390): stable compaction over all levels'
// Gaussians (level-major, then block) of those whose own camera distance
// selects the wanted level.  Emits packed (cloud << 40 | local) entries.
constexpr int kPwThreads = 256;
__global__ void __launch_bounds__(kPwThreads)
k_pointwise(LodTables T, cs_camera cam, int force_level, uint64_t* __restrict__ status,
            uint64_t* __restrict__ list, DevStats* __restrict__ stats) {
  __shared__ int64_t s_chunk;
  __shared__ uint32_t s_scan[kPwThreads / 32 + 1];
  __shared__ uint64_t s_prefix;
  if (threadIdx.x == 0) s_chunk = atomicAdd(&stats->tickets[1], 1u);
  __syncthreads();
  const int64_t chunk = s_chunk;
  const int64_t n = T.total_all;
  const int64_t base = chunk * kPwThreads;
  if (base >= n) return;
  const int64_t i = base + threadIdx.x;
  bool keep = false;
  int ci = 0;
  int64_t local = 0;
  if (i < n) {
    const int si = find_seg(T.all_segs, T.n_levels * T.n_blocks, i);
    const Seg sg = T.all_segs[si];
    ci = sg.cloud;
    local = i - sg.start;
    const int level = ci / T.n_blocks;
    const int want = force_level >= 0 ? force_level : level;
    if (level == want) {
      double x, y, z;
      load_pos(T.clouds[ci], local, x, y, z);
      const double d = norm3(dsub(x, cam.center[0]), dsub(y, cam.center[1]), dsub(z, cam.center[2]));
      int cnt = 0;  // searchsorted(los, d, side="right")
      for (int k = 0; k < T.n_levels; ++k) cnt += (T.intervals[2 * k] <= d) ? 1 : 0;
      keep = (T.n_levels - 1 - (cnt - 1)) == want;  // _select_levels, lod.py:324-327
    }
  }
  uint32_t total;
  uint32_t excl = block_excl_scan<uint32_t>(keep ? 1u : 0u, s_scan, total);
  if (threadIdx.x < 32) {
    uint64_t pre = lookback_exclusive(status, chunk, total);
    if (threadIdx.x == 0) {
      s_prefix = pre;
      if (base + kPwThreads >= n) stats->assembled = (int64_t)(pre + total);
    }
  }
  __syncthreads();
  if (keep) list[s_prefix + excl] = ((uint64_t)ci << 40) | (uint64_t)local;
}

// Segment table for list mode: one pseudo-segment; the projection resolves
// (cloud, local) through the list.
__global__ void k_pointwise_finish(Seg* segs, DevStats* stats) {
  segs[0].start = 0;
  segs[0].count = stats->assembled;
  segs[0].cloud = -1;
  segs[0].pad = 0;
  stats->n_segs = 1;
}

// Batch block_visible for the Python API (lod.py:267-295).
__global__ void k_block_visible(int n, const double* bmin, const double* bmax, cs_camera cam,
                                uint8_t* vis, double* dist) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  bool v;
  double d, box[4];
  block_decision(bmin + 3 * j, bmax + 3 * j, cam, v, d, box);
  vis[j] = v;
  dist[j] = d;
}

// Batch select_level (lod.py:311-321).  level -1: no interval, -2: negative.
__global__ void k_select_level(int n, const double* d, int ni, const double* iv, int32_t* out) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double x = d[j];
  out[j] = x < 0.0 ? -2 : select_level_dev(x, iv, ni);
}

const void* lod_select_kernel() { return reinterpret_cast<const void*>(&k_lod_select); }

void launch_lod_select(const LodTables& T, const cs_camera& cam, int force_level,
                       cs_decision* dec, Seg* segs, DevStats* stats, cudaStream_t s) {
  k_lod_select<<<1, 256, 0, s>>>(T, cam, force_level, dec, segs, stats);
}
void launch_pointwise(const LodTables& T, const cs_camera& cam, int force_level, uint64_t* status,
                      uint64_t* list, Seg* segs, DevStats* stats, cudaStream_t s) {
  const int64_t chunks = (T.total_all + kPwThreads - 1) / kPwThreads;
  if (chunks > 0)
    k_pointwise<<<(unsigned)chunks, kPwThreads, 0, s>>>(T, cam, force_level, status, list, stats);
  k_pointwise_finish<<<1, 1, 0, s>>>(segs, stats);
}
void launch_block_visible(int n, const double* bmin, const double* bmax, const cs_camera& cam,
                          uint8_t* vis, double* dist, cudaStream_t s) {
  if (n > 0) k_block_visible<<<(n + 127) / 128, 128, 0, s>>>(n, bmin, bmax, cam, vis, dist);
}
void launch_select_level(int n, const double* d, int ni, const double* iv, int32_t* out,
                         cudaStream_t s) {
  if (n > 0) k_select_level<<<(n + 127) / 128, 128, 0, s>>>(n, d, ni, iv, out);
}

}  // namespace cs

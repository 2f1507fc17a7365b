// cs_bin.cu -- K5/K6/K8: depth-rank gather, tile-count scan, pair
// duplication and tile ranges.  Replaces render._bin_tiles (render.py:217-249)
// together with the depth-order gather at the end of _project_cloud
// (render.py:178-188).
#include "cs_internal.cuh"

namespace cs {

constexpr int kGatherThreads = 256;

// For every depth rank r (0..M-1): gather the projected record of the r-th
// splat in depth order, compute its tile rectangle exactly as numpy does
// (render.py:226-231, astype(int64) then clip), emit the blend records and
// scan the pair counts (render.py:233-236) with a decoupled look-back.
__global__ void __launch_bounds__(kGatherThreads)
k_gather_count(const uint32_t* __restrict__ order, const ProjRec* __restrict__ recs,
               DevStats* __restrict__ stats, int tile_size, int width, int height,
               double alpha_floor, int64_t pair_cap, uint64_t* __restrict__ status,
               HotRec* __restrict__ hot, ColdRec* __restrict__ cold, int4* __restrict__ rects,
               int64_t* __restrict__ src_sorted, int64_t* __restrict__ pair_off) {
  __shared__ int64_t s_chunk;
  __shared__ uint64_t s_scan[kGatherThreads / 32 + 1];
  __shared__ uint64_t s_prefix;
  const int64_t M = stats->visible;
  if (threadIdx.x == 0) s_chunk = atomicAdd(&stats->tickets[2], 1u);
  __syncthreads();
  const int64_t chunk = s_chunk;
  const int64_t base = chunk * kGatherThreads;
  if (base >= M) return;
  const int64_t r = base + threadIdx.x;
  uint64_t cnt = 0;
  int4 rect = make_int4(0, 0, 0, 0);
  if (r < M) {
    const ProjRec rec = recs[order[r]];
    const int64_t ntx = (width + tile_size - 1) / tile_size;
    const int64_t nty = (height + tile_size - 1) / tile_size;
    const double ts = (double)tile_size;
    const int64_t tx0 = clip_i64(np_to_i64(floor(ddiv(dsub(dsub(rec.mx, rec.rx), 0.5), ts))), 0, ntx - 1);
    const int64_t tx1 = clip_i64(np_to_i64(floor(ddiv(dsub(dadd(rec.mx, rec.rx), 0.5), ts))), 0, ntx - 1);
    const int64_t ty0 = clip_i64(np_to_i64(floor(ddiv(dsub(dsub(rec.my, rec.ry), 0.5), ts))), 0, nty - 1);
    const int64_t ty1 = clip_i64(np_to_i64(floor(ddiv(dsub(dadd(rec.my, rec.ry), 0.5), ts))), 0, nty - 1);
    rect = make_int4((int)tx0, (int)tx1, (int)ty0, (int)ty1);
    cnt = (uint64_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
    HotRec h;
    h.mx = rec.mx; h.my = rec.my; h.c0 = rec.c0; h.c1 = rec.c1; h.c2 = rec.c2;
    // fast-reject threshold: alpha = o*exp(power) < alpha_floor whenever
    // power < log(alpha_floor/o) - 1e-6 (margin >> exp/log rounding).
    const double lt = rec.opacity > 0.0 ? log(alpha_floor / rec.opacity) - 1e-6
                                        : __longlong_as_double(0x7ff0000000000000ll);
    h.lthr = __double2float_rd(lt);
    h.rank = (uint32_t)r;
    hot[r] = h;
    ColdRec c;
    c.opacity = rec.opacity;
    c.r = rec.r; c.g = rec.g; c.b = rec.bl; c.pad = 0.f; c.pad2 = 0.0;
    cold[r] = c;
    rects[r] = rect;
    src_sorted[r] = rec.src;
  }
  uint64_t total;
  const uint64_t excl = block_excl_scan<uint64_t>(cnt, s_scan, total);
  if (threadIdx.x < 32) {
    const uint64_t pre = lookback_exclusive(status, chunk, total);
    if (threadIdx.x == 0) {
      s_prefix = pre;
      if (base + kGatherThreads >= M) {
        const int64_t P = (int64_t)(pre + total);
        stats->pairs = P;
        stats->pairs_eff = P <= pair_cap ? P : 0;
        if (P > pair_cap) atomicOr(&stats->status, 1);
      }
    }
  }
  __syncthreads();
  if (r < M) pair_off[r] = (int64_t)(s_prefix + excl);
}

constexpr int kDupThreads = 256;
constexpr int kDupTile = 1024;

// Load-balanced duplication (render.py:233-243): each CTA owns kDupTile
// consecutive output pairs; the splats whose pair ranges intersect it are
// found by binary search and staged in shared memory.  Pairs are emitted
// row-major over each rect in depth-rank order: key = tile id, value = rank.
__global__ void __launch_bounds__(kDupThreads)
k_duplicate(const int64_t* __restrict__ pair_off, const int4* __restrict__ rects,
            const DevStats* __restrict__ stats, int ntx, uint32_t* __restrict__ keys,
            uint32_t* __restrict__ vals) {
  __shared__ int64_t s_off[kDupTile + 1];
  __shared__ int4 s_rect[kDupTile + 1];
  __shared__ int64_t s_rlo, s_rhi;
  const int64_t P = stats->pairs_eff;
  const int64_t M = stats->visible;
  const int64_t p0 = (int64_t)blockIdx.x * kDupTile;
  if (p0 >= P) return;
  const int64_t p1 = min(p0 + kDupTile, P);
  if (threadIdx.x < 2) {
    const int64_t target = threadIdx.x == 0 ? p0 : p1 - 1;
    int64_t lo = 0, hi = M - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (pair_off[mid] <= target) lo = mid; else hi = mid - 1;
    }
    if (threadIdx.x == 0) s_rlo = lo; else s_rhi = lo;
  }
  __syncthreads();
  const int64_t rlo = s_rlo;
  const int nr = (int)(s_rhi - rlo + 1);
  for (int i = threadIdx.x; i < nr; i += kDupThreads) {
    s_off[i] = pair_off[rlo + i];
    s_rect[i] = rects[rlo + i];
  }
  __syncthreads();
  for (int64_t p = p0 + threadIdx.x; p < p1; p += kDupThreads) {
    int lo = 0, hi = nr - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= p) lo = mid; else hi = mid - 1;
    }
    const int4 rc = s_rect[lo];
    const int64_t local = p - s_off[lo];
    const int w = rc.y - rc.x + 1;
    const int ly = (int)(local / w), lx = (int)(local - (int64_t)ly * w);
    keys[p] = (uint32_t)((rc.z + ly) * ntx + (rc.x + lx));
    vals[p] = (uint32_t)(rlo + lo);
  }
}

// CSR tile ranges from the tile-sorted keys (render.py:247-248).
__global__ void k_tile_ranges(const uint32_t* __restrict__ keys, const DevStats* __restrict__ stats,
                              uint2* __restrict__ ranges) {
  const int64_t P = stats->pairs_eff;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P; p += stride) {
    const uint32_t t = keys[p];
    if (p == 0 || keys[p - 1] != t) ranges[t].x = (uint32_t)p;
    if (p == P - 1 || keys[p + 1] != t) ranges[t].y = (uint32_t)(p + 1);
  }
}

void launch_gather_count(const uint32_t* order, const ProjRec* recs, DevStats* stats,
                         int tile_size, int width, int height, double alpha_floor,
                         int64_t pair_cap, int64_t capacity, uint64_t* status, HotRec* hot,
                         ColdRec* cold, int4* rects, int64_t* src_sorted, int64_t* pair_off,
                         cudaStream_t s) {
  const int64_t chunks = (capacity + kGatherThreads - 1) / kGatherThreads;
  if (chunks == 0) return;
  k_gather_count<<<(unsigned)chunks, kGatherThreads, 0, s>>>(order, recs, stats, tile_size, width,
                                                             height, alpha_floor, pair_cap, status,
                                                             hot, cold, rects, src_sorted, pair_off);
}

void launch_duplicate(const int64_t* pair_off, const int4* rects, const DevStats* stats, int ntx,
                      int64_t pair_cap, uint32_t* keys, uint32_t* vals, cudaStream_t s) {
  const int64_t blocks = (pair_cap + kDupTile - 1) / kDupTile;
  if (blocks == 0) return;
  k_duplicate<<<(unsigned)blocks, kDupThreads, 0, s>>>(pair_off, rects, stats, ntx, keys, vals);
}

void launch_tile_ranges(const uint32_t* keys, const DevStats* stats, uint2* ranges,
                        cudaStream_t s) {
  k_tile_ranges<<<148 * 8, 256, 0, s>>>(keys, stats, ranges);
}

// ---------------------------------------------------------------------------
// dumps (golden-intermediate comparison; not on the timed path)

__global__ void k_dump_projected(const uint32_t* order, const ProjRec* recs,
                                 const DevStats* stats, double* means, double* conics,
                                 double* covs, double* depths, double* colors, double* opac,
                                 double* radii, int64_t* src) {
  const int64_t M = stats->visible;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < M;
       r += (int64_t)gridDim.x * blockDim.x) {
    const ProjRec p = recs[order[r]];
    means[2 * r] = p.mx; means[2 * r + 1] = p.my;
    conics[3 * r] = p.c0; conics[3 * r + 1] = p.c1; conics[3 * r + 2] = p.c2;
    covs[3 * r] = p.a; covs[3 * r + 1] = p.b; covs[3 * r + 2] = p.c;
    depths[r] = p.depth;
    colors[3 * r] = p.r; colors[3 * r + 1] = p.g; colors[3 * r + 2] = p.bl;
    opac[r] = p.opacity;
    radii[2 * r] = p.rx; radii[2 * r + 1] = p.ry;
    src[r] = p.src;
  }
}

__global__ void k_dump_tiles(const uint32_t* vals, const uint2* ranges, const DevStats* stats,
                             int n_tiles, int64_t* tile_ids, int64_t* offsets) {
  const int64_t P = stats->pairs_eff;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P; p += stride)
    tile_ids[p] = vals[p];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= n_tiles; t += stride) {
    // offsets[t] = start of tile t; empty tiles take the next non-empty start
    if (t == n_tiles) { offsets[t] = P; continue; }
    int64_t tt = t;
    while (tt < n_tiles && ranges[tt].y == ranges[tt].x) ++tt;
    offsets[t] = tt < n_tiles ? (int64_t)ranges[tt].x : P;
  }
}

void launch_dump_projected(const uint32_t* order, const ProjRec* recs, const DevStats* stats,
                           double* means, double* conics, double* covs, double* depths,
                           double* colors, double* opac, double* radii, int64_t* src,
                           cudaStream_t s) {
  k_dump_projected<<<148 * 4, 256, 0, s>>>(order, recs, stats, means, conics, covs, depths,
                                           colors, opac, radii, src);
}
void launch_dump_tiles(const uint32_t* vals, const uint2* ranges, const DevStats* stats,
                       int n_tiles, int64_t* tile_ids, int64_t* offsets, cudaStream_t s) {
  k_dump_tiles<<<148 * 4, 256, 0, s>>>(vals, ranges, stats, n_tiles, tile_ids, offsets);
}

}  // namespace cs

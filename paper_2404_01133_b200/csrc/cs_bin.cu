// cs_bin.cu -- K5/K6 (fused) and K8: pair counts in depth order, pair
// duplication and tile ranges.  Replaces render._bin_tiles (render.py:217-249).
//
// The tile rectangles were computed by the projection (render.py:226-231);
// here only the depth permutation is applied: pairs are emitted in depth-rank
// order (row-major over each rect, render.py:233-243) carrying the splat's
// compact index, so after the stable tile sort every tile's list is in
// (depth, assembled index) order (render.py:245) and the blend reads the
// splat records directly by compact index -- no gather pass.
#include "cs_internal.cuh"

namespace cs {

// Each thread emits 4 consecutive pairs: one binary search in shared memory for
// its first pair's rank, then a sequential walk over the rect row-major
// (render.py:233-243) and on to the next rank, and two 16-byte stores.
// key = tile id, value = splat id.
constexpr int kDupItems = 4;
constexpr int kMaxHistPasses = 3;

// Digit histograms of the tile sort that follows (equal-width digits, as
// radix_sort_items splits end_bit): counted here from the pair keys.
struct DigitHist {
  uint32_t* hist;  // [n_passes][256], zeroed by the caller
  int n_passes, width, end_bit;
};

__device__ __forceinline__ void emit_pairs(uint32_t p, uint32_t p1, int nr, const uint32_t* s_off,
                                           const uint2* s_rect, const uint32_t* s_id, int ntx,
                                           uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                           const DigitHist& dh, uint32_t (*s_hist)[256],
                                           uint64_t out_base = 0) {
  // 32-bit throughout: pairs < 2^30 (pair_cap), a rank owns <= n_tiles pairs
  int lo = 0, hi = nr - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_off[mid] <= p) lo = mid; else hi = mid - 1;
  }
  int4 rc = unpack_rect(s_rect[lo]);
  int w = rc.y - rc.x + 1;
  const int local = (int)(p - s_off[lo]);
  int ly = local / w, lx = local - ly * w;
  uint32_t next = s_off[lo + 1];  // sentinel 0xffffffff beyond the last rank
  uint32_t k[kDupItems], v[kDupItems];
#pragma unroll
  for (int j = 0; j < kDupItems; ++j) {
    k[j] = (uint32_t)((rc.z + ly) * ntx + (rc.x + lx));
    v[j] = s_id[lo];
    if (p + j + 1 == next) {  // next rank starts at its first tile
      ++lo;
      rc = unpack_rect(s_rect[lo]);
      w = rc.y - rc.x + 1;
      lx = ly = 0;
      next = s_off[lo + 1];
    } else if (++lx == w) {
      lx = 0;
      ++ly;
    }
  }
  const uint64_t o = out_base + p;
  if (p + kDupItems <= p1 && (o & 3) == 0) {
    *reinterpret_cast<uint4*>(keys + o) = make_uint4(k[0], k[1], k[2], k[3]);
    *reinterpret_cast<uint4*>(vals + o) = make_uint4(v[0], v[1], v[2], v[3]);
  } else {
#pragma unroll
    for (int j = 0; j < kDupItems; ++j)
      if (p + j < p1) { keys[o + j] = k[j]; vals[o + j] = v[j]; }
  }
#pragma unroll
  for (int j = 0; j < kDupItems; ++j)
    if (p + j < p1)
      for (int q = 0; q < dh.n_passes; ++q)
        atomicAdd(&s_hist[q][(k[j] >> (dh.width * q)) & ((1u << min(dh.width, dh.end_bit - dh.width * q)) - 1u)], 1u);
}

// K5+K6 fused: per chunk of 2048 depth ranks (warp-striped, coalesced), the
// tile rectangles are gathered once into shared memory, the pair counts
// scanned (block scan + decoupled look-back across chunks), and the chunk's
// pairs emitted right away -- four per thread, owner rank by binary search in
// shared memory, row-major over each rect (render.py:233-243) -- together
// with the tile sort's digit histograms.  emit = false (projection-only
// renders) stops after the count.
//
// A chunk of near, large splats can own far more pairs than the average
// (a top-down or close-up view: one chunk with 10^5-10^6 pairs), and one CTA
// emitting them would be the kernel's tail.  Chunks above kBinHeavy pairs are
// therefore only registered (chunk, first slice, prefix, total) and their
// pairs emitted by k_emit_heavy in kBinSlice-pair slices spread over the
// whole GPU.  The output is the same: every pair lands at prefix + local.
constexpr int kBinThreads = 256;
#ifndef CS_BIN_ITEMS
#define CS_BIN_ITEMS 8
#endif
constexpr int kBinItems = CS_BIN_ITEMS;
constexpr int kBinRanks = kBinThreads * kBinItems;
#ifndef CS_BIN_HEAVY
#define CS_BIN_HEAVY 32768
#endif
#ifndef CS_BIN_SLICE
#define CS_BIN_SLICE 8192
#endif
constexpr uint32_t kBinHeavy = CS_BIN_HEAVY;
constexpr uint32_t kBinSlice = CS_BIN_SLICE;
constexpr int kHeavyCtas = 148 * 4;

struct BinSmem {
  uint32_t off[kBinRanks + 1];
  uint2 rect[kBinRanks];
  uint32_t id[kBinRanks];
  uint32_t hist[kMaxHistPasses][256];
  uint32_t scan[kBinThreads / 32 + 1];
};

// Gathers chunk [base, base + nr) of the depth order into shared memory and
// writes each rank's exclusive pair offset inside the chunk (off[nr] = the
// 0xffffffff sentinel: every rank owns >= 1 pair).  Returns the chunk total.
__device__ __forceinline__ uint32_t gather_chunk(const uint32_t* __restrict__ order,
                                                 const uint2* __restrict__ rects, int64_t base,
                                                 int nr, BinSmem& sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t cnt[kBinItems], run = 0;
#pragma unroll
  for (int i = 0; i < kBinItems; ++i) {
    const int li = warp * (32 * kBinItems) + i * 32 + lane;  // chunk-local rank
    uint32_t c = 0;
    if (li < nr) {
      const uint32_t id = __ldg(order + base + li);
      const uint2 pr = __ldg(rects + id);
      const int4 rc = unpack_rect(pr);
      sm.rect[li] = pr;
      sm.id[li] = id;
      c = (uint32_t)((rc.y - rc.x + 1) * (rc.w - rc.z + 1));
    }
    const uint32_t incl = warp_incl_scan(c);
    cnt[i] = run + incl - c;  // exclusive offset inside the warp's 256 ranks
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) sm.scan[warp] = run;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < kBinThreads / 32 ? sm.scan[lane] : 0u;
    const uint32_t wi = warp_incl_scan(w);
    if (lane < kBinThreads / 32) sm.scan[lane] = wi - w;
    if (lane == 31) sm.scan[kBinThreads / 32] = wi;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kBinItems; ++i) {
    const int li = warp * (32 * kBinItems) + i * 32 + lane;
    if (li < nr) sm.off[li] = sm.scan[warp] + cnt[i];
  }
  if (threadIdx.x == 0) sm.off[nr] = 0xffffffffu;
  return sm.scan[kBinThreads / 32];  // <= 2048 x 2^16 pairs
}

__device__ __forceinline__ void flush_hist(const DigitHist& dh, BinSmem& sm) {
  for (int i = threadIdx.x; i < dh.n_passes * 256; i += kBinThreads) {
    const uint32_t c = sm.hist[i >> 8][i & 255];
    if (c) atomicAdd(dh.hist + i, c);
  }
}

#ifndef CS_BIN_PERSIST
#define CS_BIN_PERSIST 1
#endif

__global__ void __launch_bounds__(kBinThreads)
k_bin_pairs(const uint32_t* __restrict__ order, const uint2* __restrict__ rects,
            DevStats* __restrict__ stats, int64_t pair_cap, uint64_t* __restrict__ status,
            uint4* __restrict__ heavy, int ntx, uint32_t* __restrict__ keys,
            uint32_t* __restrict__ vals, DigitHist dh, int emit, int64_t* host_overflow) {
  __shared__ BinSmem sm;
  __shared__ uint64_t s_prefix;
  __shared__ uint32_t s_chunk;
  const int64_t M = stats->visible;
  for (int i = threadIdx.x; i < dh.n_passes * 256; i += kBinThreads) sm.hist[i >> 8][i & 255] = 0;
  // CS_BIN_PERSIST: one wave of CTAs looping over chunk tickets (the grid is
  // not sized by the visible capacity); digit counts flushed once per CTA
  while (true) {
    if (threadIdx.x == 0) s_chunk = atomicAdd(&stats->tickets[2], 1u);
    __syncthreads();
    const int64_t chunk = s_chunk;
    const int64_t base = chunk * kBinRanks;
    if (base >= M) break;
    const int nr = (int)min((int64_t)kBinRanks, M - base);
    const uint32_t total = gather_chunk(order, rects, base, nr, sm);
    if (threadIdx.x < 32) {
      const uint64_t pre = lookback_exclusive(status, chunk, total);
      if (threadIdx.x == 0) {
        s_prefix = pre;
        if (base + kBinRanks >= M) {
          const int64_t P = (int64_t)(pre + total);
          stats->pairs = P;
          stats->pairs_eff = P <= pair_cap ? P : 0;
          if (P > pair_cap) {
            atomicOr(&stats->status, 1);
            // report to the host (mapped pinned memory): an asynchronous frame
            // that overflowed is raised by the context's next call
            if (emit && host_overflow) {
              volatile int64_t* h = host_overflow;
              h[1] = pair_cap;
              h[0] = P;
              __threadfence_system();
            }
          }
        }
        if (emit && total > kBinHeavy && pre + total <= (uint64_t)pair_cap) {
          // register the chunk: entry index and first slice from one 64-bit
          // atomic, so entries are ordered by first slice
          const uint32_t ns = (total + kBinSlice - 1) / kBinSlice;
          const unsigned long long old = atomicAdd(
              reinterpret_cast<unsigned long long*>(&stats->tickets[8]), (1ull << 32) | ns);
          heavy[old >> 32] = make_uint4((uint32_t)chunk, (uint32_t)old, (uint32_t)pre, total);
        }
      }
    }
    __syncthreads();
    const uint64_t prefix = s_prefix;
    // overflow: the SYNC path re-renders; heavy chunks: k_emit_heavy's
    if (emit && prefix + total <= (uint64_t)pair_cap && total <= kBinHeavy)
      for (uint32_t q = threadIdx.x * kDupItems; q < total; q += kBinThreads * kDupItems)
        emit_pairs(q, total, nr, sm.off, sm.rect, sm.id, ntx, keys, vals, dh, sm.hist, prefix);
    if (!CS_BIN_PERSIST) break;
    __syncthreads();  // shared arrays are reused by the next chunk
  }
  __syncthreads();
  flush_hist(dh, sm);
}

// Pairs of the registered heavy chunks, one kBinSlice slice per ticket; a CTA
// re-gathers a chunk's offsets only when its slice moves to another chunk.
__global__ void __launch_bounds__(kBinThreads)
k_emit_heavy(const uint32_t* __restrict__ order, const uint2* __restrict__ rects,
             DevStats* __restrict__ stats, const uint4* __restrict__ heavy, int ntx,
             uint32_t* __restrict__ keys, uint32_t* __restrict__ vals, DigitHist dh) {
  __shared__ BinSmem sm;
  __shared__ uint32_t s_t[2];  // double-buffered ticket: thread 0 writes the next while others read this one
  const unsigned long long hc = *reinterpret_cast<const unsigned long long*>(&stats->tickets[8]);
  const uint32_t n_entries = (uint32_t)(hc >> 32), n_slices = (uint32_t)hc;
  if (n_slices == 0) return;
  const int64_t M = stats->visible;
  for (int i = threadIdx.x; i < dh.n_passes * 256; i += kBinThreads) sm.hist[i >> 8][i & 255] = 0;
  int64_t cur = -1;
  int nr = 0;
  for (uint32_t it = 0;; ++it) {
    if (threadIdx.x == 0) s_t[it & 1] = atomicAdd(&stats->tickets[10], 1u);
    __syncthreads();
    const uint32_t t = s_t[it & 1];
    if (t >= n_slices) break;
    int lo = 0, hi = (int)n_entries - 1;  // last entry whose first slice <= t
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(&heavy[mid].y) <= t) lo = mid; else hi = mid - 1;
    }
    const uint4 e = __ldg(heavy + lo);
    if ((int64_t)e.x != cur) {
      __syncthreads();  // the previous chunk's shared arrays are no longer read
      cur = e.x;
      const int64_t base = cur * kBinRanks;
      nr = (int)min((int64_t)kBinRanks, M - base);
      gather_chunk(order, rects, base, nr, sm);
      __syncthreads();
    }
    const uint32_t q0 = (t - e.y) * kBinSlice, q1 = min(e.w, q0 + kBinSlice);
    for (uint32_t q = q0 + threadIdx.x * kDupItems; q < q1; q += kBinThreads * kDupItems)
      emit_pairs(q, q1, nr, sm.off, sm.rect, sm.id, ntx, keys, vals, dh, sm.hist, e.z);
  }
  __syncthreads();
  flush_hist(dh, sm);
}

// CSR tile ranges from the tile-sorted keys (render.py:247-248), and the
// pair-major cull boxes the blend tests (boxes[vals[p]] split into one u32 per
// axis, so a warp's 32 box reads are two coalesced 128-byte loads).
__global__ void k_tile_ranges(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                              const uint2* __restrict__ boxes, const int64_t* __restrict__ n_pairs,
                              uint2* __restrict__ ranges, uint32_t* __restrict__ bxs,
                              uint32_t* __restrict__ bys) {
  // four consecutive pairs per thread (16-byte loads / stores, four independent
  // box gathers in flight); pairs < 2^30, so 32-bit indices
  const uint32_t P = (uint32_t)*n_pairs;
  const uint32_t groups = (P + 3) / 4;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x; gi < groups; gi += stride) {
    const uint32_t p = 4 * gi;
    uint32_t k[4], v[4];
    if (p + 4 <= P) {
      const uint4 k4 = __ldg(reinterpret_cast<const uint4*>(keys) + gi);
      const uint4 v4 = __ldg(reinterpret_cast<const uint4*>(vals) + gi);
      k[0] = k4.x; k[1] = k4.y; k[2] = k4.z; k[3] = k4.w;
      v[0] = v4.x; v[1] = v4.y; v[2] = v4.z; v[3] = v4.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        k[j] = p + j < P ? __ldg(keys + p + j) : 0xffffffffu;
        v[j] = p + j < P ? __ldg(vals + p + j) : 0u;
      }
    }
    uint2 b[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (p + j < P) b[j] = __ldg(boxes + v[j]);  // short4 (x0, x1, y0, y1)
    const uint32_t prev = p == 0 ? 0xffffffffu : __ldg(keys + p - 1);
    const uint32_t next = p + 4 < P ? __ldg(keys + p + 4) : 0xffffffffu;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (p + j >= P) break;
      const uint32_t before = j == 0 ? prev : k[j - 1];
      const uint32_t after = j == 3 ? next : (p + j + 1 < P ? k[j + 1] : 0xffffffffu);
      if (p + j == 0 || before != k[j]) ranges[k[j]].x = p + j;
      if (p + j + 1 == P || after != k[j]) ranges[k[j]].y = p + j + 1;
    }
    if (p + 4 <= P) {
      reinterpret_cast<uint4*>(bxs)[gi] = make_uint4(b[0].x, b[1].x, b[2].x, b[3].x);
      reinterpret_cast<uint4*>(bys)[gi] = make_uint4(b[0].y, b[1].y, b[2].y, b[3].y);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (p + j < P) { bxs[p + j] = b[j].x; bys[p + j] = b[j].y; }
    }
  }
}

int64_t bin_chunks(int64_t capacity) { return (capacity + kBinRanks - 1) / kBinRanks; }
// 8-byte words of the K5+K6 workspace: look-back status, then 16-byte heavy entries
int64_t bin_status_words(int64_t capacity) {
  const int64_t chunks = bin_chunks(capacity);
  return chunks + 2 + 2 * chunks;
}

void launch_bin_pairs(const uint32_t* order, const uint2* rects, DevStats* stats, int64_t pair_cap,
                      int64_t capacity, uint64_t* status, int ntx, uint32_t* keys, uint32_t* vals,
                      uint32_t* hist, int key_bits, bool emit, int64_t* host_overflow,
                      cudaStream_t s) {
  const int64_t chunks = bin_chunks(capacity);
  if (chunks == 0) return;
  DigitHist dh;  // hist == nullptr (keys wider than kMaxHistPasses digits): no counting
  dh.hist = hist;
  dh.n_passes = hist ? (key_bits + 7) / 8 : 0;
  dh.width = dh.n_passes ? (key_bits + dh.n_passes - 1) / dh.n_passes : 8;
  dh.end_bit = key_bits;
  if (hist) cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 256 * dh.n_passes, s);
  // status: chunks + 1 look-back words, then the heavy-chunk entries
  uint4* heavy = reinterpret_cast<uint4*>(status + chunks + 1 + ((chunks + 1) & 1));
  static int wave = 0;  // resident CTAs on the whole GPU
  if (!wave) {
    int per_sm = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bin_pairs, kBinThreads, 0);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    wave = std::max(1, per_sm * sms);
  }
  const unsigned grid = CS_BIN_PERSIST ? (unsigned)std::min<int64_t>(chunks, wave) : (unsigned)chunks;
  k_bin_pairs<<<grid, kBinThreads, 0, s>>>(order, rects, stats, pair_cap, status, heavy, ntx, keys,
                                           vals, dh, emit ? 1 : 0, host_overflow);
  if (emit)
    k_emit_heavy<<<(unsigned)std::min<int64_t>(kHeavyCtas, chunks), kBinThreads, 0, s>>>(
        order, rects, stats, heavy, ntx, keys, vals, dh);
}

void launch_tile_ranges(const uint32_t* keys, const uint32_t* vals, const short4* boxes,
                        const int64_t* n_pairs, uint2* ranges, uint32_t* bxs, uint32_t* bys,
                        cudaStream_t s) {
  k_tile_ranges<<<148 * 8, 256, 0, s>>>(keys, vals, reinterpret_cast<const uint2*>(boxes), n_pairs,
                                        ranges, bxs, bys);
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

__global__ void k_rank_of(const uint32_t* order, const DevStats* stats, int64_t* rank_of) {
  const int64_t M = stats->visible;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < M;
       r += (int64_t)gridDim.x * blockDim.x)
    rank_of[order[r]] = r;
}

// tile_ids as render._bin_tiles returns them: indices into the depth-sorted splats
__global__ void k_dump_tiles(const uint32_t* vals, const uint2* ranges, const DevStats* stats,
                             const int64_t* rank_of, int n_tiles, int64_t* tile_ids,
                             int64_t* offsets) {
  const int64_t P = stats->pairs_eff;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P; p += stride)
    tile_ids[p] = rank_of[vals[p]];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= n_tiles; t += stride) {
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
void launch_dump_tiles(const uint32_t* order, const uint32_t* vals, const uint2* ranges,
                       const DevStats* stats, int n_tiles, int64_t* rank_of, int64_t* tile_ids,
                       int64_t* offsets, cudaStream_t s) {
  k_rank_of<<<148 * 4, 256, 0, s>>>(order, stats, rank_of);
  k_dump_tiles<<<148 * 4, 256, 0, s>>>(vals, ranges, stats, rank_of, n_tiles, tile_ids, offsets);
}

}  // namespace cs

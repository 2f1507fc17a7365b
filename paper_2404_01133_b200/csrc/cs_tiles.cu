// cs_tiles.cu -- tile-local binning: the pair lists of render._bin_tiles
// (render.py:217-249) built per tile instead of by a global sort of all pairs.
//
// The reference emits, for every splat in depth order, one pair per tile of
// its rectangle and sorts the pairs stably by tile, so each tile's list holds
// its splats in depth-rank order.  After the global depth order (K4/K4b) that
// list is fully determined by the set of depth ranks covering the tile, so:
//
//   TL1 k_tl_count    per-tile pair counts (shared-memory histogram per CTA);
//   TL2 k_tl_scan     CSR offsets (the tile ranges), the frame's pair count
//                     and overflow report, per-tile cursors, and the tiles
//                     sorted into three size classes;
//   TL3 k_tl_scatter  every (rank, tile) pair claims a slot of its tile with
//                     one atomic (slot order arbitrary) and stores the rank;
//   TL4 k_tl_sort     each tile's ranks sorted in shared memory (LSD radix,
//                     8-bit digits, stable warp ranking by ballots; tiles of
//                     up to 2 x 16384 entries: two pieces and a merge), then
//                     written as the splat ids of the list with their
//                     pair-major cull boxes (what K8 did).
//
// Ranks are distinct, so the sorted list is exactly the reference's.  The
// global path (K5+K6 emission, K7 two-pass tile sort, K8) is kept for frames
// whose largest tile exceeds 2 x 16384 pairs (close-up / no-LoD views): TL2
// decides on the device (DevStats::tl_mode), and the kernels of the path not
// taken return at once, so a frame stays one fixed launch sequence (graph
// capturable).
#include <algorithm>
#include <cstdlib>

#include "cs_internal.cuh"

namespace cs {

constexpr int kTLCountThreads = 512;
constexpr int kTLMaxTiles = 49152;  // per-CTA tile histogram / cursors in shared memory (192 KB)
constexpr int kTLPiece = 1024 * 16;  // one CTA sort (1024 threads x 16 keys)
constexpr int kTLMax = 2 * kTLPiece;  // larger tiles -> the global-sort path
constexpr int kTLSmall = 1024, kTLMed = 4096;

// The pairs of ranks [lo, hi) with f(tile, rank), warp by warp: 32 ranks at a
// time, their rect areas scanned and the resulting pairs spread one per lane
// (owner lane by binary search over the scan), so a warp's work does not
// depend on its largest rect (a near splat can cover thousands of tiles).
// Pairs of a rank are visited row-major (render.py:233-243); the order across
// ranks is irrelevant here (TL4 sorts each tile).  Warp-collective.
template <typename F>
__device__ __forceinline__ void for_chunk_pairs(int64_t lo, int64_t hi, const uint32_t* __restrict__ order,
                                                const uint2* __restrict__ rects, int ntx, F f) {
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const uint32_t lane = lane_id();
  for (int64_t b = lo + 32 * warp; b < hi; b += 32 * nwarps) {
    const int64_t r = b + lane;
    const bool valid = r < hi;
    const uint2 pr = valid ? __ldg(rects + __ldg(order + r)) : make_uint2(0, 0);
    const int4 rc = unpack_rect(pr);
    const uint32_t w = (uint32_t)(rc.y - rc.x + 1);
    const uint32_t a = valid ? w * (uint32_t)(rc.w - rc.z + 1) : 0u;
    const uint32_t incl = warp_incl_scan(a);
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    for (uint32_t base = 0; base < total; base += 32) {
      const uint32_t p = base + lane;
      int o = 0;  // owner: the first lane whose inclusive scan exceeds p
#pragma unroll
      for (int st = 16; st > 0; st >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, incl, o + st - 1);
        if (v <= p) o += st;
      }
      const uint32_t oi = __shfl_sync(0xffffffffu, incl, o), oa = __shfl_sync(0xffffffffu, a, o);
      const uint32_t ow = __shfl_sync(0xffffffffu, w, o);
      const uint32_t ox = __shfl_sync(0xffffffffu, pr.x, o), oy = __shfl_sync(0xffffffffu, pr.y, o);
      const uint32_t orank = __shfl_sync(0xffffffffu, (uint32_t)r, o);
      if (p < total) {
        const uint32_t local = p - (oi - oa);
        const uint32_t ty = local / ow, tx = local - ty * ow;
        f((int)(((oy & 0xffffu) + ty) * (uint32_t)ntx + (ox & 0xffffu) + tx), orank);
      }
    }
  }
}

// TL1: CTA c counts the pairs of its contiguous chunk of depth ranks per tile
// (shared-memory histogram) and writes them as row c of H [G][n_tiles].
__global__ void __launch_bounds__(kTLCountThreads)
k_tl_count(const uint32_t* __restrict__ order, const uint2* __restrict__ rects,
           const DevStats* __restrict__ stats, int ntx, int n_tiles, uint32_t* __restrict__ H) {
  extern __shared__ uint32_t s_h[];
  for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) s_h[i] = 0;
  __syncthreads();
  const int64_t M = stats->visible;
  const int64_t lo = M * blockIdx.x / gridDim.x, hi = M * (blockIdx.x + 1) / gridDim.x;
  for_chunk_pairs(lo, hi, order, rects, ntx, [&](int t, uint32_t) { atomicAdd(&s_h[t], 1u); });
  __syncthreads();
  uint32_t* row = H + (int64_t)blockIdx.x * n_tiles;
  for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) row[i] = s_h[i];
}

// TL2: per tile, the exclusive prefix of its G chunk counts (in place: where
// chunk c's pairs start inside the tile) and its total; tile offsets by a
// block scan + decoupled look-back; size-class queues.  The last CTA to finish
// takes the frame decisions: pair count / overflow (reported as K5+K6 would),
// tile-local vs global path.
constexpr int kTLScanThreads = 256;
__global__ void __launch_bounds__(kTLScanThreads)
k_tl_scan(uint32_t* __restrict__ H, int G, int n_tiles, DevStats* __restrict__ stats, int64_t pair_cap,
          uint2* __restrict__ ranges, uint32_t* __restrict__ queues, uint64_t* __restrict__ status,
          uint32_t* __restrict__ ctl /* [0] max, [1] done */, int emit, int64_t* host_overflow,
          uint32_t tl_max) {
  __shared__ uint32_t s_scan[kTLScanThreads / 32 + 1];
  __shared__ uint32_t s_nq[3], s_qb[3], s_max, s_chunk;
  __shared__ uint64_t s_pre;
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    s_chunk = atomicAdd(&stats->tickets[15], 1u);
    s_nq[0] = s_nq[1] = s_nq[2] = 0;
    s_max = 0;
  }
  __syncthreads();
  const int chunk = (int)s_chunk;
  const int t = chunk * kTLScanThreads + threadIdx.x;
  uint32_t tot = 0;
  if (t < n_tiles) {
    constexpr int U = 8;
    int c = 0;
    for (; c + U <= G; c += U) {
      uint32_t v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) v[j] = H[(int64_t)(c + j) * n_tiles + t];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        H[(int64_t)(c + j) * n_tiles + t] = tot;
        tot += v[j];
      }
    }
    for (; c < G; ++c) {
      const uint32_t v = H[(int64_t)c * n_tiles + t];
      H[(int64_t)c * n_tiles + t] = tot;
      tot += v;
    }
  }
  uint32_t btot;
  const uint32_t ex = block_excl_scan<uint32_t>(tot, s_scan, btot);
  if (threadIdx.x < 32) {
    const uint64_t pre = lookback_exclusive(status, chunk, btot);
    if (threadIdx.x == 0) s_pre = pre;
  }
  int q = -1;
  if (t < n_tiles && tot) q = tot <= (uint32_t)kTLSmall ? 0 : (tot <= (uint32_t)kTLMed ? 1 : 2);
  uint32_t qs = 0;
  if (q >= 0) qs = atomicAdd(&s_nq[q], 1u);
  atomicMax(&s_max, tot);
  __syncthreads();
  if (threadIdx.x < 3 && s_nq[threadIdx.x]) s_qb[threadIdx.x] = atomicAdd(&stats->tl_nq[threadIdx.x], s_nq[threadIdx.x]);
  if (threadIdx.x == 0) atomicMax(&ctl[0], s_max);
  __syncthreads();
  const uint64_t off = s_pre + ex;
  if (t < n_tiles) {
    ranges[t] = make_uint2((uint32_t)off, (uint32_t)(off + tot));  // overflow: cleared below
    if (q >= 0) queues[(int64_t)q * n_tiles + s_qb[q] + qs] = (uint32_t)t;
  }
  if (chunk == (int)gridDim.x - 1 && threadIdx.x == 0) stats->pairs = (int64_t)(s_pre + btot);
  // the last CTA to arrive decides for the frame
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&ctl[1], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int64_t P = *((volatile int64_t*)&stats->pairs);
  const uint32_t mx = *((volatile uint32_t*)&ctl[0]);
  const bool over = P > pair_cap;
  if (threadIdx.x == 0) {
    stats->pairs_eff = over ? 0 : P;
    if (over) {
      atomicOr(&stats->status, 1);
      if (emit && host_overflow) {  // raised by the context's next call, like k_bin_pairs
        volatile int64_t* hp = host_overflow;
        hp[1] = pair_cap;
        hp[0] = P;
        __threadfence_system();
      }
    }
    const bool fast = !over && mx <= tl_max;
    stats->tl_mode = (fast || over) ? 1 : 0;   // overflow: nothing is emitted on either path
    stats->pairs_sort = (fast || over) ? 0 : P;
  }
  if (over)
    for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) ranges[i] = make_uint2(0, 0);
}

// TL3: CTA c re-walks its chunk; each pair takes the next slot of its tile's
// chunk-c segment (shared-memory cursors; order inside a segment arbitrary,
// fixed by TL4) and stores its depth rank there.
__global__ void __launch_bounds__(kTLCountThreads)
k_tl_scatter(const uint32_t* __restrict__ order, const uint2* __restrict__ rects,
             const DevStats* __restrict__ stats, int ntx, int n_tiles, const uint32_t* __restrict__ H,
             const uint2* __restrict__ ranges, uint32_t* __restrict__ slots) {
  extern __shared__ uint32_t s_cur[];
  if (stats->tl_mode != 1 || stats->pairs_eff == 0) return;
  const uint32_t* row = H + (int64_t)blockIdx.x * n_tiles;
  for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) s_cur[i] = ranges[i].x + row[i];
  __syncthreads();
  const int64_t M = stats->visible;
  const int64_t lo = M * blockIdx.x / gridDim.x, hi = M * (blockIdx.x + 1) / gridDim.x;
  for_chunk_pairs(lo, hi, order, rects, ntx, [&](int t, uint32_t rank) {
    slots[atomicAdd(&s_cur[t], 1u)] = rank;
  });
}

// Stable LSD radix sort (8-bit digits, npass passes) of n <= THREADS * ITEMS
// distinct keys in shared memory, in place.  Warp w holds positions
// [w * 32 * ITEMS, (w + 1) * 32 * ITEMS), item i lane l = position
// w * 32 * ITEMS + 32 i + l; a key's rank among equal digits comes from 8
// ballots (peer mask) plus its warp's running digit counter, and warps are
// combined in order -- so each pass is stable.  CTA-collective.
template <int THREADS, int ITEMS>
__device__ __forceinline__ void block_sort_keys(uint32_t* s, int n, int npass, uint32_t (*s_cnt)[256],
                                                uint32_t* s_dbase) {
  constexpr int WARPS = THREADS / 32;
  const int warp = threadIdx.x >> 5;
  const uint32_t lane = lane_id(), lt = lanemask_lt();
  const int seg = warp * 32 * ITEMS;
  // ranks inside the warp's segment (< 32 * ITEMS <= 65536) packed two per register
  uint32_t key[ITEMS], rnk[(ITEMS + 1) / 2];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int e = seg + i * 32 + (int)lane;
    key[i] = e < n ? s[e] : 0u;
  }
  for (int pass = 0; pass < npass; ++pass) {
    const int shift = 8 * pass;
    for (int j = (int)lane; j < 256; j += 32) s_cnt[warp][j] = 0;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int e0 = seg + i * 32;
      if (e0 >= n) break;  // warp-uniform
      const bool valid = e0 + (int)lane < n;
      const uint32_t d = (key[i] >> shift) & 255u;
      uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        peers &= ((d >> b) & 1u) ? bal : ~bal;
      }
      const uint32_t before = valid ? s_cnt[warp][d] : 0u;
      __syncwarp();
      const uint32_t below = __popc(peers & lt);
      if (valid && below == (uint32_t)__popc(peers) - 1u) s_cnt[warp][d] = before + below + 1u;
      __syncwarp();
      const uint32_t rr = before + below;
      rnk[i >> 1] = (i & 1) ? (rnk[i >> 1] | (rr << 16)) : rr;
    }
    __syncthreads();
    // per digit: exclusive prefix over the warps, and the digit totals
    for (int d = threadIdx.x; d < 256; d += THREADS) {
      constexpr int G = WARPS < 8 ? WARPS : 8;  // loads in flight per group
      uint32_t sum = 0;
#pragma unroll
      for (int w0 = 0; w0 < WARPS; w0 += G) {
        uint32_t c[G];
#pragma unroll
        for (int w = 0; w < G; ++w) c[w] = s_cnt[w0 + w][d];
#pragma unroll
        for (int w = 0; w < G; ++w) {
          s_cnt[w0 + w][d] = sum;
          sum += c[w];
        }
      }
      s_dbase[d] = sum;
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 256 digit totals, 8 per lane
      uint32_t v[8], run = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        v[j] = s_dbase[lane * 8 + j];
        run += v[j];
      }
      const uint32_t incl = warp_incl_scan(run);
      uint32_t acc = incl - run;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        s_dbase[lane * 8 + j] = acc;
        acc += v[j];
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int e = seg + i * 32 + (int)lane;
      if (e < n) {
        const uint32_t d = (key[i] >> shift) & 255u;
        s[s_dbase[d] + s_cnt[warp][d] + ((rnk[i >> 1] >> (16 * (i & 1))) & 0xffffu)] = key[i];
      }
    }
    __syncthreads();
    if (pass + 1 < npass) {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const int e = seg + i * 32 + (int)lane;
        if (e < n) key[i] = s[e];
      }
    }
  }
}

// TL4: one tile per CTA iteration from size-class queue q.  Memory accesses
// are batched per thread (all key loads, then all id gathers, then all box
// gathers in flight at once) -- each tile is a few dependent latencies, not a
// few per element.
template <int THREADS, int N>
__device__ __forceinline__ void tl_emit_batch(const uint32_t (&key)[N], int cnt, const uint32_t (&pos)[N],
                                              const uint32_t* __restrict__ order, const uint2* __restrict__ boxes,
                                              uint32_t* __restrict__ list, uint32_t* __restrict__ bxs,
                                              uint32_t* __restrict__ bys) {
  uint32_t id[N];
  uint2 b[N];
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (j < cnt) id[j] = __ldg(order + key[j]);
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (j < cnt) b[j] = __ldg(boxes + id[j]);  // short4 (x0, x1, y0, y1)
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (j < cnt) {
      list[pos[j]] = id[j];
      bxs[pos[j]] = b[j].x;
      bys[pos[j]] = b[j].y;
    }
}

template <int THREADS, int ITEMS, int PIECES>
__global__ void __launch_bounds__(THREADS, 1024 / THREADS)
k_tl_sort(const uint32_t* __restrict__ queue, int q, const uint32_t* __restrict__ slots,
          const uint2* __restrict__ ranges, const uint32_t* __restrict__ order,
          const uint2* __restrict__ boxes, DevStats* __restrict__ stats, uint32_t* __restrict__ list,
          uint32_t* __restrict__ bxs, uint32_t* __restrict__ bys) {
  constexpr int WARPS = THREADS / 32;
  constexpr int CAP = THREADS * ITEMS;
  constexpr int OB = THREADS >= 1024 ? 4 : 8;  // outputs per batch (register budget)
  extern __shared__ __align__(16) uint32_t s_dyn[];
  uint32_t* s_keys = s_dyn;                                                          // [CAP * PIECES]
  uint32_t(*s_cnt)[256] = reinterpret_cast<uint32_t(*)[256]>(s_dyn + CAP * PIECES);  // [WARPS][256]
  uint32_t* s_dbase = s_dyn + CAP * PIECES + WARPS * 256;                            // [256]
  __shared__ uint32_t s_tile;
  if (stats->tl_mode != 1) return;
  const uint32_t nq = stats->tl_nq[q];
  const int64_t M = stats->visible;
  const int nbits = M > 1 ? 64 - __clzll((unsigned long long)(M - 1)) : 1;
  const int npass = (nbits + 7) / 8;
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&stats->tickets[12 + q], 1u);
    __syncthreads();
    const uint32_t ti = s_tile;
    if (ti >= nq) break;
    const uint32_t t = queue[ti];
    const uint2 rg = ranges[t];
    const int n = (int)(rg.y - rg.x);
    for (int e0 = 0; e0 < n; e0 += THREADS * OB) {  // coalesced, OB loads in flight per thread
      uint32_t v[OB];
#pragma unroll
      for (int j = 0; j < OB; ++j) {
        const int e = e0 + j * THREADS + (int)threadIdx.x;
        if (e < n) v[j] = __ldg(slots + rg.x + e);
      }
#pragma unroll
      for (int j = 0; j < OB; ++j) {
        const int e = e0 + j * THREADS + (int)threadIdx.x;
        if (e < n) s_keys[e] = v[j];
      }
    }
    __syncthreads();
    if (PIECES == 1 || n <= CAP) {
      block_sort_keys<THREADS, ITEMS>(s_keys, n, npass, s_cnt, s_dbase);
      for (int e0 = 0; e0 < n; e0 += THREADS * OB) {
        uint32_t k[OB], pos[OB];
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < OB; ++j) {
          const int e = e0 + j * THREADS + (int)threadIdx.x;
          if (e < n) {
            k[j] = s_keys[e];
            pos[j] = rg.x + e;
            cnt = j + 1;
          }
        }
        tl_emit_batch<THREADS, OB>(k, cnt, pos, order, boxes, list, bxs, bys);
      }
    } else {
      // two pieces of <= CAP keys sorted separately, then merged (merge path)
      const int na = (n + 1) / 2, nb = n - na;
      block_sort_keys<THREADS, ITEMS>(s_keys, na, npass, s_cnt, s_dbase);
      block_sort_keys<THREADS, ITEMS>(s_keys + na, nb, npass, s_cnt, s_dbase);
      const uint32_t* A = s_keys;
      const uint32_t* B = s_keys + na;
      const int per = (n + THREADS - 1) / THREADS;
      const int k0 = min(n, (int)threadIdx.x * per), k1 = min(n, k0 + per);
      if (k0 < k1) {
        int lo = max(0, k0 - nb), hi = min(k0, na);
        while (lo < hi) {  // first i with A[i] > B[k0 - i - 1] (keys distinct)
          const int mid = (lo + hi) >> 1;
          if (A[mid] < B[k0 - mid - 1]) lo = mid + 1; else hi = mid;
        }
        int i = lo, j = k0 - lo;
        for (int kb = k0; kb < k1; kb += OB) {
          uint32_t k[OB], pos[OB];
          int cnt = 0;
#pragma unroll
          for (int u = 0; u < OB; ++u) {
            if (kb + u < k1) {
              const bool takeA = j >= nb || (i < na && A[i] < B[j]);
              k[u] = takeA ? A[i++] : B[j++];
              pos[u] = rg.x + kb + u;
              cnt = u + 1;
            }
          }
          tl_emit_batch<THREADS, OB>(k, cnt, pos, order, boxes, list, bxs, bys);
        }
      }
    }
    __syncthreads();  // shared keys are reused by the next tile
  }
}

template <int THREADS, int ITEMS, int PIECES>
static void launch_tl_sort(int grid, const uint32_t* queue, int q, const uint32_t* slots, const uint2* ranges,
                           const uint32_t* order, const uint2* boxes, DevStats* stats, uint32_t* list,
                           uint32_t* bxs, uint32_t* bys, cudaStream_t s) {
  constexpr size_t smem = sizeof(uint32_t) * ((size_t)THREADS * ITEMS * PIECES + (THREADS / 32) * 256 + 256);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tl_sort<THREADS, ITEMS, PIECES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    attr = true;
  }
  k_tl_sort<THREADS, ITEMS, PIECES><<<grid, THREADS, smem, s>>>(queue, q, slots, ranges, order, boxes, stats,
                                                                list, bxs, bys);
}

static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

// chunks of depth ranks (TL1 / TL3 grid): G rows of the per-tile count matrix
static int tl_chunks() { return 2 * sm_count(); }
static int tl_scan_blocks(int n_tiles) { return (n_tiles + kTLScanThreads - 1) / kTLScanThreads; }

// workspace (u32 words): H [G][n_tiles], queues [3][n_tiles], look-back status
// (u64 per scan block), control words (max, done)
int64_t tl_words(int n_tiles) {
  return (int64_t)(tl_chunks() + 3) * n_tiles + 2 * (tl_scan_blocks(n_tiles) + 1) + 4;
}

bool tile_local_enabled(int n_tiles) {
  // opt-in while its kernels are slower than the global path (CS_TILE_LOCAL=1);
  // read per frame (direct frames follow changes; a cached frame graph keeps
  // the binning it was captured with)
  const char* e = getenv("CS_TILE_LOCAL");
  return e && e[0] == '1' && n_tiles <= kTLMaxTiles;
}

struct TLLayout {
  uint32_t* H;
  uint32_t* queues;
  uint64_t* status;
  uint32_t* ctl;
};
static TLLayout tl_layout(uint32_t* tl, int n_tiles) {
  TLLayout L;
  const int G = tl_chunks();
  L.H = tl;
  L.queues = tl + (int64_t)G * n_tiles;
  int64_t off = (int64_t)(G + 3) * n_tiles;
  off += off & 1;  // 8-byte alignment
  L.status = reinterpret_cast<uint64_t*>(tl + off);
  L.ctl = tl + off + 2 * (tl_scan_blocks(n_tiles) + 1);
  return L;
}

template <typename K>
static void smem_attr(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// TL1 + TL2 (before the global path's K5+K6, which returns at once when the
// tile-local path was chosen)
void launch_tl_count_scan(const uint32_t* order, const uint2* rects, DevStats* stats, int ntx, int n_tiles,
                          uint32_t* tl, int64_t pair_cap, uint2* ranges, bool emit, int64_t* host_overflow,
                          cudaStream_t s) {
  const TLLayout L = tl_layout(tl, n_tiles);
  const int nb = tl_scan_blocks(n_tiles);
  cudaMemsetAsync(L.status, 0, sizeof(uint64_t) * (nb + 1) + 2 * sizeof(uint32_t), s);
  const size_t smem = sizeof(uint32_t) * n_tiles;
  smem_attr(k_tl_count, smem);
  k_tl_count<<<tl_chunks(), kTLCountThreads, smem, s>>>(order, rects, stats, ntx, n_tiles, L.H);
  // CS_TL_MAX (tests / A-B runs): a lower largest-tile limit for the tile-local
  // path (0: always the global path); read per call, so direct frames see changes
  uint32_t tl_max = kTLMax;
  if (const char* e = getenv("CS_TL_MAX")) tl_max = (uint32_t)std::min<long>(kTLMax, std::max<long>(0, atol(e)));
  k_tl_scan<<<nb, kTLScanThreads, 0, s>>>(L.H, tl_chunks(), n_tiles, stats, pair_cap, ranges, L.queues, L.status,
                                          L.ctl, emit ? 1 : 0, host_overflow, tl_max);
}

// TL3 (slots: a free pair buffer)
void launch_tl_scatter(const uint32_t* order, const uint2* rects, DevStats* stats, int ntx, int n_tiles,
                       uint32_t* tl, const uint2* ranges, uint32_t* slots, cudaStream_t s) {
  const TLLayout L = tl_layout(tl, n_tiles);
  const size_t smem = sizeof(uint32_t) * n_tiles;
  smem_attr(k_tl_scatter, smem);
  k_tl_scatter<<<tl_chunks(), kTLCountThreads, smem, s>>>(order, rects, stats, ntx, n_tiles, L.H, ranges, slots);
}

// TL4: the three size classes, largest first
void launch_tl_sort(const uint32_t* order, const uint2* boxes, DevStats* stats, int n_tiles, uint32_t* tl,
                    const uint32_t* slots, const uint2* ranges, uint32_t* list, uint32_t* bxs, uint32_t* bys,
                    cudaStream_t s) {
  const uint32_t* queues = tl_layout(tl, n_tiles).queues;
  const int sms = sm_count();
  launch_tl_sort<1024, 16, 2>(sms, queues + 2ll * n_tiles, 2, slots, ranges, order, boxes, stats, list, bxs,
                              bys, s);
  launch_tl_sort<256, 16, 1>(sms * 4, queues + 1ll * n_tiles, 1, slots, ranges, order, boxes, stats, list, bxs,
                             bys, s);
  launch_tl_sort<128, 8, 1>(sms * 8, queues, 0, slots, ranges, order, boxes, stats, list, bxs, bys, s);
}

}  // namespace cs

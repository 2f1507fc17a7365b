// cs_sort.cu -- K4/K7: stable LSD radix sort (onesweep-style), device-side count.
//
// Used for the global depth order (np.argsort(depths, kind="stable"),
// render.py:176-177; the 32-bit coarsened depth key of cs_project.cu, exact
// order restored by K4b in cs_depth.cu), for the stable tile grouping
// (np.argsort(tiles, kind="stable"), render.py:245; keys = tile id, only
// ceil(log2 n_tiles) bits sorted) and, with 64-bit keys, for the LoD
// generation's priority and block orders (cs_lodgen.cu).
//
// Per pass one kernel reads keys+values once and writes them once:
//   * chunks of kTile elements are taken in launch order (ticket counter);
//   * each warp ranks its keys stably from NB ballots over the digit bits
//     (the peer mask of every key) and per-warp digit counters; warps are
//     combined in warp order, so the chunk-local order equals the input order
//     within every digit (stability);
//   * per-digit chunk counts are published and a decoupled look-back per
//     digit gives the chunk's global offset (no separate scan pass);
//   * keys are first scattered to shared memory in digit order, then written
//     out so consecutive threads store consecutive addresses of one digit run.
// A single histogram kernel computes the digit counts of every pass up front;
// the scan kernel after it also clears the look-back status of every pass for
// the actual count, and each pass runs one wave of CTAs that loop over chunk
// tickets, so a large pair capacity costs nothing when a view has few pairs.
// The element count is read from device memory, so the whole frame runs
// without a host round trip (and is CUDA-graph capturable).
#include <algorithm>

#include "cs_internal.cuh"

namespace cs {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr uint32_t kStFlagAgg = 1u << 30;
constexpr uint32_t kStFlagPre = 2u << 30;
constexpr uint32_t kStMask = (1u << 30) - 1;
#ifndef CS_SORT_LB
#define CS_SORT_LB 8
#endif
constexpr int kLookback = CS_SORT_LB;

// Programmatic dependent launch between the passes (CS_SORT_PDL): a pass is
// launched while its predecessor drains, its CTAs wait at griddepcontrol.wait
// (predecessor complete, memory visible) before touching any data, and every
// CTA lets its dependents launch as soon as it starts.
#ifndef CS_SORT_PDL
#define CS_SORT_PDL 1
#endif
__device__ __forceinline__ void pdl_wait() {
  if (CS_SORT_PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger() {
  if (CS_SORT_PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... Params, typename... Args>
static void launch_pdl(void (*kernel)(Params...), unsigned grid, unsigned block, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = CS_SORT_PDL ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <typename K> struct SortCfg;
template <> struct SortCfg<uint64_t> { static constexpr int kItems = 8, kMinBlocks = 1; };
#ifndef CS_SORT_ITEMS32
#define CS_SORT_ITEMS32 16
#endif
#ifndef CS_SORT_MINB32
#define CS_SORT_MINB32 3
#endif
template <> struct SortCfg<uint32_t> { static constexpr int kItems = CS_SORT_ITEMS32, kMinBlocks = CS_SORT_MINB32; };

// Digit counts of every pass in one read of the keys.  Keys that arrive in
// assembled order are spatially coherent (the depth key's top digits repeat
// for long stretches), so each thread counts a run of 8 consecutive keys and
// adds each run of equal digits with one shared atomic: a hot bin is not hit
// by every lane of every warp.  (match.any-aggregation measured slower: its
// latency sits on every key.)
constexpr int kHistRun = 8;
template <typename K>
__global__ void __launch_bounds__(kSortThreads)
k_radix_hist(const K* __restrict__ keys, const int64_t* __restrict__ n_ptr, int begin_bit,
             int n_passes, int width, int end_bit, uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[8 * 256];
  for (int i = threadIdx.x; i < n_passes * 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int64_t n = *n_ptr;
  const int64_t groups = (n + kHistRun - 1) / kHistRun;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups; g += stride) {
    const int64_t i0 = g * kHistRun;
    K k[kHistRun];
    int cnt = kHistRun;
    if (sizeof(K) == 4 && i0 + kHistRun <= n) {
      const uint4* q = reinterpret_cast<const uint4*>(keys + i0);
      const uint4 a = q[0], b = q[1];
      k[0] = (K)a.x; k[1] = (K)a.y; k[2] = (K)a.z; k[3] = (K)a.w;
      k[4] = (K)b.x; k[5] = (K)b.y; k[6] = (K)b.z; k[7] = (K)b.w;
    } else {
      cnt = (int)(n - i0 < kHistRun ? n - i0 : kHistRun);
#pragma unroll
      for (int j = 0; j < kHistRun; ++j) k[j] = j < cnt ? keys[i0 + j] : K(0);
    }
    for (int p = 0; p < n_passes; ++p) {
      const int sh_p = begin_bit + width * p;
      const uint32_t m = (1u << min(width, end_bit - sh_p)) - 1u;
      uint32_t cur = (uint32_t)(k[0] >> sh_p) & m, run = 1;
#pragma unroll
      for (int j = 1; j < kHistRun; ++j) {
        if (j >= cnt) break;
        const uint32_t d = (uint32_t)(k[j] >> sh_p) & m;
        if (d == cur) {
          ++run;
        } else {
          atomicAdd(&sh[p * 256 + cur], run);
          cur = d;
          run = 1;
        }
      }
      atomicAdd(&sh[p * 256 + cur], run);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_passes * 256; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// exclusive scan of each pass's 256-bin histogram, in place (block 0), and
// the look-back status of every pass zeroed for the ACTUAL element count (all
// blocks; pass p's words start at p * ceil(n / tile) * 256), so neither the
// status clear nor the pass grids scale with the buffer capacity
__global__ void k_radix_hist_scan(uint32_t* hist, int n_passes, uint32_t* __restrict__ status,
                                  const int64_t* __restrict__ n_ptr, int tile) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint32_t scratch[kSortWarps + 1];
  if (blockIdx.x == 0) {
    for (int p = 0; p < n_passes; ++p) {
      uint32_t v = hist[p * 256 + threadIdx.x];
      uint32_t total;
      uint32_t ex = block_excl_scan<uint32_t>(v, scratch, total);
      hist[p * 256 + threadIdx.x] = ex;
    }
  }
  const uint64_t chunks = ((uint64_t)*n_ptr + tile - 1) / tile;
  const uint64_t n4 = chunks * 64 * n_passes;  // uint4 words
  uint4* st4 = reinterpret_cast<uint4*>(status);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4;
       i += (uint64_t)gridDim.x * blockDim.x)
    st4[i] = make_uint4(0, 0, 0, 0);
}

// The pass body, FULL = the chunk holds kTile keys (no bounds checks, the
// common case), NB = digit width (ballot count known at compile time).
// Indices are 32-bit (n < 2^31).
template <typename K, int ITEMS, bool FULL, int NB, bool EARLY, bool IDV>
__device__ __forceinline__ void onesweep_body(
    const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, K* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, uint32_t n, uint32_t chunk, int shift,
    const uint32_t* __restrict__ digit_base, uint32_t* __restrict__ status,
    uint32_t (*warp_hist)[256], uint32_t* chunk_hist, uint32_t* digit_off, uint32_t* gbase,
    uint32_t* scratch, K* keys_s, uint32_t* vals_s) {
  constexpr int kItems = ITEMS;
  constexpr int kTile = kSortThreads * kItems;
  constexpr uint32_t dmask = (1u << NB) - 1u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t base = chunk * kTile;
  const uint32_t valid_count = FULL ? kTile : n - base;
  K key[kItems];
  uint32_t val[kItems];
  uint32_t rank[kItems];
  const uint32_t wbase = base + warp * 32 * kItems;
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const uint32_t idx = wbase + r * 32 + lane;
    if (FULL || idx < n) {
      key[r] = keys_in[idx];
      val[r] = IDV ? idx : vals_in[idx];  // IDV: the identity as input values (first depth pass)
    }
  }
  // 1) EARLY: chunk histogram first, published immediately so successors'
  //    look-back finds this chunk's aggregate while it is still ranking.
  //    Otherwise the ranking's group leaders also count the chunk histogram
  //    (one atomic per digit group instead of one per key) and it is
  //    published right after the ranking.
  const int d = threadIdx.x;  // 256 threads == 256 digits
  uint32_t* my_status = status + (size_t)chunk * 256 + d;
  uint32_t my_count = 0;
  if (EARLY) {
#pragma unroll
    for (int r = 0; r < kItems; ++r)
      if (FULL || wbase + r * 32 + lane < n) atomicAdd(&chunk_hist[(uint32_t)(key[r] >> shift) & dmask], 1u);
    __syncthreads();
    my_count = chunk_hist[d];
    atomicExch(my_status, (chunk == 0 ? kStFlagPre : kStFlagAgg) | my_count);
  }
  // 2) stable in-warp ranks (warp order == input order): the lanes holding
  //    the same digit from NB ballots; all peer masks first (the vote
  //    latencies overlap), then per item the leader lane of each digit group
  //    bumps the warp's counter with one shared atomic and broadcasts the old
  //    value.  A warp's atomics to one address execute in issue order, so
  //    items keep their input order.
  const uint32_t lt = lanemask_lt();
  uint32_t peers[kItems];
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const bool valid = FULL || wbase + r * 32 + lane < n;
    const uint32_t dg = (uint32_t)(key[r] >> shift) & dmask;
    uint32_t pm = FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int bit = 0; bit < NB; ++bit) {
      const bool on = (dg >> bit) & 1u;
      const uint32_t bal = __ballot_sync(0xffffffffu, on);
      pm &= on ? bal : ~bal;
    }
    peers[r] = valid ? pm : 0u;
  }
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const uint32_t pm = peers[r];
    const uint32_t dg = (uint32_t)(key[r] >> shift) & dmask;
    const int leader = pm ? __ffs(pm) - 1 : (int)lane;
    uint32_t old = 0;
    if (pm && (int)lane == leader) {
      old = atomicAdd(&warp_hist[warp][dg], (uint32_t)__popc(pm));
      if (!EARLY) atomicAdd(&chunk_hist[dg], (uint32_t)__popc(pm));
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    rank[r] = old + __popc(pm & lt);
  }
  __syncthreads();
  if (!EARLY) {
    my_count = chunk_hist[d];
    atomicExch(my_status, (chunk == 0 ? kStFlagPre : kStFlagAgg) | my_count);
  }
  // 3) combine warps and the chunk-local digit starts
  uint32_t sum = 0;
#pragma unroll
  for (int w = 0; w < kSortWarps; ++w) {
    const uint32_t c = warp_hist[w][d];
    warp_hist[w][d] = sum;
    sum += c;
  }
  uint32_t total;
  const uint32_t local_start = block_excl_scan<uint32_t>(sum, scratch, total);
  digit_off[d] = local_start;
  __syncthreads();
  // 4) scatter into shared memory in chunk-local sorted order
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    if (FULL || wbase + r * 32 + lane < n) {
      const uint32_t dg = (uint32_t)(key[r] >> shift) & dmask;
      const uint32_t pos = digit_off[dg] + warp_hist[warp][dg] + rank[r];
      keys_s[pos] = key[r];
      vals_s[pos] = val[r];
    }
  }
  // 5) decoupled look-back for this digit, kLookback predecessors per round
  //    trip (a chunk of the first wave may have to sum hundreds of
  //    predecessors' aggregates before any inclusive prefix exists)
  uint32_t excl = 0;
  if (chunk > 0) {
    int p = (int)chunk - 1;
    bool found = false;
    while (!found) {
      uint32_t st[kLookback];
#pragma unroll
      for (int k = 0; k < kLookback; ++k)
        st[k] = p - k >= 0 ? ld_volatile_u32(status + (size_t)(p - k) * 256 + d) : (kStFlagPre | 0u);
#pragma unroll
      for (int k = 0; k < kLookback; ++k) {
        if (found) break;
        const uint32_t flag = st[k] >> 30;
        if (flag == 0) break;          // not published yet: re-read from here
        excl += st[k] & kStMask;
        --p;
        if (flag == 2) found = true;
      }
    }
    atomicExch(my_status, kStFlagPre | (excl + my_count));
  }
  gbase[d] = digit_base[d] + excl - local_start;
  __syncthreads();
  // 6) coalesced write-out: consecutive threads store consecutive addresses of one digit run
#pragma unroll 4
  for (uint32_t i = threadIdx.x; i < valid_count; i += kSortThreads) {
    const K k = keys_s[i];
    const uint32_t o = gbase[(uint32_t)(k >> shift) & dmask] + i;
    keys_out[o] = k;
    vals_out[o] = vals_s[i];
  }
}

#ifndef CS_SORT_PERSIST
#define CS_SORT_PERSIST 1
#endif

template <typename K, int ITEMS = SortCfg<K>::kItems, int MINB = 1, int NB = 8, bool EARLY = true,
          bool IDV = false>
__global__ void __launch_bounds__(kSortThreads, MINB)
k_onesweep(const K* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
           K* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
           const int64_t* __restrict__ n_ptr, int shift,
           const uint32_t* __restrict__ digit_base, uint32_t* __restrict__ status, int pass,
           uint32_t* __restrict__ ticket) {
  constexpr int kTile = kSortThreads * ITEMS;
  __shared__ uint32_t warp_hist[kSortWarps][256];
  __shared__ uint32_t chunk_hist[256];
  __shared__ uint32_t digit_off[256];
  __shared__ uint32_t gbase[256];
  __shared__ uint32_t scratch[kSortWarps + 1];
  __shared__ uint32_t s_chunk;
  __shared__ K keys_s[kTile];
  __shared__ uint32_t vals_s[kTile];

  pdl_wait();
  pdl_trigger();
  const uint32_t n = (uint32_t)*n_ptr;
  status += (size_t)pass * ((n + kTile - 1) / kTile) * 256;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // CS_SORT_PERSIST: the grid is at most one wave and every CTA loops over
  // chunk tickets until the actual count is covered (no capacity-sized grid
  // of CTAs that only exit)
  while (true) {
    if (threadIdx.x == 0) s_chunk = atomicAdd(ticket, 1u);
    for (int d = lane; d < 256; d += 32) warp_hist[warp][d] = 0;
    chunk_hist[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t chunk = s_chunk;
    const uint64_t base = (uint64_t)chunk * kTile;
    if (base >= n) return;
    if (base + kTile <= n)
      onesweep_body<K, ITEMS, true, NB, EARLY, IDV>(keys_in, vals_in, keys_out, vals_out, n, chunk, shift,
                                               digit_base, status, warp_hist, chunk_hist, digit_off,
                                               gbase, scratch, keys_s, vals_s);
    else
      onesweep_body<K, ITEMS, false, NB, EARLY, IDV>(keys_in, vals_in, keys_out, vals_out, n, chunk, shift,
                                                digit_base, status, warp_hist, chunk_hist, digit_off,
                                                gbase, scratch, keys_s, vals_s);
    if (!CS_SORT_PERSIST) return;
    __syncthreads();  // shared arrays are reused by the next chunk
  }
}

// Workspace: hist (8*256 u32), status (passes*chunks*256 u32), tickets (8 u32).
size_t radix_status_words(int64_t capacity, int key_bytes) {
  const int items = key_bytes == 8 ? SortCfg<uint64_t>::kItems : SortCfg<uint32_t>::kItems;
  const int64_t tile = (int64_t)kSortThreads * items;
  return (size_t)((capacity + tile - 1) / tile) * 256 * key_bytes;  // <= key_bytes 8-bit passes
}

// Sorts (keys, vals) of length *n_dev (<= capacity) by bits [begin_bit, end_bit).
// Ping-pongs between (k0,v0) and (k1,v1); returns 1 when the result is in
// (k1,v1), 0 when in (k0,v0).
template <typename K, int ITEMS, int MINB, int NB, bool EARLY, bool IDV = false>
static void launch_pass(unsigned chunks, cudaStream_t s, const K* kin, const uint32_t* vin, K* kout,
                        uint32_t* vout, const int64_t* n_dev, int shift, const uint32_t* hist,
                        uint32_t* status, int pass, uint32_t* ticket) {
  static bool carveout = false;  // shared memory is the occupancy limit: take all of it
  if (!carveout) {
    cudaFuncSetAttribute(k_onesweep<K, ITEMS, MINB, NB, EARLY, IDV>,
                         cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    carveout = true;
  }
  static int wave = 0;  // resident CTAs of this instantiation on the whole GPU
  if (!wave) {
    int per_sm = 0, dev = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_onesweep<K, ITEMS, MINB, NB, EARLY, IDV>,
                                                  kSortThreads, 0);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    wave = std::max(1, per_sm * sms);
  }
  const unsigned g = CS_SORT_PERSIST ? std::min<unsigned>(chunks, (unsigned)wave) : chunks;
  launch_pdl(k_onesweep<K, ITEMS, MINB, NB, EARLY, IDV>, g, kSortThreads, s, kin, vin, kout, vout, n_dev,
             shift, hist, status, pass, ticket);
}

template <typename K, int ITEMS, int MINB = SortCfg<K>::kMinBlocks, bool EARLY = true>
int radix_sort_items(K* k0, uint32_t* v0, K* k1, uint32_t* v1, const int64_t* n_dev,
                     int64_t capacity, int begin_bit, int end_bit, uint32_t* hist,
                     uint32_t* status, uint32_t* tickets, cudaStream_t s, bool hist_ready = false,
                     bool identity_vals = false) {
  // equal-width digits of <= 8 bits (13 tile bits -> 7 + 6: fewer ballots per key)
  const int n_passes = (end_bit - begin_bit + 7) / 8;
  if (n_passes <= 0 || capacity <= 0) return 0;
  if (identity_vals && (end_bit - begin_bit) % 8) return -1;  // identity values need 8-bit digits
  const int width = (end_bit - begin_bit + n_passes - 1) / n_passes;
  constexpr int kTile = kSortThreads * ITEMS;
  const int64_t chunks = (capacity + kTile - 1) / kTile;
  cudaMemsetAsync(tickets, 0, sizeof(uint32_t) * n_passes, s);
  if (!hist_ready) {  // else the producer counted the digits (K6 for the tile sort)
    cudaMemsetAsync(hist, 0, sizeof(uint32_t) * 256 * n_passes, s);
    int hist_grid = (int)std::min<int64_t>(148 * 4, (capacity + kSortThreads - 1) / kSortThreads);
    k_radix_hist<K><<<hist_grid, kSortThreads, 0, s>>>(k0, n_dev, begin_bit, n_passes, width, end_bit, hist);
  }
  launch_pdl(k_radix_hist_scan, (unsigned)std::min<int64_t>(148 * 2, chunks), 256, s, hist, n_passes,
             status, n_dev, (int)kTile);
  K* kin = k0; K* kout = k1;
  uint32_t* vin = v0; uint32_t* vout = v1;
  for (int p = 0; p < n_passes; ++p) {
    const int shift = begin_bit + width * p;
    const int nb = std::min(width, end_bit - shift);
    // identity input values (first pass, 8-bit digits: the depth sort) are
    // generated in the pass instead of read
    const uint32_t* vsrc = (p == 0 && identity_vals) ? nullptr : vin;
    const unsigned g = (unsigned)chunks;
    uint32_t* tk = tickets + p;
    const uint32_t* hp = hist + 256 * p;
    if (!vsrc) {  // identity values (callers use 8-bit digits)
      launch_pass<K, ITEMS, MINB, 8, EARLY, true>(g, s, kin, vsrc, kout, vout, n_dev, shift, hp, status, p, tk);
    } else switch (nb) {
      case 8: launch_pass<K, ITEMS, MINB, 8, EARLY>(g, s, kin, vsrc, kout, vout, n_dev, shift, hp, status, p, tk); break;
      case 7: launch_pass<K, ITEMS, MINB, 7, EARLY>(g, s, kin, vsrc, kout, vout, n_dev, shift, hp, status, p, tk); break;
      case 6: launch_pass<K, ITEMS, MINB, 6, EARLY>(g, s, kin, vsrc, kout, vout, n_dev, shift, hp, status, p, tk); break;
      case 5: launch_pass<K, ITEMS, MINB, 5, EARLY>(g, s, kin, vsrc, kout, vout, n_dev, shift, hp, status, p, tk); break;
      case 4: launch_pass<K, ITEMS, MINB, 4, EARLY>(g, s, kin, vsrc, kout, vout, n_dev, shift, hp, status, p, tk); break;
      case 3: launch_pass<K, ITEMS, MINB, 3, EARLY>(g, s, kin, vsrc, kout, vout, n_dev, shift, hp, status, p, tk); break;
      case 2: launch_pass<K, ITEMS, MINB, 2, EARLY>(g, s, kin, vsrc, kout, vout, n_dev, shift, hp, status, p, tk); break;
      default: launch_pass<K, ITEMS, MINB, 1, EARLY>(g, s, kin, vsrc, kout, vout, n_dev, shift, hp, status, p, tk); break;
    }
    K* t0 = kin; kin = kout; kout = t0;
    uint32_t* t1 = vin; vin = vout; vout = t1;
  }
  return (n_passes & 1) ? 1 : 0;
}

template <typename K>
int radix_sort(K* k0, uint32_t* v0, K* k1, uint32_t* v1, const int64_t* n_dev, int64_t capacity,
               int begin_bit, int end_bit, uint32_t* hist, uint32_t* status, uint32_t* tickets,
               cudaStream_t s, bool hist_ready, bool identity_vals) {
  return radix_sort_items<K, SortCfg<K>::kItems>(k0, v0, k1, v1, n_dev, capacity, begin_bit,
                                                 end_bit, hist, status, tickets, s, hist_ready,
                                                 identity_vals);
}

template int radix_sort<uint64_t>(uint64_t*, uint32_t*, uint64_t*, uint32_t*, const int64_t*,
                                  int64_t, int, int, uint32_t*, uint32_t*, uint32_t*, cudaStream_t,
                                  bool, bool);
template int radix_sort<uint32_t>(uint32_t*, uint32_t*, uint32_t*, uint32_t*, const int64_t*,
                                  int64_t, int, int, uint32_t*, uint32_t*, uint32_t*, cudaStream_t,
                                  bool, bool);

}  // namespace cs

// cs_blend.cu -- K9: per-tile front-to-back alpha blending.
//
// Replaces _kernels.blend_tiles (_kernels.py:17-76), the reference's only
// native kernel.  One CTA per tile, one thread per pixel (tile_size <= 16;
// 4 or 16 pixels per thread for 32/64).  For 16x16 tiles each warp owns an
// 8x4 pixel box.
//
// Every warp walks the tile's splat list (depth order) independently, 32
// entries per round: each lane tests one splat's 8-byte alpha-floor support
// box against the warp's pixel box, __ballot_sync compacts the hits, and the
// warp evaluates only those (64-byte HotRec: mean, conic, opacity, colour,
// fast-reject threshold), so a splat whose support misses the warp's 32
// pixels costs 1/32 of a box test instead of 32 float64 quadratic forms, and
// no warp ever waits at a block barrier for another.  Tiles are launched
// heaviest list first (K8b) so hot-tile lists start in the first wave.
//
// Precision: the quadratic form is float64 in the
// reference's exact op order (no FMA).  A float64 power below
// log(alpha_floor / o) - 1e-6 is a guaranteed skip and costs no exp; every
// other fragment takes the reference path exactly: alpha = min(0.99,
// o * exp(power)) in float64, float64 alpha/transmittance decisions, so the
// accepted-fragment set equals the reference's.  Colour accumulates in
// float32 (SURVEY.md H2 recipe m3: 0 px > 1e-4); a kept-state (training)
// forward also keeps the float64 colour sums its backward re-derives
// (cs_backward.cu).  The AABB cull never drops a fragment the exact path
// could accept: it bounds {power >= threshold} (cs_project.cu).
//
// Staging: 4 x 16-byte cp.async (LDGSTS) per record.  A cp.async.bulk per
// record completing on a per-warp mbarrier was measured 23% slower (1.19 vs
// 0.97 ms on C3, profiles/r2f_blend_ab.txt): the bulk copy takes uniform
// operands, so a warp's scattered 64-byte records are issued one lane at a
// time (ELECT loop), while one LDGSTS moves every hitting lane's chunk.
//
// Accept-phase batching was measured too and not kept: staging up to 32 hits
// per warp, evaluating every quadratic form first and then letting each lane
// walk its own accepted candidates (so a warp iteration serves one fragment of
// every lane) was 29% slower (1.32 vs 0.97 ms; 16-hit batches 1.25 ms,
// profiles/r2k_blend_ab.txt): the quadratic forms of hits staged after a box
// has terminated are wasted, the per-(hit, lane) power array costs shared
// memory and occupancy, and with ~3 hits per round the per-hit accept path it
// replaces is already short.
#include "cs_internal.cuh"

namespace cs {

#ifndef CS_BLEND_THREADS
#define CS_BLEND_THREADS 256
#endif
constexpr int kBlendThreads = CS_BLEND_THREADS;

// Warp-independent blend, persistent: every warp repeatedly takes the next
// work item -- one 8x4 pixel box of one tile, tiles in heaviest-list-first
// order -- from a device-wide ticket, so no warp ever waits for another and a
// CTA's slots are never held by finished warps.  For its box a warp walks the
// tile's depth-ordered list 32 entries per round: each lane reads one entry's
// compact id and packed cull box (pair-major arrays written by K8: coalesced,
// and the 8 boxes of a tile run concurrently so the list stays in L1/L2), a
// __ballot_sync compacts the entries whose alpha-floor box meets the warp's
// pixel box, and each hitting lane cp.async-copies its splat's 64-byte HotRec
// into the warp's shared-memory slot.  The copies of round r are in flight
// while the warp evaluates round r-1 (two stages per warp).  The walk stops
// as soon as the box's 32 pixels have terminated.
template <int PX>
__device__ __forceinline__ int blend_box_pixel(int b, int lane, int ts, int j) {
  return PX == 1 ? box_pixel(b, lane, ts) : box_pixel2(b, lane, ts, j);
}

// PX pixels per lane (1: 8x4 boxes, 2: 8x8 boxes).  With two pixels a lane
// reads each staged record once for both, and a tile is walked by half as
// many warps.
#ifndef CS_BLEND_MINB
#define CS_BLEND_MINB 3   // 3 CTAs/SM (<= 85 registers) for every variant, kept-state included
#endif
#ifndef CS_BLEND_PAIR
#define CS_BLEND_PAIR 0
#endif
constexpr bool kPairHits = CS_BLEND_PAIR != 0;  // evaluate hits two at a time

template <typename OutT, bool KEEP, bool DIAG, int PX>
__global__ void __launch_bounds__(kBlendThreads, CS_BLEND_MINB)
k_blend(const uint32_t* __restrict__ list, const uint32_t* __restrict__ bxs,
        const uint32_t* __restrict__ bys, const uint2* __restrict__ ranges,
        const HotRec* __restrict__ hot, const uint32_t* __restrict__ tile_order, int n_items,
        int nboxes, BlendParams bp, OutT* __restrict__ out, int32_t* __restrict__ frag_tile,
        DevStats* __restrict__ stats, BlendState state) {
  __shared__ __align__(16) HotRec s_hot[kBlendThreads / 32][2][32];
  __shared__ ExpTable s_exp;
  const ExpCoef ec = load_exp_table(&s_exp);
  __syncthreads();
  const int ts = bp.tile_size;
  const uint32_t lane = lane_id();
  const uint32_t lt_mask = (1u << lane) - 1u;
  HotRec (*wbuf)[32] = s_hot[threadIdx.x >> 5];
  long long frags = 0, whits = 0;
  uint32_t evals = 0, whits_empty = 0;  // per lane: well below 2^32 per launch
  for (;;) {
    int item = 0;
    if (lane == 0) item = (int)atomicAdd(&stats->tickets[4], 1u);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_items) break;
    const long long item_t0 = DIAG ? clock64() : 0;
    const int tr = item / nboxes, b = item - tr * nboxes;
    const int t = tile_order ? (int)tile_order[tr] : tr;
    const int tx = t % bp.ntx, ty = t / bp.ntx;
    const uint2 rg = ranges[t];
    const int64_t s0 = rg.x, s1 = rg.y;
    int px[PX], py[PX];
    bool valid[PX], done[PX];
    double sx[PX], sy[PX], T[PX];
    float cr[PX], cg[PX], cb[PX];  // colour accumulates in float32 (SURVEY.md H2 recipe m3)
    double kr[PX], kg[PX], kb[PX];  // KEEP: the float64 sums the backward re-derives
    int cnt[PX];
    int64_t last[PX];
    int x0 = 1 << 20, x1 = -(1 << 20), y0 = 1 << 20, y1 = -(1 << 20);
#pragma unroll
    for (int j = 0; j < PX; ++j) {
      const int li = blend_box_pixel<PX>(b, lane, ts, j);
      px[j] = tx * ts + li % ts;
      py[j] = ty * ts + li / ts;
      valid[j] = li < ts * ts && px[j] < bp.width && py[j] < bp.height;
      if (valid[j]) {
        x0 = min(x0, px[j]); x1 = max(x1, px[j]);
        y0 = min(y0, py[j]); y1 = max(y1, py[j]);
      }
      sx[j] = (double)px[j] + 0.5;  // _kernels.py:43-45
      sy[j] = (double)py[j] + 0.5;
      T[j] = 1.0;
      cr[j] = cg[j] = cb[j] = 0.f;
      kr[j] = kg[j] = kb[j] = 0.0;
      cnt[j] = 0;
      last[j] = s0;
      done[j] = !valid[j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      x0 = min(x0, __shfl_xor_sync(0xffffffffu, x0, o));
      x1 = max(x1, __shfl_xor_sync(0xffffffffu, x1, o));
      y0 = min(y0, __shfl_xor_sync(0xffffffffu, y0, o));
      y1 = max(y1, __shfl_xor_sync(0xffffffffu, y1, o));
    }
    if (x0 > x1) continue;  // no pixel of this box in the image (warp-uniform)

    // one staged round: evaluate its hits (slots 0..popc-1) for this lane's pixels
    // (the quadratic form is computed by terminated pixels too: a branch around
    // it costs more issue slots than the idle lanes' share of the DP pipe)
    // the quadratic form of one hit for this lane's pixels (pure)
    auto quad = [&](const HotRec& h, double (&power)[PX]) {
      const double mx = h.mx, my = h.my, c0 = h.c0, c1 = h.c1, c2 = h.c2;
#pragma unroll
      for (int j = 0; j < PX; ++j) {
        const double dx = dsub(sx[j], mx);
        const double dy = dsub(sy[j], my);
        // -0.5 * (c0*dx*dx + c2*dy*dy) - c1*dx*dy   (_kernels.py:54-57)
        power[j] = dsub(dmul(-0.5, dadd(dmul(dmul(c0, dx), dx), dmul(dmul(c2, dy), dy))),
                        dmul(dmul(c1, dx), dy));
      }
    };
    // the reference's sequential decisions for one hit (_kernels.py:58-72)
    auto accept = [&](const HotRec& h, const double (&power)[PX], int src, int64_t k0) {
      const double lthr = (double)h.lthr;
      bool pass[PX];
#pragma unroll
      for (int j = 0; j < PX; ++j) {
        if (DIAG) evals += done[j] ? 0u : 1u;
        pass[j] = !done[j] && power[j] >= lthr;  // else alpha < alpha_floor guaranteed
      }
      if (DIAG) {
        bool any = false;
#pragma unroll
        for (int j = 0; j < PX; ++j) any |= pass[j];
        if (!__any_sync(0xffffffffu, any)) ++whits_empty;
      }
#pragma unroll
      for (int j = 0; j < PX; ++j) {
        if (!pass[j]) continue;
        double alpha = dmul(h.opacity, exp_le0(power[j], s_exp, ec));  // _kernels.py:58
        if (alpha > ec.clamp) alpha = ec.clamp;      // 0.99, _kernels.py:59-60
        if (alpha < bp.alpha_floor) continue;        // _kernels.py:61-62
        const double nt = dmul(T[j], dsub(1.0, alpha));
        if (nt < bp.t_floor) { done[j] = true; continue; }  // _kernels.py:63-66
        const double wd = dmul(T[j], alpha);
        const float w = (float)wd;
        cr[j] = fmaf(w, h.r, cr[j]);
        cg[j] = fmaf(w, h.g, cg[j]);
        cb[j] = fmaf(w, h.b, cb[j]);
        if (KEEP && CS_BWD_SP_F64) {
          kr[j] = dadd(kr[j], dmul(wd, (double)h.r));
          kg[j] = dadd(kg[j], dmul(wd, (double)h.g));
          kb[j] = dadd(kb[j], dmul(wd, (double)h.b));
        }
        T[j] = nt;
        cnt[j] += 1;
        last[j] = k0 + src + 1;
      }
    };
    // one staged round: its hits (slots 0..popc-1), two at a time so the two
    // independent quadratic-form chains overlap; the decisions stay in order
    auto eval_round = [&](const HotRec* buf, uint32_t mask, int64_t k0) {
      int slot = 0;
      whits += __popc(mask);
      while (mask) {
        const int src0 = __ffs(mask) - 1;
        mask &= mask - 1;
        const HotRec& h0 = buf[slot++];
        double p0[PX];
        quad(h0, p0);
        if (kPairHits && mask) {  // warp-uniform
          const int src1 = __ffs(mask) - 1;
          mask &= mask - 1;
          const HotRec& h1 = buf[slot++];
          double p1[PX];
          quad(h1, p1);
          accept(h0, p0, src0, k0);
          accept(h1, p1, src1, k0);
        } else {
          accept(h0, p0, src0, k0);
        }
      }
    };

    // software-pipelined (id, box) for the next round of 32 entries
    uint32_t nid = 0, nbx = kEmptyBox, nby = kEmptyBox;
    if (s0 + lane < s1) {
      nid = __ldg(list + s0 + lane);
      nbx = __ldg(bxs + s0 + lane);
      nby = __ldg(bys + s0 + lane);
    }
    uint32_t pmask = 0;
    bool live_lane = false;
#pragma unroll
    for (int j = 0; j < PX; ++j) live_lane |= !done[j];
    uint32_t live = __ballot_sync(0xffffffffu, live_lane);
    uint32_t live_px = 0;  // per-lane bitmask of live pixels (box recomputed when it changes)
#pragma unroll
    for (int j = 0; j < PX; ++j) live_px |= (done[j] ? 0u : 1u) << j;
    int64_t pk0 = 0;
    int stage = 0;
    bool alldone = false;
    for (int64_t k0 = s0; k0 < s1; k0 += 32) {
      const uint32_t id = nid, bx = nbx, by = nby;
      if (k0 + 32 + lane < s1) {
        nid = __ldg(list + k0 + 32 + lane);
        nbx = __ldg(bxs + k0 + 32 + lane);
        nby = __ldg(bys + k0 + 32 + lane);
      } else {
        nbx = nby = kEmptyBox;
      }
      const int bx0 = (int)(int16_t)(bx & 0xffffu), bx1 = (int)(int16_t)(bx >> 16);
      const int by0 = (int)(int16_t)(by & 0xffffu), by1 = (int)(int16_t)(by >> 16);
      const bool hit = !(bx0 > x1 || bx1 < x0 || by0 > y1 || by1 < y0);
      const uint32_t mask = __ballot_sync(0xffffffffu, hit);
      if (!mask) continue;
      if (hit) {
        const char* g = reinterpret_cast<const char*>(hot + id);
        char* d = reinterpret_cast<char*>(&wbuf[stage][__popc(mask & lt_mask)]);
#pragma unroll
        for (int c = 0; c < kHotChunks; ++c) cp_async16(d + 16 * c, g + 16 * c);
      }
      cp_async_commit();
      if (pmask) {
        cp_async_wait<1>();
        __syncwarp();
        eval_round(wbuf[stage ^ 1], pmask, pk0);
        __syncwarp();
        uint32_t lp = 0;
#pragma unroll
        for (int j = 0; j < PX; ++j) lp |= (done[j] ? 0u : 1u) << j;
        const uint32_t live_now = __ballot_sync(0xffffffffu, lp != 0);
        if (!live_now) { alldone = true; break; }
        if (__any_sync(0xffffffffu, lp != live_px)) {
          // shrink the warp's cull box to its still-live pixels: a splat that
          // only meets terminated pixels is no longer staged or evaluated
          live_px = lp;
          live = live_now;
          x0 = 1 << 20; x1 = -(1 << 20); y0 = 1 << 20; y1 = -(1 << 20);
#pragma unroll
          for (int j = 0; j < PX; ++j)
            if (!done[j]) {
              x0 = min(x0, px[j]); x1 = max(x1, px[j]);
              y0 = min(y0, py[j]); y1 = max(y1, py[j]);
            }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            x0 = min(x0, __shfl_xor_sync(0xffffffffu, x0, o));
            x1 = max(x1, __shfl_xor_sync(0xffffffffu, x1, o));
            y0 = min(y0, __shfl_xor_sync(0xffffffffu, y0, o));
            y1 = max(y1, __shfl_xor_sync(0xffffffffu, y1, o));
          }
        }
      }
      pmask = mask;
      pk0 = k0;
      stage ^= 1;
    }
    (void)live;
    cp_async_wait<0>();
    __syncwarp();
    if (pmask && !alldone) eval_round(wbuf[stage ^ 1], pmask, pk0);
    __syncwarp();
    int box_cnt = 0;
#pragma unroll
    for (int j = 0; j < PX; ++j) {
      if (!valid[j]) continue;
      box_cnt += cnt[j];
      const int64_t pix = (int64_t)py[j] * bp.width + px[j];
      double o[3] = {(double)cr[j] + T[j] * bp.bg[0], (double)cg[j] + T[j] * bp.bg[1],
                     (double)cb[j] + T[j] * bp.bg[2]};
      if (!(bp.flags & CS_RENDER_NO_CLIP)) {
#pragma unroll
        for (int c = 0; c < 3; ++c) o[c] = o[c] < 0.0 ? 0.0 : (o[c] > 1.0 ? 1.0 : o[c]);
      }
      out[3 * pix] = (OutT)o[0];
      out[3 * pix + 1] = (OutT)o[1];
      out[3 * pix + 2] = (OutT)o[2];
      if (KEEP) {
        state.final_t[pix] = T[j];
        state.last[pix] = (int32_t)last[j];
        state.color_acc[3 * pix] = CS_BWD_SP_F64 ? kr[j] : (double)cr[j];
        state.color_acc[3 * pix + 1] = CS_BWD_SP_F64 ? kg[j] : (double)cg[j];
        state.color_acc[3 * pix + 2] = CS_BWD_SP_F64 ? kb[j] : (double)cb[j];
      }
    }
    const int box_frags = warp_sum(box_cnt);
    frags += box_frags;
    if (lane == 0 && box_frags) atomicAdd(frag_tile + t, box_frags);
    if (DIAG && lane == 0) {
      const unsigned long long dt = (unsigned long long)(clock64() - item_t0);
      atomicMax(reinterpret_cast<unsigned long long*>(&stats->blend_max_item_cycles), dt);
      atomicAdd(reinterpret_cast<unsigned long long*>(&stats->blend_item_cycles), dt);
    }
  }
  const long long wevals = warp_sum((long long)evals);
  if (lane == 0) {
    if (whits) atomicAdd(reinterpret_cast<unsigned long long*>(&stats->warp_hits), (unsigned long long)whits);
    if (DIAG && whits_empty)
      atomicAdd(reinterpret_cast<unsigned long long*>(&stats->warp_hits_empty), (unsigned long long)whits_empty);
    if (frags) atomicAdd(reinterpret_cast<unsigned long long*>(&stats->fragments), (unsigned long long)frags);
    if (wevals) atomicAdd(reinterpret_cast<unsigned long long*>(&stats->evals), (unsigned long long)wevals);
  }
}

#ifndef CS_BLEND_PX
#define CS_BLEND_PX 1
#endif

template <typename OutT, bool KEEP, bool DIAG>
static void launch_blend_d(int n_tiles, const uint32_t* list, const uint32_t* bxs,
                           const uint32_t* bys, const uint2* ranges, const HotRec* hot,
                           const uint32_t* order, const BlendParams& bp, OutT* out,
                           int32_t* frag_tile, DevStats* stats, BlendState st, cudaStream_t s) {
  constexpr int PX = CS_BLEND_PX;
  static int grid = 0;  // persistent: one wave of resident CTAs
  if (grid == 0) grid = persistent_grid(k_blend<OutT, KEEP, DIAG, PX>, kBlendThreads);
  const int nboxes = PX == 1 ? boxes_per_tile(bp.tile_size) : boxes_per_tile2(bp.tile_size);
  k_blend<OutT, KEEP, DIAG, PX><<<grid, kBlendThreads, 0, s>>>(list, bxs, bys, ranges, hot, order,
                                                               n_tiles * nboxes, nboxes, bp, out,
                                                               frag_tile, stats, st);
}

template <typename OutT, bool KEEP>
static void launch_blend_t(int n_tiles, const uint32_t* list, const uint32_t* bxs,
                           const uint32_t* bys, const uint2* ranges, const HotRec* hot,
                           const uint32_t* order, const BlendParams& bp, OutT* out,
                           int32_t* frag_tile, DevStats* stats, BlendState st, cudaStream_t s) {
  if (bp.flags & CS_RENDER_DIAG)
    launch_blend_d<OutT, KEEP, true>(n_tiles, list, bxs, bys, ranges, hot, order, bp, out, frag_tile, stats, st, s);
  else
    launch_blend_d<OutT, KEEP, false>(n_tiles, list, bxs, bys, ranges, hot, order, bp, out, frag_tile, stats, st, s);
}

// K8b: heaviest-first tile order.  Tiles are bucketed by floor(log2(list
// length)) and emitted bucket-descending (order inside a bucket is arbitrary;
// tiles are independent, so the image does not depend on it).  One CTA keeps
// ascending tile ids inside a bucket, which the blend measured faster (L2
// locality of neighbouring tiles' records) than the two-kernel multi-CTA
// form (CS_TILE_ORDER_MULTI=1: 0.934 vs 0.928 ms) despite its 11 us.

#ifndef CS_TILE_ORDER_SHIFT
#define CS_TILE_ORDER_SHIFT 0   // bucket = floor(log2(len)) >> shift (coarser buckets keep more raster order)
#endif
#ifndef CS_TILE_ORDER_SUB
#define CS_TILE_ORDER_SUB 1     // extra mantissa bits per octave (finer heaviest-first order)
#endif
#ifndef CS_TILE_ORDER_RASTER
#define CS_TILE_ORDER_RASTER 0  // 1: no reordering at all
#endif
constexpr int kOrderBuckets = CS_TILE_ORDER_SUB ? (34 << CS_TILE_ORDER_SUB) : 34;

__device__ __forceinline__ int tile_bucket(const uint2* __restrict__ ranges, int t, int n_tiles) {
  if (t >= n_tiles) return -1;
  const uint2 r = ranges[t];
  const uint32_t c = r.y - r.x;
  if (CS_TILE_ORDER_RASTER) return 0;
  if (CS_TILE_ORDER_SUB == 0) return (c ? 32 - __clz(c) : 0) >> CS_TILE_ORDER_SHIFT;
  // finer: floor(log2 c) plus the next CS_TILE_ORDER_SUB bits of c
  if (c < (2u << CS_TILE_ORDER_SUB)) return (int)c;
  const int e = 31 - __clz(c);  // >= SUB + 1
  const int m = (int)((c >> (e - CS_TILE_ORDER_SUB)) & ((1u << CS_TILE_ORDER_SUB) - 1u));
  return (2 << CS_TILE_ORDER_SUB) + ((e - CS_TILE_ORDER_SUB - 1) << CS_TILE_ORDER_SUB) + m;
}

__global__ void k_tile_hist(const uint2* __restrict__ ranges, int n_tiles, int* __restrict__ hist) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int bk = tile_bucket(ranges, t, n_tiles);
  const uint32_t peers = __match_any_sync(0xffffffffu, bk);
  if (bk >= 0 && (peers & lanemask_lt()) == 0) atomicAdd(&hist[bk], __popc(peers));
}

__global__ void k_tile_scatter(const uint2* __restrict__ ranges, int n_tiles, const int* __restrict__ hist,
                               int* __restrict__ cursor, uint32_t* __restrict__ order) {
  __shared__ int s_base[kOrderBuckets];
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int b = kOrderBuckets - 1; b >= 0; --b) { s_base[b] = acc; acc += hist[b]; }
  }
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int bk = tile_bucket(ranges, t, n_tiles);
  const uint32_t peers = __match_any_sync(0xffffffffu, bk);
  const int leader = __ffs(peers) - 1;
  int base = 0;
  if (bk >= 0 && (int)(threadIdx.x & 31) == leader) base = atomicAdd(&cursor[bk], __popc(peers));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (bk >= 0) order[s_base[bk] + base + __popc(peers & lanemask_lt())] = (uint32_t)t;
}

// the single-CTA form (CS_TILE_ORDER_MULTI=0): tiles in ascending id order
// inside a bucket
__global__ void k_tile_order(const uint2* __restrict__ ranges, int n_tiles, uint32_t* __restrict__ order) {
  __shared__ int hist[kOrderBuckets];
  __shared__ int cursor[kOrderBuckets];
  if (threadIdx.x < kOrderBuckets) hist[threadIdx.x] = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) atomicAdd(&hist[tile_bucket(ranges, t, n_tiles)], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int b = kOrderBuckets - 1; b >= 0; --b) { cursor[b] = acc; acc += hist[b]; }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x)
    order[atomicAdd(&cursor[tile_bucket(ranges, t, n_tiles)], 1)] = (uint32_t)t;
}

#ifndef CS_TILE_ORDER_MULTI
#define CS_TILE_ORDER_MULTI 0
#endif

// order: n_tiles entries followed by 2 * kOrderBuckets ints of scratch
void launch_tile_order(const uint2* ranges, int n_tiles, uint32_t* order, cudaStream_t s) {
  if (!CS_TILE_ORDER_MULTI) {
    k_tile_order<<<1, 1024, 0, s>>>(ranges, n_tiles, order);
    return;
  }
  int* hist = reinterpret_cast<int*>(order + n_tiles);
  cudaMemsetAsync(hist, 0, sizeof(int) * 2 * kOrderBuckets, s);
  const int grid = (n_tiles + 255) / 256;
  if (grid == 0) return;
  k_tile_hist<<<grid, 256, 0, s>>>(ranges, n_tiles, hist);
  k_tile_scatter<<<grid, 256, 0, s>>>(ranges, n_tiles, hist, hist + kOrderBuckets, order);
}

int blend_ppt(int tile_size) {  // 0 = unsupported tile size
  return tile_size * tile_size <= 4096 ? 1 : 0;
}

void launch_blend(int n_tiles, const uint32_t* list, const uint32_t* bxs, const uint32_t* bys,
                  const uint2* ranges, const HotRec* hot, const uint32_t* order,
                  const BlendParams& bp, void* out, bool f64_out, int32_t* frag_tile,
                  DevStats* stats, const BlendState* keep, cudaStream_t s) {
  BlendState st = keep ? *keep : BlendState{nullptr, nullptr, nullptr};
  cudaMemsetAsync(frag_tile, 0, sizeof(int32_t) * n_tiles, s);
  cudaMemsetAsync(&stats->tickets[4], 0, sizeof(uint32_t), s);
  if (f64_out) {
    if (keep) launch_blend_t<double, true>(n_tiles, list, bxs, bys, ranges, hot, order, bp, (double*)out, frag_tile, stats, st, s);
    else launch_blend_t<double, false>(n_tiles, list, bxs, bys, ranges, hot, order, bp, (double*)out, frag_tile, stats, st, s);
  } else {
    if (keep) launch_blend_t<float, true>(n_tiles, list, bxs, bys, ranges, hot, order, bp, (float*)out, frag_tile, stats, st, s);
    else launch_blend_t<float, false>(n_tiles, list, bxs, bys, ranges, hot, order, bp, (float*)out, frag_tile, stats, st, s);
  }
}

// ---------------------------------------------------------------------------
// cs_blend_tiles: the numba kernel's exact interface (_kernels.py:18-30).
// Packs the caller's float64 arrays into HotRec records and the int64 CSR into
// (list, ranges); then runs the same blend kernel.  The caller's conics need
// not come from our projection, so no cull box is assumed (infinite AABB).

__global__ void k_pack_records(int64_t m, const double* means, const double* conics,
                               const double* colors, const double* opac, double alpha_floor,
                               HotRec* hot) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m;
       s += (int64_t)gridDim.x * blockDim.x) {
    HotRec h;
    h.mx = means[2 * s]; h.my = means[2 * s + 1];
    h.c0 = conics[3 * s]; h.c1 = conics[3 * s + 1]; h.c2 = conics[3 * s + 2];
    const double o = opac[s];
    h.opacity = o;
    h.r = (float)colors[3 * s]; h.g = (float)colors[3 * s + 1]; h.b = (float)colors[3 * s + 2];
    const double lt = o > 0.0 ? log(alpha_floor / o) - 1e-6
                              : __longlong_as_double(0x7ff0000000000000ll);
    h.lthr = __double2float_rd(lt);
    hot[s] = h;
  }
}

__global__ void k_pack_tiles(int64_t p, const int64_t* tile_ids, int64_t n_tiles,
                             const int64_t* offsets, uint32_t* list, uint32_t* bxs, uint32_t* bys,
                             uint2* ranges) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint32_t full = pack_box(-1, 32000);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += stride) {
    list[i] = (uint32_t)tile_ids[i];
    bxs[i] = full;
    bys[i] = full;
  }
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tiles; t += stride)
    ranges[t] = make_uint2((uint32_t)offsets[t], (uint32_t)offsets[t + 1]);
}

void launch_pack(int64_t m, const double* means, const double* conics, const double* colors,
                 const double* opac, double alpha_floor, HotRec* hot, int64_t p,
                 const int64_t* tile_ids, int64_t n_tiles, const int64_t* offsets, uint32_t* list,
                 uint32_t* bxs, uint32_t* bys, uint2* ranges, cudaStream_t s) {
  if (m > 0)
    k_pack_records<<<148 * 4, 256, 0, s>>>(m, means, conics, colors, opac, alpha_floor, hot);
  k_pack_tiles<<<148 * 4, 256, 0, s>>>(p, tile_ids, n_tiles, offsets, list, bxs, bys, ranges);
}

}  // namespace cs

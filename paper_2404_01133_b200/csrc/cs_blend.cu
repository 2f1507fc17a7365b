// cs_blend.cu -- K9: per-tile front-to-back alpha blending.
//
// Replaces _kernels.blend_tiles (_kernels.py:17-76), the reference's only
// native kernel.  One CTA per tile, one thread per pixel (tile_size <= 16;
// 4 or 16 pixels per thread for 32/64).  For 16x16 tiles each warp owns an
// 4x8 pixel box (CS_BOX_W).
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
// 0.97 ms on C3, profiles/r2k_blend_ab.txt): the bulk copy takes uniform
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
// work item -- one 4x8 pixel box of one tile, tiles in heaviest-list-first
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

// PX pixels per lane (1: 4x8 boxes, 2: 8x8 boxes).  With two pixels a lane
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

// ---------------------------------------------------------------------------
// K9f: the certified float32 blend (frames without kept state).
//
// Same work decomposition as k_blend (persistent warps, 4x8 pixel boxes,
// list rounds of 32 entries culled by box, hit records cp.async-staged two
// rounds deep), but each hit's 64-byte FastRec (cs_internal.cuh) is evaluated
// in float32 on the FMA pipe and MUFU.EX2 instead of the float64 chain.  Every
// reference decision (_kernels.py:52-66) is taken from float32 values only
// when a proven error bound keeps it on the same side of its threshold:
//   * alpha < alpha_floor, in the log2 domain: P32 = log2(alpha32) < Flo
//     skips, P32 >= Fhi accepts (one compare each; the skip test is all an
//     empty hit costs); in between (|P32 - P| <= dP straddles log2(afl)) the
//     fragment's float64 alpha is computed from its HotRec (exact_alpha);
//   * T (1 - alpha) < t_floor: the pixel carries its float32 transmittance T
//     and a bound eT on |T32/T - 1| (each accepted fragment adds
//     eps alpha/(1 - alpha) for the error of (1 - alpha), plus roundings);
//     a termination test inside t_floor (1 +- eT) replays the pixel's
//     transmittance in float64 over the list so far (replay_transmittance)
//     and decides exactly.
// Ill-conditioned splats (FastRec flag) are decided in float64 by every lane.
// So the accepted-fragment set is the exact kernel's; the colour carries
// float32 weights (relative error <= eT + eps, ~1e-5 at worst).
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// float64 alpha of one fragment in the reference's operation order
// (_kernels.py:52-60); 0 when power < lthr (alpha < alpha_floor guaranteed).
__device__ __forceinline__ double exact_alpha(const HotRec& h, double sx, double sy, const ExpTable& tab,
                                              const ExpCoef& ec) {
  const double dx = dsub(sx, h.mx);
  const double dy = dsub(sy, h.my);
  const double power = dsub(dmul(-0.5, dadd(dmul(dmul(h.c0, dx), dx), dmul(dmul(h.c2, dy), dy))),
                            dmul(dmul(h.c1, dx), dy));
  if (!(power >= (double)h.lthr)) return 0.0;
  double a = dmul(h.opacity, exp_le0(power, tab, ec));
  return a > ec.clamp ? ec.clamp : a;
}

__device__ __forceinline__ HotRec load_hot(const HotRec* __restrict__ hot, uint32_t id) {
  const float4* p = reinterpret_cast<const float4*>(hot + id);
  HotRec h;
  float4* q = reinterpret_cast<float4*>(&h);
#pragma unroll
  for (int c = 0; c < kHotChunks; ++c) q[c] = __ldg(p + c);
  return h;
}

__device__ __forceinline__ ExpCoef exp_coef_const() {
  ExpCoef c;
  c.c3 = 1.0 / 6.0;  // == one / 6.0 of load_exp_table (correctly rounded either way)
  c.c4 = 1.0 / 24.0;
  c.c5 = 1.0 / 120.0;
  c.inv = 369.3299304675746; c.hi = -0.0027076061742263846; c.lo = 1.6409824502660487e-13; c.clamp = 0.99;
  return c;
}

// the float64 alpha of splat `id` at pixel (px, py) -- the rare float64
// re-decisions of the fast blend, out of line so they cost it no registers
__device__ __forceinline__ double exact_alpha_at(const HotRec* __restrict__ hot, uint32_t id, int px, int py,
                                              const ExpTable* tab) {
  return exact_alpha(load_hot(hot, id), (double)px + 0.5, (double)py + 0.5, *tab, exp_coef_const());
}

// Float64 transmittance of pixel (px, py) in front of list position kq, and
// the float64 alpha of entry kq (an accepted fragment): the whole warp walks
// [s0, kq] 32 entries per step, each lane tests one entry's cull box and
// evaluates its float64 alpha, then the accepted alphas are applied in list
// order (_kernels.py:50-72).  Entries before kq were all skipped or
// accepted-and-continued by certified decisions, so none terminates the pixel.
// Warp-collective (all 32 lanes, converged).
__device__ __forceinline__ double replay_transmittance(const uint32_t* __restrict__ list,
                                                    const uint32_t* __restrict__ bxs,
                                                    const uint32_t* __restrict__ bys,
                                                    const HotRec* __restrict__ hot, uint32_t s0, uint32_t kq,
                                                    int px, int py, const ExpTable* tab, double alpha_floor,
                                                    double* alpha_kq) {
  const ExpCoef ec = exp_coef_const();
  const uint32_t lane = lane_id();
  const double sx = (double)px + 0.5, sy = (double)py + 0.5;
  double T = 1.0, akq = 0.0;
  uint32_t nid = 0, nbx = kEmptyBox, nby = kEmptyBox;
  if (s0 + lane <= kq) {
    nid = __ldg(list + s0 + lane);
    nbx = __ldg(bxs + s0 + lane);
    nby = __ldg(bys + s0 + lane);
  }
  for (uint32_t base = s0; base <= kq; base += 32) {
    const uint32_t id = nid, bx = nbx, by = nby;
    const uint32_t e = base + 32 + lane;
    if (e <= kq) {
      nid = __ldg(list + e);
      nbx = __ldg(bxs + e);
      nby = __ldg(bys + e);
    } else {
      nbx = nby = kEmptyBox;
    }
    const int bx0 = (int)(int16_t)(bx & 0xffffu), bx1 = (int)(int16_t)(bx >> 16);
    const int by0 = (int)(int16_t)(by & 0xffffu), by1 = (int)(int16_t)(by >> 16);
    double a = 0.0;
    if (px >= bx0 && px <= bx1 && py >= by0 && py <= by1) a = exact_alpha(load_hot(hot, id), sx, sy, *tab, ec);
    uint32_t m = __ballot_sync(0xffffffffu, a >= alpha_floor);
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      const double aj = __shfl_sync(0xffffffffu, a, j);
      if (base + j == kq) {
        akq = aj;
        break;
      }
      T = dmul(T, dsub(1.0, aj));  // _kernels.py:63, 71
    }
  }
  *alpha_kq = akq;
  return T;
}

#ifndef CS_FAST_MINB
#define CS_FAST_MINB 3
#endif
#ifndef CS_FAST_PF
#define CS_FAST_PF 1
#endif
constexpr int kFastPf = CS_FAST_PF;   // list rounds prefetched ahead (k_blend_fast)

// GUARD: every certified bound widened guard_scale-fold (tests only, see
// blend_guard_env); the production instantiation has no guard arithmetic.
template <typename OutT, bool DIAG, bool GUARD>
__global__ void __launch_bounds__(kBlendThreads, CS_FAST_MINB)
k_blend_fast(const uint32_t* __restrict__ list, const uint32_t* __restrict__ bxs,
             const uint32_t* __restrict__ bys, const uint2* __restrict__ ranges,
             const FastRec* __restrict__ fast, const HotRec* __restrict__ hot,
             const uint32_t* __restrict__ tile_order, int n_items, int nboxes, BlendParams bp,
             float guard_scale, OutT* __restrict__ out, int32_t* __restrict__ frag_tile,
             DevStats* __restrict__ stats) {
  constexpr float u = 5.9604645e-8f;
  __shared__ __align__(16) FastRec s_rec[kBlendThreads / 32][2][32];
  __shared__ uint32_t s_id[kBlendThreads / 32][2][32];
  __shared__ ExpTable s_exp;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_exp.t[i] = c_exp2_256[i];
  __syncthreads();
  const int ts = bp.tile_size;
  const uint32_t lane = lane_id();
  const uint32_t lt_mask = (1u << lane) - 1u;
  FastRec (*const wrec)[32] = s_rec[threadIdx.x >> 5];
  uint32_t (*const wid)[32] = s_id[threadIdx.x >> 5];
  // shared-window address of the warp's stages (through an opaque move, so the
  // compiler keeps it in a register instead of re-deriving it from %tid per hit)
  uint32_t wbase;
  asm volatile("mov.b32 %0, %1;" : "=r"(wbase) : "r"(smem_u32(&wrec[0][0])));
  uint32_t frags = 0, whits = 0, evals = 0, whits_empty = 0, n_exact = 0, n_floor = 0, n_replay = 0;
  const float l2afl = (float)log2(bp.alpha_floor);  // GUARD only
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
    const uint32_t s0 = rg.x, s1 = rg.y;
    // the lane's pixel centre (exact in float32, _kernels.py:43-45); integer
    // coordinates are derived from it where needed (px = (int)sx)
    float sx, sy;
    bool valid;
    {
      const int li = box_pixel(b, lane, ts);
      const int px = tx * ts + li % ts, py = ty * ts + li / ts;
      valid = li < ts * ts && px < bp.width && py < bp.height;
      sx = (float)px + 0.5f;
      sy = (float)py + 0.5f;
    }
    float T = 1.f, eT = 0.f, cr = 0.f, cg = 0.f, cb = 0.f;
    int cnt = 0;
    bool done = !valid;
    int x0 = valid ? (int)sx : (1 << 20), x1 = valid ? (int)sx : -(1 << 20);
    int y0 = valid ? (int)sy : (1 << 20), y1 = valid ? (int)sy : -(1 << 20);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      x0 = min(x0, __shfl_xor_sync(0xffffffffu, x0, o));
      x1 = max(x1, __shfl_xor_sync(0xffffffffu, x1, o));
      y0 = min(y0, __shfl_xor_sync(0xffffffffu, y0, o));
      y1 = max(y1, __shfl_xor_sync(0xffffffffu, y1, o));
    }
    if (x0 > x1) continue;  // no pixel of this box in the image (warp-uniform)

    // the nh hits of one staged round, slots in list order; fslot: slots
    // holding a flagged splat's HotRec; mask: the round's hit lanes (list
    // positions k0 + lane), only needed by the rare replays
    // Per-lane step of one accepted-or-not fragment.  a: alpha (float32, or the
    // float64 value rounded), eps: its relative error bound.  Returns false
    // when the termination test falls inside the bound (the lane freezes at
    // this hit; nothing was applied).  Branch-free apart from the caller's.
    auto apply = [&](bool acc, float a, float eps, float fr, float fg, float fb) -> bool {
      const bool clamp = a >= 0.99f;
      const float ac = clamp ? 0.99f : a;
      const float om = clamp ? 0.01f : 1.0f - a;   // 1 - min(alpha, 0.99)  (_kernels.py:59-63)
      const float nt = T * om;
      // |om32/om - 1| <= eps alpha / (1 - alpha) (+ roundings), accumulated into T's bound
      // (+3u roundings: rcp >= 1, so folding 3u into the numerator covers them)
      const float en = fmaf(fmaf(eps, ac, 3.0f * u), rcp_approx(om), eT);
      const float band = fmaf(en, bp.tfl_b, bp.tfl_c);
      const float r = nt - bp.tfl;
      // |r| >= band: the float32 test is the reference's; inside the band the
      // lane freezes (returns false) for a float64 replay
      const bool sure = acc && !(fabsf(r) < band);
      const bool cont = sure && r >= 0.0f;         // _kernels.py:67-72
      const bool stop = sure && r < 0.0f;          // the crossing fragment is dropped (_kernels.py:64-66)
      const float wgt = cont ? T * ac : 0.0f;
      cr = fmaf(wgt, fr, cr);
      cg = fmaf(wgt, fg, cg);
      cb = fmaf(wgt, fb, cb);
      T = cont ? nt : T;
      eT = cont ? en : eT;
      asm("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %1, 0;\n\t@p add.s32 %0, %0, 1;\n\t}" : "+r"(cnt) : "r"((int)cont));
      done = done || stop;
      return sure || !acc;
    };
    // The float32 evaluation of FastRec `ra` for this lane: P32 = log2 of the
    // unclamped alpha, and the alpha-floor pass (P32 >= Flo: may reach the floor).
    auto fast_power = [&](uint32_t ra, float& P) -> bool {
      const float4 q0 = lds128(ra + kFrMean);   // mxh D myh E
      const float4 q1 = lds128(ra + kFrQuad);   // A B C F
      const float flo = lds32(ra + kFrFloor);
      // P = A dx^2 + B dx dy + C dy^2 + log2(o), dx = dxh - mxl, expanded in
      // dxh = sx - mxh: the low parts of the mean sit in D, E, F (cs_internal.cuh)
      const float dxh = sx - q0.x;
      const float dyh = sy - q0.z;
      P = fmaf(fmaf(q1.x, dxh, fmaf(q1.y, dyh, q0.y)), dxh, fmaf(fmaf(q1.z, dyh, q0.w), dyh, q1.w));
      return P >= (GUARD ? flo - (l2afl - flo) * (guard_scale - 1.0f) : flo);  // else skipped (_kernels.py:61-62)
    };
    // ... and for a passing lane: alpha32 = 2^P32, its error bound, and the
    // alpha-floor decision (acc; amb when inside the bound)
    auto fast_alpha = [&](uint32_t ra, float P, float& a, float& eps, bool& acc, bool& amb) {
      const float4 q2 = lds128(ra + kFrFloor);  // flo fhi ek1 ek0
      const float l2o = lds32(ra + kFrColour + 12);
      a = ex2_approx(P);                              // alpha = o exp(power)  (_kernels.py:58)
      eps = fmaf(fabsf(P - l2o), q2.z, q2.w);         // this fragment's alpha error bound
      float fhi = q2.y;
      if (GUARD) {
        eps *= guard_scale;
        fhi = l2afl + (fhi - l2afl) * guard_scale;
      }
      acc = P >= fhi;
      amb = !acc;   // (callers pass only lanes with P >= flo): alpha straddles alpha_floor within its bound
    };

    // the nh hits of one staged round, slots in list order; fslot: slots
    // holding a flagged splat's HotRec; mask: the round's hit lanes (list
    // positions k0 + lane), only needed by the rare float64 resolutions
    auto eval_round = [&](int st_, int nh, uint32_t fslot, uint32_t mask, uint32_t k0) {
      const uint32_t rbase = wbase + (uint32_t)st_ * (32u * (uint32_t)sizeof(FastRec));
      whits += nh;
      int frozen = nh;     // slot this lane stopped at for a float64 resolution (nh: none)
      bool famb = false;   // ... because of its alpha-floor test (else its termination test)
      // one float32-path hit for every lane (warp-converged)
      auto fast_hit = [&](int sl, bool live) {
        const uint32_t ra = rbase + (uint32_t)sl * (uint32_t)sizeof(FastRec);
        float P;
        const bool pass = fast_power(ra, P) && live;
        if (!__any_sync(0xffffffffu, pass)) {
          if (DIAG) whits_empty += lane == 0;
          return;
        }
        float a, eps;
        bool acc, amb;
        fast_alpha(ra, P, a, eps, acc, amb);
        acc = acc && pass;
        amb = amb && pass;
        const float4 q3 = lds128(ra + kFrColour);   // r g b -
        const bool ok = apply(acc, a, eps, q3.x, q3.y, q3.z);
        if (amb || !ok) { frozen = sl; famb = amb; }
      };
      if (fslot == 0) {   // (almost every round) no flagged splat
        for (int sl = 0; sl < nh; ++sl) {
          const bool live = !done && frozen == nh;
          if (DIAG) evals += live ? 1u : 0u;
          fast_hit(sl, live);
        }
      } else {
        for (int sl = 0; sl < nh; ++sl) {
          const bool live = !done && frozen == nh;
          if (DIAG) evals += live ? 1u : 0u;
          if ((fslot >> sl) & 1u) {  // warp-uniform: a flagged splat; float64 decides
            if (DIAG) n_exact += lane == 0;
            if (!__any_sync(0xffffffffu, live)) continue;
            // the slot holds the splat's HotRec (mx my c0 c1 c2 opacity lthr r g b)
            const uint32_t ra = rbase + (uint32_t)sl * (uint32_t)sizeof(FastRec);
            const double dx = dsub((double)sx, lds64(ra)), dy = dsub((double)sy, lds64(ra + 8));
            const double c0 = lds64(ra + 16), c1 = lds64(ra + 24), c2 = lds64(ra + 32);
            const double power = dsub(dmul(-0.5, dadd(dmul(dmul(c0, dx), dx), dmul(dmul(c2, dy), dy))),
                                      dmul(dmul(c1, dx), dy));      // _kernels.py:52-57
            const bool pass = live && power >= (double)lds32(ra + 48);  // else alpha < alpha_floor
            if (!__any_sync(0xffffffffu, pass)) continue;   // no lane reaches the floor
            double ad = 0.0;
            if (pass) {
              const ExpCoef ec = exp_coef_const();
              ad = dmul(lds64(ra + 40), exp_le0(power, s_exp, ec));
              ad = ad > ec.clamp ? ec.clamp : ad;
            }
            const bool acc = pass && ad >= bp.alpha_floor;
            if (!__any_sync(0xffffffffu, acc)) continue;    // nothing accepted: no state changes
            if (!apply(acc, (float)ad, 2.0f * u, lds32(ra + 52), lds32(ra + 56), lds32(ra + 60))) {
              frozen = sl; famb = false;
            }
            continue;
          }
          fast_hit(sl, live);
        }
      }
      // rare: lanes frozen at a hit whose decision fell inside its bound --
      // decide it in float64, then finish the round's remaining hits
      uint32_t fz = __ballot_sync(0xffffffffu, frozen < nh);
      while (fz) {
        bool need_replay = false;
        if (frozen < nh) {
          const int sl = frozen;
          const uint32_t ra = rbase + (uint32_t)sl * (uint32_t)sizeof(FastRec);
          const bool flg = (fslot >> sl) & 1u;
          const float fr = flg ? wrec[st_][sl].as_hot().r : lds32(ra + kFrColour);
          const float fg = flg ? wrec[st_][sl].as_hot().g : lds32(ra + kFrColour + 4);
          const float fb = flg ? wrec[st_][sl].as_hot().b : lds32(ra + kFrColour + 8);
          if (famb) {   // the alpha-floor test in float64, then the termination test as usual
            if (DIAG) ++n_floor;
            const double ad = exact_alpha_at(hot, wid[st_][sl], (int)sx, (int)sy, &s_exp);
            need_replay = !apply(ad >= bp.alpha_floor, (float)ad, 2.0f * u, fr, fg, fb);
          } else {
            need_replay = true;
          }
          if (!need_replay) frozen = nh + 1 + sl;   // resolved: continue after slot sl
        }
        uint32_t rp = __ballot_sync(0xffffffffu, need_replay);
        while (rp) {  // the exact transmittance of each such pixel, one at a time (warp-collective)
          const int l = __ffs(rp) - 1;
          rp &= rp - 1;
          const int qx = (int)__shfl_sync(0xffffffffu, sx, l), qy = (int)__shfl_sync(0xffffffffu, sy, l);
          const int sl = __shfl_sync(0xffffffffu, frozen, l);
          const uint32_t kq = k0 + (uint32_t)(__fns(mask, 0, sl + 1));  // list position of slot sl
          double akq;
          const double Tb = replay_transmittance(list, bxs, bys, hot, s0, kq, qx, qy, &s_exp,
                                                 bp.alpha_floor, &akq);
          if ((int)lane == l) {
            if (DIAG) ++n_replay;
            const uint32_t ra = rbase + (uint32_t)sl * (uint32_t)sizeof(FastRec);
            const bool flg = (fslot >> sl) & 1u;
            const float fr = flg ? wrec[st_][sl].as_hot().r : lds32(ra + kFrColour);
            const float fg = flg ? wrec[st_][sl].as_hot().g : lds32(ra + kFrColour + 4);
            const float fb = flg ? wrec[st_][sl].as_hot().b : lds32(ra + kFrColour + 8);
            const double nt = dmul(Tb, dsub(1.0, akq));
            if (akq < bp.alpha_floor) {
              T = (float)Tb;          // (not reached: the fragment was accepted)
            } else if (nt < bp.t_floor) {
              done = true;
            } else {
              const float wgt = (float)dmul(Tb, akq);
              cr = fmaf(wgt, fr, cr);
              cg = fmaf(wgt, fg, cg);
              cb = fmaf(wgt, fb, cb);
              T = (float)nt;
              ++cnt;
            }
            eT = 2.0f * u;
            frozen = nh + 1 + sl;
          }
        }
        // lane-local continuation over the remaining hits (may freeze again)
        if (frozen > nh) {
          int sl = frozen - nh;   // first slot not yet processed
          frozen = nh;
          for (; sl < nh && !done; ++sl) {
            const uint32_t ra = rbase + (uint32_t)sl * (uint32_t)sizeof(FastRec);
            if ((fslot >> sl) & 1u) {
              const HotRec& h = wrec[st_][sl].as_hot();
              const double ad = exact_alpha(h, (double)sx, (double)sy, s_exp, exp_coef_const());
              if (!apply(ad >= bp.alpha_floor, (float)ad, 2.0f * u, h.r, h.g, h.b)) {
                frozen = sl; famb = false; break;
              }
              continue;
            }
            float P, a, eps;
            bool acc, amb;
            if (!fast_power(ra, P)) continue;
            fast_alpha(ra, P, a, eps, acc, amb);
            if (amb) { frozen = sl; famb = true; break; }
            const float4 q3 = lds128(ra + kFrColour);
            if (!apply(acc, a, eps, q3.x, q3.y, q3.z)) { frozen = sl; famb = false; break; }
          }
        }
        fz = __ballot_sync(0xffffffffu, frozen < nh);
      }
    };


    // (id, box) of the next kFastPf rounds are in flight ahead of the current
    // one: a long list whose entries mostly miss this box is walked at L2
    // throughput, not one L2 latency per 32 entries
    uint32_t rid[kFastPf], rbx[kFastPf], rby[kFastPf];
#pragma unroll
    for (int j = 0; j < kFastPf; ++j) {
      const uint32_t e = s0 + 32u * j + lane;
      rid[j] = 0; rbx[j] = rby[j] = kEmptyBox;
      if (e < s1) {
        rid[j] = __ldg(list + e);
        rbx[j] = __ldg(bxs + e);
        rby[j] = __ldg(bys + e);
      }
    }
    bool live_px = !done;
    uint32_t pmask = 0, pfslot = 0, pk0 = 0;
    int stage = 0;
    bool alldone = false;
    for (uint32_t k0 = s0; k0 < s1; k0 += 32) {
      const uint32_t id = rid[0], bx = rbx[0], by = rby[0];
#pragma unroll
      for (int j = 0; j + 1 < kFastPf; ++j) {
        rid[j] = rid[j + 1]; rbx[j] = rbx[j + 1]; rby[j] = rby[j + 1];
      }
      {
        const uint32_t e = k0 + 32u * kFastPf + lane;
        rbx[kFastPf - 1] = rby[kFastPf - 1] = kEmptyBox;
        if (e < s1) {
          rid[kFastPf - 1] = __ldg(list + e);
          rbx[kFastPf - 1] = __ldg(bxs + e);
          rby[kFastPf - 1] = __ldg(bys + e);
        }
      }
      const int bx0 = (int)(int16_t)(bx & 0xffffu), bx1 = (int)(int16_t)(bx >> 16);
      const int by0 = (int)(int16_t)(by & 0xffffu), by1 = (int)(int16_t)(by >> 16);
      const bool hit = !(bx0 > x1 || bx1 < x0 || by0 > y1 || by1 < y0);
      const uint32_t mask = __ballot_sync(0xffffffffu, hit);
      if (!mask) continue;
      const int slot = __popc(mask & lt_mask);
      const bool flagged = bx0 == kBoxExact;
      const uint32_t fslot = __reduce_or_sync(0xffffffffu, (hit && flagged) ? (1u << slot) : 0u);
      if (hit) {
        const char* g = flagged ? reinterpret_cast<const char*>(hot + id) : reinterpret_cast<const char*>(fast + id);
        char* d = reinterpret_cast<char*>(&wrec[stage][slot]);
#pragma unroll
        for (int c = 0; c < 4; ++c) cp_async16(d + 16 * c, g + 16 * c);
        wid[stage][slot] = id;
      }
      cp_async_commit();
      if (pmask) {
        cp_async_wait<1>();
        __syncwarp();
        eval_round(stage ^ 1, __popc(pmask), pfslot, pmask, pk0);
        __syncwarp();
        const uint32_t live_now = __ballot_sync(0xffffffffu, !done);
        if (!live_now) { alldone = true; break; }
        if (__any_sync(0xffffffffu, done == live_px)) {
          // shrink the warp's cull box to its still-live pixels
          live_px = !done;
          x0 = done ? (1 << 20) : (int)sx; x1 = done ? -(1 << 20) : (int)sx;
          y0 = done ? (1 << 20) : (int)sy; y1 = done ? -(1 << 20) : (int)sy;
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
      pfslot = fslot;
      pk0 = k0;
      stage ^= 1;
    }
    cp_async_wait<0>();
    __syncwarp();
    if (pmask && !alldone) eval_round(stage ^ 1, __popc(pmask), pfslot, pmask, pk0);
    __syncwarp();
    if (valid) {
      const int64_t pix = (int64_t)(int)sy * bp.width + (int)sx;
      double o[3] = {(double)cr + (double)T * bp.bg[0], (double)cg + (double)T * bp.bg[1],
                     (double)cb + (double)T * bp.bg[2]};
      if (!(bp.flags & CS_RENDER_NO_CLIP)) {
#pragma unroll
        for (int c = 0; c < 3; ++c) o[c] = o[c] < 0.0 ? 0.0 : (o[c] > 1.0 ? 1.0 : o[c]);
      }
      out[3 * pix] = (OutT)o[0];
      out[3 * pix + 1] = (OutT)o[1];
      out[3 * pix + 2] = (OutT)o[2];
    }
    const int box_frags = warp_sum(cnt);
    frags += box_frags;
    if (lane == 0 && box_frags) atomicAdd(frag_tile + t, box_frags);
    if (DIAG && lane == 0) {
      const unsigned long long dt = (unsigned long long)(clock64() - item_t0);
      atomicMax(reinterpret_cast<unsigned long long*>(&stats->blend_max_item_cycles), dt);
      atomicAdd(reinterpret_cast<unsigned long long*>(&stats->blend_item_cycles), dt);
    }
  }
  auto add = [&](int64_t* dst, long long v) {
    if (v) atomicAdd(reinterpret_cast<unsigned long long*>(dst), (unsigned long long)v);
  };
  const long long wevals = warp_sum((long long)evals);
  if (DIAG) {
    const long long wf = warp_sum((long long)n_floor), wr = warp_sum((long long)n_replay);
    if (lane == 0) {
      add(&stats->blend_floor_resolved, wf);
      add(&stats->blend_replays, wr);
      add(&stats->blend_exact_hits, n_exact);
      add(&stats->warp_hits_empty, whits_empty);
    }
  }
  if (lane == 0) {
    add(&stats->warp_hits, whits);
    add(&stats->fragments, frags);
    add(&stats->evals, wevals);
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

template <typename OutT, bool DIAG>
static void launch_blend_fast_t(int n_tiles, const uint32_t* list, const uint32_t* bxs, const uint32_t* bys,
                                const uint2* ranges, const FastRec* fast, const HotRec* hot,
                                const uint32_t* order, const BlendParams& bp, float guard, OutT* out,
                                int32_t* frag_tile, DevStats* stats, cudaStream_t s) {
  const int nboxes = boxes_per_tile(bp.tile_size);
  if (guard != 1.0f) {
    static int grid = 0;
    if (grid == 0) grid = persistent_grid(k_blend_fast<OutT, DIAG, true>, kBlendThreads);
    k_blend_fast<OutT, DIAG, true><<<grid, kBlendThreads, 0, s>>>(list, bxs, bys, ranges, fast, hot, order,
                                                                 n_tiles * nboxes, nboxes, bp, guard, out,
                                                                 frag_tile, stats);
    return;
  }
  static int grid = 0;  // persistent: one wave of resident CTAs
  if (grid == 0) grid = persistent_grid(k_blend_fast<OutT, DIAG, false>, kBlendThreads);
  k_blend_fast<OutT, DIAG, false><<<grid, kBlendThreads, 0, s>>>(list, bxs, bys, ranges, fast, hot, order,
                                                                n_tiles * nboxes, nboxes, bp, guard, out,
                                                                frag_tile, stats);
}

// CS_BLEND_EXACT=1: frames without kept state use the float64 kernel too (A/B
// runs).  CS_BLEND_GUARD_SCALE=g (tests only): every certified error bound of
// the float32 blend is widened g-fold, so its float64 re-decisions and
// transmittance replays run on most fragments -- the result must not change.
static bool blend_exact_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("CS_BLEND_EXACT");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}
static float blend_guard_env() {
  static float v = -1.f;
  if (v < 0.f) {
    const char* e = getenv("CS_BLEND_GUARD_SCALE");
    v = e ? (float)atof(e) : 1.0f;
    if (!(v >= 1.0f)) v = 1.0f;
  }
  return v;
}

void launch_blend(int n_tiles, const uint32_t* list, const uint32_t* bxs, const uint32_t* bys,
                  const uint2* ranges, const HotRec* hot, const FastRec* fast, const uint32_t* order,
                  const BlendParams& bp, void* out, bool f64_out, int32_t* frag_tile,
                  DevStats* stats, const BlendState* keep, cudaStream_t s) {
  BlendState st = keep ? *keep : BlendState{nullptr, nullptr, nullptr};
  cudaMemsetAsync(frag_tile, 0, sizeof(int32_t) * n_tiles, s);
  cudaMemsetAsync(&stats->tickets[4], 0, sizeof(uint32_t), s);
  if (!keep && fast && !blend_exact_env()) {
    const float g = blend_guard_env();
    BlendParams bpf = bp;
    bpf.tfl = (float)bp.t_floor;
    bpf.tfl_b = bpf.tfl * 1.01f;
    bpf.tfl_c = bpf.tfl * (4.0f * 5.9604645e-8f);
    bpf.tfl_far = bpf.tfl * 1.5f;
    const bool diag = (bp.flags & CS_RENDER_DIAG) != 0;
    if (f64_out) {
      if (diag) launch_blend_fast_t<double, true>(n_tiles, list, bxs, bys, ranges, fast, hot, order, bpf, g, (double*)out, frag_tile, stats, s);
      else launch_blend_fast_t<double, false>(n_tiles, list, bxs, bys, ranges, fast, hot, order, bpf, g, (double*)out, frag_tile, stats, s);
    } else {
      if (diag) launch_blend_fast_t<float, true>(n_tiles, list, bxs, bys, ranges, fast, hot, order, bpf, g, (float*)out, frag_tile, stats, s);
      else launch_blend_fast_t<float, false>(n_tiles, list, bxs, bys, ranges, fast, hot, order, bpf, g, (float*)out, frag_tile, stats, s);
    }
    return;
  }
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

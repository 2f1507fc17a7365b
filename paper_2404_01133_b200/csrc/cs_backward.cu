// cs_backward.cu -- K10/K11: backward of the forward in cs_project.cu +
// cs_blend.cu, used by per-block training (absent in the reference,
// SPEC.md:76; semantics from SURVEY.md Appendix A "backward-relevant forward
// semantics").
//
// K10 blend backward: the forward's persistent warp-item walk (one 8x4 pixel
// box of one tile per item, lane = pixel), front to back up to the pixel's
// last accepted fragment (kept by the forward).  The
// forward's float64 decisions are re-evaluated identically, so exactly the
// accepted fragments receive gradient; skipped / dropped fragments get none.
// With T_k the transmittance before fragment k, P_k the colour accumulated
// through k and S_k = (C_acc - P_k) + T_end*bg the light arriving from behind,
//     dC/dc_k = T_k a_k,   dC/da_k = T_k c_k - S_k / (1 - a_k)
// and a = min(0.99, o*exp(power)) passes gradient only when unclamped.
// Per-splat partials (mean2d, conic, opacity, colour) are warp-reduced and
// accumulated with one atomicAdd per warp into buffers indexed by splat id.
//
// K11 projection backward: one thread per visible splat; recomputes the
// float64 forward (t, J, V, cov2d) and chains the partials to position,
// scale, rotation (the unnormalised quaternion polynomial of core.py:74-82),
// opacity and SH, including the view-direction term of the colour.
#include <algorithm>

#include "cs_internal.cuh"

namespace cs {

constexpr int kBwdThreads = 256;
constexpr int kGradFields = 9;  // mx, my, c0, c1, c2, opacity, r, g, b
constexpr int kBwdFastSmem = CS_BWD_FAST ? (kBwdThreads / 32) * 2 * 32 * 3 * 16 : 0;  // staged FastRec heads
// CS_BWD_RED_SMEM: the warp's nine float64 partial sums go through a per-warp
// shared-memory transpose (32 x 9 doubles) instead of the shuffle tree
#ifndef CS_BWD_RED_SMEM
#define CS_BWD_RED_SMEM 2   // 1: two lanes per field, 2: three (profiles/r5i_bwd_red3_ab.txt)
#endif
constexpr int kBwdRedSmem = CS_BWD_RED_SMEM ? (kBwdThreads / 32) * 32 * kGradFields * 8 : 0;
constexpr int kBwdDynSmem = kBwdFastSmem + kBwdRedSmem;

struct BwdParams {
  double bg[3];
  double alpha_floor;
  int tile_size, width, height, ntx;
};

// Sums the 9 per-lane partials over the warp with a recursive-halving
// transpose (8 + 4 + 2 + 1 + 1 shuffles for 16 slots instead of 5 per value):
// on return lane l holds the warp total of slot (l >> 1) & 15 (slots >= 9 are
// zero padding), so nine lanes can issue their atomics in one instruction.
#ifndef CS_BWD_RED_F64
#define CS_BWD_RED_F64 1   // reduce the 32 lanes' partials in float64 (cs_internal.cuh)
#endif
#if CS_BWD_RED_F64
typedef double bred_t;
#else
typedef float bred_t;
#endif
// The same result through shared memory: lane l stores its nine partials at
// red[l * 9 + f] (stride 72 B: conflict-free 64-bit stores), then lane
// L < 18 sums half h = L & 1 of field f = L >> 1 (16 rows, the odd half
// starting 8 rows later so the two halves of a field sit 16 banks apart) and
// the pair (2f, 2f + 1) combines with one shuffle: ~45 warp instructions
// instead of the tree's ~110 (double shuffles and selects).
__device__ __forceinline__ double warp_smem_sum9(const float (&in)[kGradFields], uint32_t lane,
                                                 double* __restrict__ red) {
  __syncwarp();  // the previous call's reads are done
#pragma unroll
  for (int f = 0; f < kGradFields; ++f) red[lane * kGradFields + f] = (double)in[f];
  __syncwarp();
  double v = 0.0;
  const int f = (int)(lane >> 1), h = (int)(lane & 1);
  if (lane < 2 * kGradFields) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int row = h * 16 + ((i + 8 * h) & 15);
      v += red[row * kGradFields + f];
    }
  }
  return v + __shfl_xor_sync(0xffffffffu, v, 1);
}

// CS_BWD_RED_SMEM=2: three lanes per field (rows 0-10 / 11-21 / 22-31; lane
// 3f + p), summed with two shuffles into lane 3f: fewer loads per lane
#ifndef CS_BWD_RED_T
#define CS_BWD_RED_T 0  // float rows field-major with a 33-float stride: conflict-free stores and reads
#endif
#ifndef CS_BWD_RED_F32STORE
#define CS_BWD_RED_F32STORE 1  // rows stored as float (exact), widened when summed (profiles/r5l_bwd_f32store_ab.txt)
#endif
__device__ __forceinline__ double warp_smem_sum9_3(const float (&in)[kGradFields], uint32_t lane,
                                                   double* __restrict__ red) {
  float* redf = reinterpret_cast<float*>(red);
  __syncwarp();
#pragma unroll
  for (int f = 0; f < kGradFields; ++f) {
    if (CS_BWD_RED_F32STORE && CS_BWD_RED_T) redf[f * 33 + lane] = in[f];
    else if (CS_BWD_RED_F32STORE) redf[lane * kGradFields + f] = in[f];
    else red[lane * kGradFields + f] = (double)in[f];
  }
  __syncwarp();
  double v = 0.0;
  const int f = (int)(lane / 3u), part = (int)(lane - 3u * (uint32_t)f);
  if (lane < 3 * kGradFields) {
    const int r0 = 11 * part;
#pragma unroll
    for (int i = 0; i < 11; ++i)
      if (part < 2 || i < 10)
        v += CS_BWD_RED_F32STORE && CS_BWD_RED_T ? (double)redf[f * 33 + r0 + i]
             : CS_BWD_RED_F32STORE                ? (double)redf[(r0 + i) * kGradFields + f]
                                                  : red[(r0 + i) * kGradFields + f];
  }
  const double t1 = __shfl_down_sync(0xffffffffu, v, 1);
  const double t2 = __shfl_down_sync(0xffffffffu, v, 2);
  return (v + t1) + t2;  // valid in lane 3f
}

__device__ __forceinline__ bred_t warp_transpose_sum9(const float (&in)[kGradFields], uint32_t lane) {
  bred_t v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = i < kGradFields ? (bred_t)in[i] : (bred_t)0;
#pragma unroll
  for (int o = 16, n = 16; o >= 2; o >>= 1, n >>= 1) {
    const bool upper = (lane & o) != 0;
    const int h = n >> 1;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const bred_t send = upper ? v[i] : v[i + h];
      const bred_t keep = upper ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// Same persistent warp-item walk as the forward (cs_blend.cu): per round of 32
// list entries a coalesced read of (id, packed box), a ballot of the hits
// against the warp's pixel box, cp.async staging of the hits' HotRecs into
// the warp's two-stage shared buffer.  A warp walks only up to the largest
// `last` of its pixels.  Per evaluated hit each lane re-derives the forward's
// float64 decisions for its pixel; when any lane contributes, the nine
// partials are warp-reduced and lane 0 adds them with one atomic each.
#ifndef CS_BWD_MINB
#define CS_BWD_MINB 2
#endif
#ifndef CS_BWD_PX
#define CS_BWD_PX 2
#endif

template <int PX>
__device__ __forceinline__ int bwd_box_pixel(int b, int lane, int ts, int j) {
  return PX == 1 ? box_pixel(b, lane, ts) : box_pixel2(b, lane, ts, j);
}

// PX pixels per lane (1: 8x4 boxes, 2: 8x8 boxes): with two, a lane sums its
// pixels' partials before the warp reduction, halving reductions and atomics.
template <int PX>
__global__ void __launch_bounds__(kBwdThreads, CS_BWD_MINB)
k_blend_bwd(const uint32_t* __restrict__ list, const uint32_t* __restrict__ bxs,
            const uint32_t* __restrict__ bys, const uint2* __restrict__ ranges,
            const HotRec* __restrict__ hot, const FastRec* __restrict__ fast,
            const uint32_t* __restrict__ tile_order, int n_items,
            int nboxes, BwdParams bp, const float* __restrict__ dl_dimg, BlendState state,
            uint32_t* __restrict__ ticket, gacc_t* __restrict__ grads /* [kGradFields][cap] */,
            int64_t cap) {
  __shared__ __align__(16) HotRec s_hot[kBwdThreads / 32][2][32];
  // CS_BWD_FAST: the hits' FastRec heads (mxh D myh E | A B C F | flo fhi ek1 ek0),
  // dynamic shared memory (kBwdFastSmem bytes; the static total would pass 48 KB)
  extern __shared__ __align__(16) float4 s_fq[];  // [kBwdFastSmem | kBwdRedSmem]
  double* red = reinterpret_cast<double*>(reinterpret_cast<char*>(s_fq) + kBwdFastSmem) +
                (threadIdx.x >> 5) * 32 * kGradFields;
  __shared__ ExpTable s_exp;
  const ExpCoef ec = load_exp_table(&s_exp);
  __syncthreads();
  const int ts = bp.tile_size;
  const uint32_t lane = lane_id();
  const uint32_t lt_mask = (1u << lane) - 1u;
  HotRec (*wbuf)[32] = s_hot[threadIdx.x >> 5];
  float4 (*fbuf)[32][3] = reinterpret_cast<float4 (*)[32][3]>(s_fq + (threadIdx.x >> 5) * 2 * 32 * 3);
  const bool use_fast = CS_BWD_FAST && fast != nullptr;
  const bsp_t bg[3] = {(bsp_t)bp.bg[0], (bsp_t)bp.bg[1], (bsp_t)bp.bg[2]};
  for (;;) {
    int item = 0;
    if (lane == 0) item = (int)atomicAdd(ticket, 1u);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_items) break;
    const int tr = item / nboxes, b = item - tr * nboxes;
    const int t = tile_order ? (int)tile_order[tr] : tr;
    const int tx = t % bp.ntx, ty = t / bp.ntx;
    const uint2 rg = ranges[t];
    const int64_t s0 = rg.x, s1 = rg.y;
    int px[PX], py[PX];
    bool valid[PX];
    int64_t my_end[PX];
    // The accept decisions replay the forward's float64 arithmetic exactly
    // (float64 alpha and transmittance); the light arriving from behind a
    // fragment, S_k = (C_acc - P_k) + T_end bg, is formed in float64 from the
    // forward's float64 colour sums, so it carries no float32 cancellation
    // bias (it is divided by 1 - alpha >= 0.01); the per-splat partials are
    // float32.
    bsp_t g[PX][3], acc[PX][3], Tend[PX], T[PX], P[PX][3];
    double sx[PX], sy[PX];
    float fsx[PX], fsy[PX];  // pixel centres in float (exact)
    int x0 = 1 << 20, x1 = -(1 << 20), y0 = 1 << 20, y1 = -(1 << 20), wend = (int)s0;
#pragma unroll
    for (int j = 0; j < PX; ++j) {
      const int li = bwd_box_pixel<PX>(b, lane, ts, j);
      px[j] = tx * ts + li % ts;
      py[j] = ty * ts + li / ts;
      valid[j] = li < ts * ts && px[j] < bp.width && py[j] < bp.height;
      my_end[j] = s0;
      Tend[j] = 1;
      T[j] = 1;
#pragma unroll
      for (int c = 0; c < 3; ++c) g[j][c] = acc[j][c] = P[j][c] = 0;
      if (valid[j]) {
        const int64_t pix = (int64_t)py[j] * bp.width + px[j];
        my_end[j] = state.last[pix];
        const double te = state.final_t[pix];
        Tend[j] = (bsp_t)te;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double a = state.color_acc[3 * pix + c];
          acc[j][c] = (bsp_t)a;
          const double o = a + te * bp.bg[c];  // unclipped pixel value
          // clip to [0, 1] (render.py:273): gradient passes where 0 <= C <= 1
          g[j][c] = (o >= 0.0 && o <= 1.0) ? (bsp_t)dl_dimg[3 * pix + c] : (bsp_t)0;
        }
        x0 = min(x0, px[j]); x1 = max(x1, px[j]);
        y0 = min(y0, py[j]); y1 = max(y1, py[j]);
        wend = max(wend, (int)my_end[j]);
      }
      sx[j] = (double)px[j] + 0.5;
      sy[j] = (double)py[j] + 0.5;
      fsx[j] = (float)px[j] + 0.5f;
      fsy[j] = (float)py[j] + 0.5f;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      x0 = min(x0, __shfl_xor_sync(0xffffffffu, x0, o));
      x1 = max(x1, __shfl_xor_sync(0xffffffffu, x1, o));
      y0 = min(y0, __shfl_xor_sync(0xffffffffu, y0, o));
      y1 = max(y1, __shfl_xor_sync(0xffffffffu, y1, o));
      wend = max(wend, __shfl_xor_sync(0xffffffffu, wend, o));
    }
    if (x0 > x1) continue;  // warp-uniform
    const int64_t e1 = min((int64_t)wend, s1);

    // ids: each lane's list entry of the staged round (the hit's splat id is
    // the entry of lane src, the gradient slot of its atomics)
    auto eval_round = [&](const HotRec* buf, const float4 (*fb)[3], uint32_t mask, int64_t k0, uint32_t ids) {
      int slot = 0;
      while (mask) {
        const int src = __ffs(mask) - 1;
        mask &= mask - 1;
        // certified float32 pre-reject (make_fast_rec's bound; flagged and
        // never-passing splats have ek0 == 0 and are always evaluated exactly)
        float4 q0 = make_float4(0.f, 0.f, 0.f, 0.f), q1 = q0;
        float flo = -__int_as_float(0x7f800000);
        if (use_fast) {
          q0 = fb[slot][0];
          q1 = fb[slot][1];
          const float4 q2 = fb[slot][2];
          if (q2.w != 0.f) flo = q2.x;
        }
        const HotRec& h = buf[slot++];
        const uint32_t hid = __shfl_sync(0xffffffffu, ids, src);
        const double mx = h.mx, my = h.my, c0 = h.c0, c1 = h.c1, c2 = h.c2, lthr = (double)h.lthr;
        float gr[kGradFields];
#pragma unroll
        for (int f = 0; f < kGradFields; ++f) gr[f] = 0.f;
        bool contrib = false;
#pragma unroll
        for (int j = 0; j < PX; ++j) {
          if (use_fast) {
            const float dxh = fsx[j] - q0.x, dyh = fsy[j] - q0.z;
            const float P = fmaf(fmaf(q1.x, dxh, fmaf(q1.y, dyh, q0.y)), dxh,
                                 fmaf(fmaf(q1.z, dyh, q0.w), dyh, q1.w));
            if (P < flo) continue;  // alpha < alpha_floor for sure: not accepted by the forward
          }
          // the quadratic form for every remaining lane (cheaper than a branch)
          const double dx = dsub(sx[j], mx), dy = dsub(sy[j], my);
          const double power = dsub(dmul(-0.5, dadd(dmul(dmul(c0, dx), dx), dmul(dmul(c2, dy), dy))),
                                    dmul(dmul(c1, dx), dy));
          if (k0 + src < my_end[j] && power >= lthr) {
            const double G = exp_le0(power, s_exp, ec);
            double alpha = dmul(h.opacity, G);
            const bool clamped = alpha > ec.clamp;  // 0.99: d alpha = 0
            if (clamped) alpha = ec.clamp;
            if (alpha >= bp.alpha_floor) {
              contrib = true;
              const float col[3] = {h.r, h.g, h.b};
              bsp_t dl_da = 0;
              bsp_t w;
              if (CS_BWD_SP_F64) {
                w = (bsp_t)dmul((double)T[j], alpha);   // as the forward's kept float64 sums
                const double om = dsub(1.0, alpha);        // >= 0.01
                double inv = (double)__frcp_rn((float)om);   // + one Newton step: ~1e-14
                inv = fma(inv, fma(-om, inv, 1.0), inv);
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                  P[j][c] = (bsp_t)dadd((double)P[j][c], dmul((double)w, (double)col[c]));
                  const bsp_t S = (acc[j][c] - P[j][c]) + Tend[j] * bg[c];
                  dl_da += g[j][c] * (T[j] * (bsp_t)col[c] - S * inv);
                  gr[6 + c] += (float)(w * g[j][c]);
                }
              } else {
                const float af = (float)alpha;
                w = T[j] * af;
                const float inv = 1.f / (1.f - af);
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                  P[j][c] = fmaf(w, col[c], P[j][c]);
                  const float S = (acc[j][c] - P[j][c]) + Tend[j] * bg[c];
                  dl_da += g[j][c] * (T[j] * col[c] - S * inv);
                  gr[6 + c] += w * g[j][c];
                }
              }
              const float a = (float)alpha;
              const float dl_dpow = clamped ? 0.f : (float)dl_da * a;
              const float fdx = (float)dx, fdy = (float)dy;
              gr[5] += clamped ? 0.f : (float)(dl_da * G);
              gr[0] += dl_dpow * ((float)c0 * fdx + (float)c1 * fdy);
              gr[1] += dl_dpow * ((float)c2 * fdy + (float)c1 * fdx);
              gr[2] += dl_dpow * (-0.5f * fdx * fdx);
              gr[3] += dl_dpow * (-fdx * fdy);
              gr[4] += dl_dpow * (-0.5f * fdy * fdy);
              if (CS_BWD_SP_F64) T[j] = (bsp_t)dmul((double)T[j], dsub(1.0, alpha));
              else T[j] *= 1.f - (float)alpha;
            }
          }
        }
        if (__any_sync(0xffffffffu, contrib)) {
          if (CS_BWD_RED_SMEM == 2 && CS_BWD_RED_F64) {
            const double v = warp_smem_sum9_3(gr, lane, red);
            const uint32_t f = lane / 3u;
            if (lane == 3u * f && f < kGradFields && v != 0.0)
              atomicAdd(&grads[(int64_t)f * cap + hid], (gacc_t)v);
          } else {
            const bred_t v = CS_BWD_RED_SMEM && CS_BWD_RED_F64 ? (bred_t)warp_smem_sum9(gr, lane, red)
                                                               : warp_transpose_sum9(gr, lane);
            const uint32_t f = (lane >> 1) & 15;
            if (!(lane & 1) && f < kGradFields && v != (bred_t)0)
              atomicAdd(&grads[(int64_t)f * cap + hid], (gacc_t)v);
          }
        }
      }
    };

    uint32_t nid = 0, nbx = kEmptyBox, nby = kEmptyBox;
    if (s0 + lane < e1) {
      nid = __ldg(list + s0 + lane);
      nbx = __ldg(bxs + s0 + lane);
      nby = __ldg(bys + s0 + lane);
    }
    uint32_t pmask = 0, pid = 0;
    uint32_t live_px = 0;  // per-lane bitmask of pixels still needing entries
#pragma unroll
    for (int j = 0; j < PX; ++j) live_px |= (valid[j] && my_end[j] > s0 ? 1u : 0u) << j;
    int64_t pk0 = 0;
    int stage = 0;
    for (int64_t k0 = s0; k0 < e1; k0 += 32) {
      const uint32_t id = nid, bx = nbx, by = nby;
      if (k0 + 32 + lane < e1) {
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
        const char* gp = reinterpret_cast<const char*>(hot + id);
        char* d = reinterpret_cast<char*>(&wbuf[stage][__popc(mask & lt_mask)]);
#pragma unroll
        for (int c = 0; c < kHotChunks; ++c) cp_async16(d + 16 * c, gp + 16 * c);
        if (use_fast) {
          const char* fp = reinterpret_cast<const char*>(fast + id);
          char* fd = reinterpret_cast<char*>(fbuf[stage][__popc(mask & lt_mask)]);
#pragma unroll
          for (int c = 0; c < 3; ++c) cp_async16(fd + 16 * c, fp + 16 * c);
        }
      }
      cp_async_commit();
      if (pmask) {
        cp_async_wait<1>();
        __syncwarp();
        eval_round(wbuf[stage ^ 1], fbuf[stage ^ 1], pmask, pk0, pid);
        __syncwarp();
      }
      // shrink the cull box to the pixels whose last fragment lies beyond
      // this round (as in the forward: entries that only meet finished
      // pixels are neither staged nor evaluated)
      uint32_t lp = 0;
#pragma unroll
      for (int j = 0; j < PX; ++j) lp |= (valid[j] && my_end[j] > k0 + 32 ? 1u : 0u) << j;
      if (__any_sync(0xffffffffu, lp != live_px)) {
        live_px = lp;
        x0 = 1 << 20; x1 = -(1 << 20); y0 = 1 << 20; y1 = -(1 << 20);
#pragma unroll
        for (int j = 0; j < PX; ++j)
          if (lp & (1u << j)) {
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
      pmask = mask;
      pk0 = k0;
      pid = id;
      stage ^= 1;
    }
    cp_async_wait<0>();
    __syncwarp();
    if (pmask) eval_round(wbuf[stage ^ 1], fbuf[stage ^ 1], pmask, pk0, pid);
    __syncwarp();
  }
}

__constant__ double kB0 = 0.28209479177387814;
__constant__ double kB1 = 0.4886025119029199;
__constant__ double kB2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                              -1.0925484305920792, 0.5462742152960396};
__constant__ double kB3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                              0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                              -0.5900435899266435};

// Visits every SH basis function n <= degree with its value Y_n and its
// gradient (gx, gy, gz) w.r.t. the unit direction (core.py:114-146), without
// materialising 16 x 4 arrays (the previous form spilled 512 B per thread).
template <typename F>
__device__ __forceinline__ void for_sh_basis(double x, double y, double z, int degree, F&& f) {
  f(0, kB0, 0.0, 0.0, 0.0);
  if (degree < 1) return;
  f(1, -kB1 * y, 0.0, -kB1, 0.0);
  f(2, kB1 * z, 0.0, 0.0, kB1);
  f(3, -kB1 * x, -kB1, 0.0, 0.0);
  if (degree < 2) return;
  const double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  f(4, kB2[0] * xy, kB2[0] * y, kB2[0] * x, 0.0);
  f(5, kB2[1] * yz, 0.0, kB2[1] * z, kB2[1] * y);
  f(6, kB2[2] * (2.0 * zz - xx - yy), -2.0 * kB2[2] * x, -2.0 * kB2[2] * y, 4.0 * kB2[2] * z);
  f(7, kB2[3] * xz, kB2[3] * z, 0.0, kB2[3] * x);
  f(8, kB2[4] * (xx - yy), 2.0 * kB2[4] * x, -2.0 * kB2[4] * y, 0.0);
  if (degree < 3) return;
  f(9, kB3[0] * y * (3.0 * xx - yy), 6.0 * kB3[0] * xy, kB3[0] * (3.0 * xx - 3.0 * yy), 0.0);
  f(10, kB3[1] * xy * z, kB3[1] * yz, kB3[1] * xz, kB3[1] * xy);
  f(11, kB3[2] * y * (4.0 * zz - xx - yy), -2.0 * kB3[2] * xy, kB3[2] * (4.0 * zz - xx - 3.0 * yy),
    8.0 * kB3[2] * yz);
  f(12, kB3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy), -6.0 * kB3[3] * xz, -6.0 * kB3[3] * yz,
    kB3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy));
  f(13, kB3[4] * x * (4.0 * zz - xx - yy), kB3[4] * (4.0 * zz - 3.0 * xx - yy), -2.0 * kB3[4] * xy,
    8.0 * kB3[4] * xz);
  f(14, kB3[5] * z * (xx - yy), 2.0 * kB3[5] * xz, -2.0 * kB3[5] * yz, kB3[5] * (xx - yy));
  f(15, kB3[6] * x * (xx - 3.0 * yy), kB3[6] * (3.0 * xx - 3.0 * yy), -6.0 * kB3[6] * xy, 0.0);
}

__device__ __forceinline__ int deg_of(int c) { return c >= 16 ? 3 : c >= 9 ? 2 : c >= 4 ? 1 : 0; }

// K11a: geometry.  One thread per cloud row k (= splat id of the single-cloud
// source), in row order so every parameter, partial and gradient access is
// coalesced; rows the forward culled (depth key ~0) get zero gradients, so the
// output buffers need no separate clear.  Writes dL/d{position (without the
// view-direction term of the colour, added by K11b), scale, rotation,
// opacity}.
__global__ void __launch_bounds__(128)
k_project_bwd_geom(const cs_cloud cl, const uint64_t* __restrict__ depth_keys, cs_camera cam,
              cs_settings st, const gacc_t* __restrict__ grads, int64_t cap, cs_grads out) {
  const int64_t K = cl.count;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < K;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (depth_keys[k] == ~0ull) {  // culled by the forward projection: no gradient
      for (int i = 0; i < 3; ++i) out.positions[3 * k + i] = out.scales[3 * k + i] = 0.f;
      for (int i = 0; i < 4; ++i) out.rotations[4 * k + i] = 0.f;
      out.opacities[k] = 0.f;
      continue;
    }
    const Geom gm = load_geom(cl, k);
    float gin[kGradFields];
#pragma unroll
    for (int f = 0; f < kGradFields; ++f) gin[f] = grads[(int64_t)f * cap + k];
    const double* W = cam.R;
    // camera-space position
    double tcam[3];
    for (int i = 0; i < 3; ++i)
      tcam[i] = W[3 * i] * gm.px + W[3 * i + 1] * gm.py + W[3 * i + 2] * gm.pz + cam.t[i];
    const double z = tcam[2], iz = 1.0 / z, iz2 = iz * iz, iz3 = iz2 * iz;
    // rotation and covariance
    const double w = gm.qw, x = gm.qx, y = gm.qy, q = gm.qz;
    double R[9] = {1.0 - 2.0 * (y * y + q * q), 2.0 * (x * y - w * q), 2.0 * (x * q + w * y),
                   2.0 * (x * y + w * q), 1.0 - 2.0 * (x * x + q * q), 2.0 * (y * q - w * x),
                   2.0 * (x * q - w * y), 2.0 * (y * q + w * x), 1.0 - 2.0 * (x * x + y * y)};
    const double s[3] = {gm.sx, gm.sy, gm.sz};
    double Mm[9];  // M = R diag(s)
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) Mm[3 * i + j] = R[3 * i + j] * s[j];
    double Sig[9];
    for (int i = 0; i < 3; ++i)
      for (int l = 0; l < 3; ++l)
        Sig[3 * i + l] = Mm[3 * i] * Mm[3 * l] + Mm[3 * i + 1] * Mm[3 * l + 1] + Mm[3 * i + 2] * Mm[3 * l + 2];
    double V[9], WS[9];
    for (int i = 0; i < 3; ++i)
      for (int l = 0; l < 3; ++l)
        WS[3 * i + l] = W[3 * i] * Sig[l] + W[3 * i + 1] * Sig[3 + l] + W[3 * i + 2] * Sig[6 + l];
    for (int i = 0; i < 3; ++i)
      for (int m = 0; m < 3; ++m)
        V[3 * i + m] = WS[3 * i] * W[3 * m] + WS[3 * i + 1] * W[3 * m + 1] + WS[3 * i + 2] * W[3 * m + 2];
    const double J[6] = {cam.fx * iz, 0.0, -cam.fx * tcam[0] * iz2,
                         0.0, cam.fy * iz, -cam.fy * tcam[1] * iz2};
    // cov2d + low pass
    double JV[6];
    for (int i = 0; i < 2; ++i)
      for (int l = 0; l < 3; ++l)
        JV[3 * i + l] = J[3 * i] * V[l] + J[3 * i + 1] * V[3 + l] + J[3 * i + 2] * V[6 + l];
    const double a = JV[0] * J[0] + JV[1] * J[1] + JV[2] * J[2] + st.low_pass;
    const double b = JV[0] * J[3] + JV[1] * J[4] + JV[2] * J[5];
    const double c = JV[3] * J[3] + JV[4] * J[4] + JV[5] * J[5] + st.low_pass;
    const double det = a * c - b * b, id2 = 1.0 / (det * det);
    // conic -> (a, b, c)
    const double g0 = gin[2], g1 = gin[3], g2 = gin[4];
    const double dA = g0 * (-c * c * id2) + g1 * (b * c * id2) + g2 * (1.0 / det - a * c * id2);
    const double dB = g0 * (2.0 * b * c * id2) + g1 * (-1.0 / det - 2.0 * b * b * id2) +
                      g2 * (2.0 * a * b * id2);
    const double dC = g0 * (1.0 / det - a * c * id2) + g1 * (a * b * id2) + g2 * (-a * a * id2);
    const double G[4] = {dA, 0.5 * dB, 0.5 * dB, dC};  // symmetric dL/dcov2d
    // dL/dV = J^T G J ; dL/dJ = 2 G J V
    double GJ[6];
    for (int i = 0; i < 2; ++i)
      for (int l = 0; l < 3; ++l) GJ[3 * i + l] = G[2 * i] * J[l] + G[2 * i + 1] * J[3 + l];
    double dV[9];
    for (int j = 0; j < 3; ++j)
      for (int l = 0; l < 3; ++l) dV[3 * j + l] = J[j] * GJ[l] + J[3 + j] * GJ[3 + l];
    double dJ[6];
    for (int i = 0; i < 2; ++i)
      for (int l = 0; l < 3; ++l)
        dJ[3 * i + l] = 2.0 * (GJ[3 * i] * V[l] + GJ[3 * i + 1] * V[3 + l] + GJ[3 * i + 2] * V[6 + l]);
    // dL/dt from J and mean2d
    const double gmx = gin[0], gmy = gin[1];
    double dt[3];
    dt[0] = dJ[2] * (-cam.fx * iz2) + gmx * cam.fx * iz;
    dt[1] = dJ[5] * (-cam.fy * iz2) + gmy * cam.fy * iz;
    dt[2] = dJ[0] * (-cam.fx * iz2) + dJ[2] * (2.0 * cam.fx * tcam[0] * iz3) +
            dJ[4] * (-cam.fy * iz2) + dJ[5] * (2.0 * cam.fy * tcam[1] * iz3) -
            gmx * cam.fx * tcam[0] * iz2 - gmy * cam.fy * tcam[1] * iz2;
    double dp[3];
    for (int i = 0; i < 3; ++i) dp[i] = W[i] * dt[0] + W[3 + i] * dt[1] + W[6 + i] * dt[2];
    // dL/dSigma = W^T dV W (symmetrised)
    double tmp[9], dS[9];
    for (int j = 0; j < 3; ++j)
      for (int m = 0; m < 3; ++m) tmp[3 * j + m] = W[j] * dV[m] + W[3 + j] * dV[3 + m] + W[6 + j] * dV[6 + m];
    for (int j = 0; j < 3; ++j)
      for (int l = 0; l < 3; ++l)
        dS[3 * j + l] = tmp[3 * j] * W[l] + tmp[3 * j + 1] * W[3 + l] + tmp[3 * j + 2] * W[6 + l];
    double dSs[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) dSs[3 * i + j] = dS[3 * i + j] + dS[3 * j + i];
    // Sigma = M M^T: dL/dM = (dS + dS^T) M
    double dM[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        dM[3 * i + j] = dSs[3 * i] * Mm[j] + dSs[3 * i + 1] * Mm[3 + j] + dSs[3 * i + 2] * Mm[6 + j];
    double ds[3] = {0.0, 0.0, 0.0}, dR[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        ds[j] += dM[3 * i + j] * R[3 * i + j];
        dR[3 * i + j] = dM[3 * i + j] * s[j];
      }
    double dq[4];
    dq[0] = 2.0 * (-q * dR[1] + y * dR[2] + q * dR[3] - x * dR[5] - y * dR[6] + x * dR[7]);
    dq[1] = 2.0 * (y * dR[1] + q * dR[2] + y * dR[3] - 2.0 * x * dR[4] - w * dR[5] + q * dR[6] +
                   w * dR[7] - 2.0 * x * dR[8]);
    dq[2] = 2.0 * (-2.0 * y * dR[0] + x * dR[1] + w * dR[2] + x * dR[3] + q * dR[5] - w * dR[6] +
                   q * dR[7] - 2.0 * y * dR[8]);
    dq[3] = 2.0 * (-2.0 * q * dR[0] - w * dR[1] + x * dR[2] + w * dR[3] - 2.0 * q * dR[4] +
                   y * dR[5] + x * dR[6] + y * dR[7]);
    for (int i = 0; i < 3; ++i) {
      out.positions[3 * k + i] = (float)dp[i];
      out.scales[3 * k + i] = (float)ds[i];
    }
    for (int i = 0; i < 4; ++i) out.rotations[4 * k + i] = (float)dq[i];
    out.opacities[k] = gin[5];
  }
}

// K11b: colour.  dL/dsh = gc * Y_n for the channels the forward's clip passed
// (core.py:169-172), and the view-direction term of the colour added to
// K11a's position gradient.  A warp owns 32 consecutive rows: their SH rows
// (contiguous in HBM) are staged into shared memory with coalesced float4
// loads (row pitch padded to an odd word count: conflict-free per-lane
// access), each lane evaluates its row and overwrites it with the gradient in
// place, and the warp stores the 32 gradient rows coalesced.
constexpr int kShBwdThreads = 256;

__global__ void __launch_bounds__(kShBwdThreads)
k_project_bwd_sh(const cs_cloud cl, const uint64_t* __restrict__ depth_keys, cs_camera cam,
                 cs_settings st, const gacc_t* __restrict__ grads, int64_t cap, cs_grads out,
                 int pitch) {
  extern __shared__ float s_rows[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* buf = s_rows + (size_t)warp * 32 * pitch;
  const int64_t K = cl.count;
  const int C = cl.sh_coeffs, C3 = 3 * C, stride = cl.sh_stride;
  const int degree = min((int)st.sh_degree, deg_of(C));
  const int nb = (degree + 1) * (degree + 1);
  const float inv_stride = 1.f / (float)stride, inv_c3 = 1.f / (float)C3;
  for (int64_t base = ((int64_t)blockIdx.x * (kShBwdThreads / 32) + warp) * 32; base < K;
       base += (int64_t)gridDim.x * (kShBwdThreads / 32) * 32) {
    const int n_rows = (int)min((int64_t)32, K - base);
    {  // stage the rows (stride % 4 == 0: float4 loads)
      const float4* src = reinterpret_cast<const float4*>(cl.sh + base * stride);
      const int n4 = n_rows * stride / 4;
      for (int i = lane; i < n4; i += 32) {
        const float4 v = __ldg(src + i);
        // row of element e: (e + 0.5) / stride in float is exact here (e < 2^12,
        // the half offset keeps the quotient >= 0.5/stride away from integers)
        const int e = 4 * i, r = (int)(((float)e + 0.5f) * inv_stride), c = e - r * stride;
        float* d = buf + r * pitch + c;
        d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
      }
    }
    __syncwarp();
    const int64_t k = base + lane;
    float* row = buf + lane * pitch;
    if (lane < n_rows) {
      if (depth_keys[k] == ~0ull) {
        for (int i = 0; i < C3; ++i) row[i] = 0.f;
      } else {
        const Geom gm = load_geom(cl, k);
        double gin[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) gin[ch] = (double)grads[(int64_t)(6 + ch) * cap + k];
        const double v[3] = {gm.px - cam.center[0], gm.py - cam.center[1], gm.pz - cam.center[2]};
        const double nv = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        const double d[3] = {v[0] / nv, v[1] / nv, v[2] / nv};
        // pass 1: colour before the clip (core.py:169-172) -> which channels pass gradient
        double val[3] = {0.5, 0.5, 0.5};
        for_sh_basis(d[0], d[1], d[2], degree, [&](int n, double Yn, double, double, double) {
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) val[ch] += (double)row[ch * C + n] * Yn;
        });
        double gc[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) gc[ch] = (val[ch] >= 0.0 && val[ch] <= 1.0) ? gin[ch] : 0.0;
        // pass 2: dL/dsh = gc * Y_n (in place), dL/ddir = sum gc * sh * dY_n
        double dd[3] = {0.0, 0.0, 0.0};
        for_sh_basis(d[0], d[1], d[2], degree, [&](int n, double Yn, double gx, double gy, double gz) {
          double ws = 0.0;
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            ws += gc[ch] * (double)row[ch * C + n];
            row[ch * C + n] = (float)(gc[ch] * Yn);
          }
          dd[0] += ws * gx;
          dd[1] += ws * gy;
          dd[2] += ws * gz;
        });
        // stored bands above the evaluated degree get no gradient
        for (int n = nb; n < C; ++n)
          for (int ch = 0; ch < 3; ++ch) row[ch * C + n] = 0.f;
        const double ddot = dd[0] * d[0] + dd[1] * d[1] + dd[2] * d[2];
        for (int i = 0; i < 3; ++i) out.positions[3 * k + i] += (float)((dd[i] - d[i] * ddot) / nv);
      }
    }
    __syncwarp();
    // gradient rows are packed (3C floats per row): coalesced stores, 16-byte
    // when the packed block is 16-byte aligned (3C % 4 == 0 or an even base)
    float* dst = out.sh + base * C3;
    if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0 && (n_rows * C3) % 4 == 0) {
      float4* d4 = reinterpret_cast<float4*>(dst);
      for (int i = lane; i < n_rows * C3 / 4; i += 32) {
        float t[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int e = 4 * i + q, r = (int)(((float)e + 0.5f) * inv_c3), c = e - r * C3;
          t[q] = buf[r * pitch + c];
        }
        d4[i] = make_float4(t[0], t[1], t[2], t[3]);
      }
    } else {
      for (int e = lane; e < n_rows * C3; e += 32) {
        const int r = (int)(((float)e + 0.5f) * inv_c3), c = e - r * C3;
        dst[e] = buf[r * pitch + c];
      }
    }
    __syncwarp();
  }
}

void launch_blend_bwd(int n_tiles, const uint32_t* list, const uint32_t* bxs, const uint32_t* bys,
                      const uint2* ranges, const HotRec* hot, const FastRec* fast, const uint32_t* order,
                      const cs_settings& st, int width, int height, int ntx, const float* dl_dimg,
                      const BlendState& state, uint32_t* ticket, gacc_t* grads, int64_t cap,
                      cudaStream_t s) {
  BwdParams bp;
  for (int i = 0; i < 3; ++i) bp.bg[i] = st.background[i];
  bp.alpha_floor = st.alpha_floor;
  bp.tile_size = st.tile_size;
  bp.width = width;
  bp.height = height;
  bp.ntx = ntx;
  constexpr int PX = CS_BWD_PX;
  static int grid = 0;
  const int dyn = kBwdDynSmem;
  if (grid == 0) {
    if (dyn) cudaFuncSetAttribute(k_blend_bwd<PX>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    grid = persistent_grid(k_blend_bwd<PX>, kBwdThreads, dyn);
  }
  const int nboxes = PX == 1 ? boxes_per_tile(st.tile_size) : boxes_per_tile2(st.tile_size);
  cudaMemsetAsync(ticket, 0, sizeof(uint32_t), s);
  k_blend_bwd<PX><<<grid, kBwdThreads, dyn, s>>>(list, bxs, bys, ranges, hot, fast, order, n_tiles * nboxes,
                                               nboxes, bp, dl_dimg, state, ticket, grads, cap);
}

void launch_project_bwd(const cs_cloud& cl, const uint64_t* depth_keys, const cs_camera& cam,
                        const cs_settings& st, const gacc_t* grads, int64_t cap, const cs_grads& out,
                        cudaStream_t s) {
  const int64_t blocks = std::min<int64_t>((cl.count + 127) / 128, 148 * 16);
  if (blocks <= 0) return;
  k_project_bwd_geom<<<(unsigned)blocks, 128, 0, s>>>(cl, depth_keys, cam, st, grads, cap, out);
  const int pitch = cl.sh_stride | 1;  // odd word pitch: lane rows hit distinct banks
  const size_t smem = sizeof(float) * (kShBwdThreads / 32) * 32 * pitch;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_project_bwd_sh, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  const int64_t blocks_sh = std::min<int64_t>((cl.count + kShBwdThreads - 1) / kShBwdThreads, 148 * 4);
  k_project_bwd_sh<<<(unsigned)blocks_sh, kShBwdThreads, smem, s>>>(cl, depth_keys, cam, st, grads,
                                                                    cap, out, pitch);
}

}  // namespace cs

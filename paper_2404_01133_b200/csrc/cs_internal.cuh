// cs_internal.cuh -- shared device-side types and primitives for libcsgpu.
//
// Layouts in HBM; every per-splat array is
// indexed by assembled index (the splat id), written once by the projection:
//   HotRec    :  80 B -- staged in smem by the blend (quadratic form, opacity,
//                        colour, fast-reject threshold, cull box)
//   rect      :  16 B -- tile rectangle (render.py:226-231)
//   keys      :  8 B  -- float64 depth bits (~0 if culled), exact tie-break of K4b
//   keys32/vals: 4+4 B -- float32-rounded depth, splat id (radix-sorted, K4)
//   ProjRec   : 128 B -- full _Projected record, written only in debug/dump mode
//   pairs     :  u32 tile key + u32 splat id, sorted stably by tile
#pragma once
#include <cstddef>
#include <cuda_runtime.h>

#include <algorithm>
#include <stdint.h>

#include "../../include/cs_api.h"

namespace cs {

constexpr int kWarp = 32;

// Status word for decoupled look-back scans (single-pass chained scan).
// bits 63..62: 0 = not ready, 1 = aggregate only, 2 = inclusive prefix.
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPre = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

struct Seg {          // one assembled piece: levels[L][j] (or the single cloud)
  int64_t start;      // first assembled index of this piece
  int64_t count;
  int32_t cloud;      // index into the descriptor table
  int32_t pad;
};

struct __align__(16) ProjRec {
  double mx, my;        // mean2d  (render.py:128-129)
  double c0, c1, c2;    // conic   (render.py:172)
  double a, b, c;       // cov2d + low-pass (render.py:142-144)
  double rx, ry;        // marginal support radii (render.py:153-154)
  double opacity;
  double depth;         // camera z
  float r, g, bl;       // SH colour (fp32 of the float64 value)
  uint32_t pad;
  int64_t src;          // assembled index
  int64_t pad2;
};
static_assert(sizeof(ProjRec) == 128, "ProjRec layout");

struct __align__(16) HotRec {   // everything the blend reads per splat (64 B: 4 cp.async)
  double mx, my, c0, c1, c2;     // mean2d, conic (render.py:128-129, 172)
  double opacity;
  float lthr;                    // fast-reject threshold on power (<= log(alpha_floor/o) - margin,
                                 // rounded down to float: exact as a double)
  float r, g, b;                 // SH colour (fp32 of the float64 value)
};
static_assert(sizeof(HotRec) == 64, "HotRec layout");
// byte offsets k_blend_fast reads a staged HotRec at (ld.shared): mx 0, my 8,
// c0 16, c1 24, c2 32, opacity 40, lthr 48, r g b 52 56 60
static_assert(offsetof(HotRec, c0) == 16 && offsetof(HotRec, opacity) == 40 && offsetof(HotRec, lthr) == 48 &&
                  offsetof(HotRec, r) == 52 && offsetof(HotRec, b) == 60,
              "HotRec field offsets");
constexpr int kHotChunks = (int)(sizeof(HotRec) / 16);  // cp.async 16-byte copies per record

// ---------------------------------------------------------------------------
// FastRec: what the certified float32 blend (cs_blend.cu, k_blend_fast) stages
// per splat instead of the float64 HotRec.  The reference decides every
// fragment in float64 (_kernels.py:52-66); the fast blend evaluates the same
// quantities in float32 and carries, per splat, a PROVEN bound on how far its
// float32 results can be from the float64 ones, so that every decision whose
// float32 value is farther than the bound from its threshold is the
// reference's decision.  Decisions inside the bound are re-made in float64
// (cs_blend.cu).  Everything is in the log2 domain of alpha:
//   P = log2(o exp(power)) = log2(e) power + log2(o),  alpha = 2^P (before the
//   0.99 clamp), with dx = dxh - mxl, dxh = sx - mxh (mxh = float(mx), mxl the
//   exact double remainder mx - mxh) expanded in dxh:
//   P32 = (A dxh + (B dyh + D)) dxh + ((C dyh + E) dyh + F)   -- 2 FADD + 5 FFMA:
//   A, B, C: float(-log2(e) c0 / 2), float(-log2(e) c1), float(-log2(e) c2 / 2);
//   D, E   : the linear terms the low parts of the mean contribute,
//            -2 A mxl - B myl and -B mxl - 2 C myl (double, rounded);
//   F      : A mxl^2 + B mxl myl + C myl^2 + log2(o) -- log2(o) folded in, so
//            alpha32 = ex2(P32) costs no multiply and the floor test is one
//            compare;  L2o = float(log2(o)) is kept for the error bound;
//   (the expansion only moves the mean's low parts into coefficients: the
//   roundings are those of the hi/lo form -- dxh = sx - mxh rounds once, the
//   D/E/F roundings are below the |mxl| terms of the bound)
//   Flo/Fhi: log2(alpha_floor) -/+ dP, rounded outward, dP bounding
//            |P32 - P| on R = {power64 >= lthr - 1} (which holds the floor
//            contour): P32 < Flo is a certain skip, P32 >= Fhi a certain
//            accept (_kernels.py:61); outside R, P32 < Flo as well (the
//            error there is a tiny fraction of |P|, and P < log2(afl) - 1.44);
//   ek1/ek0: per-fragment bound on |alpha32 / alpha64 - 1|:
//            ek1 |P32 - L2o| + ek0 (the quadratic form's error is proportional
//            to |power| through S(d) <= ratio |power|, plus the L2o roundings,
//            MUFU.EX2 error) -- near the centre of an opaque splat (L2o ~ 0),
//            where 1/(1 - alpha) amplifies it, it is ~6e-7;
//   r, g, b: SH colour.
// Ill-conditioned splats (thin, edge-on: dp > kFastMaxDp, non-positive-definite
// or non-finite conic) are flagged in their cull box (kBoxExact): every lane
// takes the float64 path for them.
struct __align__(16) FastRec {
  float mxh, D, myh, E;
  float A, B, C, F;
  float flo, fhi, ek1, ek0;
  float r, g, b, L2o;
  // a staging slot holding a flagged splat's HotRec instead (k_blend_fast)
  __device__ const HotRec& as_hot() const { return *reinterpret_cast<const HotRec*>(this); }
};
static_assert(sizeof(FastRec) == 64, "FastRec layout");
static_assert(offsetof(FastRec, A) == 16 && offsetof(FastRec, flo) == 32 && offsetof(FastRec, r) == 48 &&
                  offsetof(FastRec, L2o) == 60,
              "FastRec field offsets (kFrMean / kFrQuad / kFrFloor / kFrColour)");
// byte offsets inside a staged FastRec (k_blend_fast reads them with ld.shared)
constexpr uint32_t kFrMean = 0, kFrQuad = 16, kFrFloor = 32, kFrColour = 48;
// A flagged splat's cull box carries x0 = kBoxExact (K3, fast-blend frames
// only): the blend then stages its float64 HotRec instead of the FastRec.  The
// box only widens to the left (x0 = -32768 never rejects), so the cull stays
// conservative; pixels outside the splat are rejected by its float64 power.
constexpr int kBoxExact = -32768;
constexpr float kFastMaxDp = 2e-5f;      // power-error bound above which a splat is decided in float64
// max relative error of ex2.approx.ftz.f32 over [-32, 1]: measured exhaustively
// on the B200 by tools/ex2_check.cu (profiles/r2_ex2_check.txt); the bound
// used here is twice that.
constexpr float kEx2RelErr = 4.0e-7f;

// Build the FastRec of a visible splat from the float64 values the exact path
// uses (mean, conic = inverse of (a, b, c), opacity, lthr) -- K3.  (ca, cc):
// diagonal of the conic's inverse (the 2D covariance incl. low pass), which
// bounds the pixel offsets of the region R = {power >= lthr - 1}:
// |dx| <= sqrt(2 (L + 1) ca), |dy| <= sqrt(2 (L + 1) cc).
__device__ __forceinline__ FastRec make_fast_rec(double mx, double my, double c0, double c1, double c2,
                                                 double opacity, float ln_o, float lthr, float r, float g, float b,
                                                 double ca, double cc, double log2_afl, bool& exact) {
  constexpr float u = 5.9604645e-8f;  // 2^-24
  constexpr double kLog2e = 1.4426950408889634;
  constexpr float kLn2 = 0.69314718f;
  FastRec f;
  f.mxh = (float)mx;
  f.myh = (float)my;
  const double ml = mx - (double)f.mxh, mly = my - (double)f.myh;  // exact
  const float mxl = (float)ml, myl = (float)mly;                     // (the bound's |mxl| terms)
  const double Ad = -0.5 * kLog2e * c0, Bd = -kLog2e * c1, Cd = -0.5 * kLog2e * c2;
  f.A = (float)Ad;
  f.B = (float)Bd;
  f.C = (float)Cd;
  // log2(o) from the float log of the float opacity K3 already has (ln_o =
  // logf(float(o))): |L2o - log2(o)| <= log2(e) u (opacity rounding)
  // + 3.5u |L2o| (logf <= 1 ulp, log2(e) as a float, the multiply), in l2o_err below
  f.L2o = opacity > 0.0 ? ln_o * 1.44269504f : 0.0f;
  f.D = (float)(-2.0 * Ad * ml - Bd * mly);
  f.E = (float)(-Bd * ml - 2.0 * Cd * mly);
  f.F = (float)((Ad * ml * ml + Bd * ml * mly + Cd * mly * mly) + (double)f.L2o);
  f.r = r; f.g = g; f.b = b;
  exact = false;
  const float L = -lthr;  // > 0 for any alpha_floor < opacity (else lthr >= 0: never passes)
  if (!(L > 0.0f) || !(opacity > 0.0)) {   // nothing can pass: keep the fast path, never passes
    f.flo = f.fhi = __int_as_float(0x7f800000);
    f.ek1 = f.ek0 = 0.f;
    return f;
  }
  const double det = c0 * c2 - c1 * c1;   // > 0 <=> |c1| < sqrt(c0 c2)
  const bool pd = c0 > 0.0 && c2 > 0.0 && det > 0.0 && ca > 0.0 && cc > 0.0 &&
                  isfinite(mx) && isfinite(my) && isfinite(c0) && isfinite(c1) && isfinite(c2) &&
                  isfinite(ca) && isfinite(cc);
  // Error of the float32 quadratic form on R = {power64 >= lthr - 1} = {d^T C d <= Q},
  // C = [[c0, c1], [c1, c2]], Q = 2 (L + 1), in natural-log units:
  //  * rounding (coefficients, two products, two fmas): <= 4u S(d),
  //    S(d) = 0.5 c0 dx^2 + |c1 dx dy| + 0.5 c2 dy^2 = 0.5 d^T |C| d (|C|: |c1|);
  //  * offsets: |dx32 - dx| <= 2u |dx| + u |mxl| (dx = (sx - mxh) - mxl), so
  //    |grad . e| <= 2u (|c0 dx + c1 dy| |dx| + |c1 dx + c2 dy| |dy|) <= 4u S(d)
  //    plus the |mxl| terms;
  //  * max of S on R: 0.5 Q lambda_max(|C|, C) = 0.5 Q (1 + rho) / (1 - rho),
  //    rho = |c1| / sqrt(c0 c2) (the generalized eigenvalue of the pair).
  // Thin, edge-on splats (rho -> 1) exceed kFastMaxDp and are flagged.
  // The log2(o) term adds its own error, the rounding of F and two roundings
  // of sums that contain it (l2o_err below, log2 units).
  const float Q = 2.0f * (L + 1.0f) * 1.0001f;
  // max of S(d) / |power(d)|: (1 + rho) / (1 - rho) = (s + |c1|)^2 / det, s = sqrt(c0 c2),
  // in float (relative error < 1e-6 while det / (c0 c2) > 1e-6; below that the
  // ratio exceeds 4e6 and dp flags the splat whatever the rounding)
  const float sq = sqrtf((float)(c0 * c2)) + fabsf((float)c1);
  const float ratio = __fdiv_ru(sq * sq, (float)det) * 1.0002f;
  const float Smax = 0.5f * Q * ratio;
  const float DX = sqrtf(Q * (float)ca) * 1.0001f + 1e-3f;   // |dx| on R
  const float DY = sqrtf(Q * (float)cc) * 1.0001f + 1e-3f;
  const float a0 = fabsf((float)c0) * 1.0001f, a1 = fabsf((float)c1) * 1.0001f,
              a2 = fabsf((float)c2) * 1.0001f;
  const float lo_terms = 2.0f * u * ((a0 * DX + a1 * DY) * (fabsf(mxl) + 1e-30f) + (a1 * DX + a2 * DY) * fabsf(myl));
  const float dp = 1.25f * (8.0f * u * Smax + lo_terms) + 1e-9f;
  if (!pd || !(dp <= kFastMaxDp)) {
    exact = true;
    f.flo = lthr;
    f.fhi = f.ek1 = f.ek0 = 0.f;
    return f;
  }
  // |P32 - P| on R, log2 units (the reference's own float64 rounding of
  // o * exp(power) is ~1e-16: inside the 1e-9 slack)
  // log2(o) error (log2e u + 3.5u |L2o|: logf, log2(e) as a float, the multiply),
  // the rounding of F and two FMA roundings
  // of sums holding it (3u |L2o|)
  const float l2o_err = 1.01f * (1.4426950f * u + 7.0f * u * fabsf(f.L2o));
  const float dP = 1.01f * ((float)kLog2e * dp + l2o_err) + 1e-9f;
  const double F = log2_afl;
  f.flo = __double2float_rd(F - (double)dP);
  f.fhi = __double2float_ru(F + (double)dP);
  // per fragment, |alpha32 / alpha - 1| <= ln2 dP(d) (1 + dP) + ex2 error, with
  // dP(d) <= log2e (10u S(d) + lo_terms) + l2o_err, S(d) <= ratio |power|,
  // |power| <= ln2 (|P32 - L2o| + dP): eps(d) <= ek1 |P32 - L2o| + ek0
  const float k10 = 1.01f * (1.0f + dP) * 10.0f * u * ratio * kLn2;
  f.ek1 = k10 + 2.02f * u;
  f.ek0 = k10 * dP + 1.01f * (1.0f + dP) * (lo_terms + kLn2 * l2o_err + 1e-9f) + 1.01f * (kEx2RelErr + 3.0f * u);
  return f;
}

// pair-major cull boxes for the blend: (lo | hi << 16) as two int16, one word
// per axis; kEmptyBox = (32767, -32768) never intersects
__host__ __device__ __forceinline__ uint32_t pack_box(int lo, int hi) {
  return (uint32_t)(uint16_t)(int16_t)lo | ((uint32_t)(uint16_t)(int16_t)hi << 16);
}
constexpr uint32_t kEmptyBox = 0x7fffu | (0x8000u << 16);

// Backward precision (tests/test_gpu_backward_scale.py, 1080p, N(0,1) dL/dimage,
// bar max(1e-4, 1e-3 |g|) per element).  A splat near the camera collects
// 10^4-10^5 per-pixel terms whose sum is a random walk; a per-pixel term can be
// ~100x its neighbours' (dL/dalpha carries S/(1 - alpha), alpha up to 0.99),
// so small final gradients of large splats need every accumulation stage in
// float64: the per-splat partials (CS_BWD_ACC_F64: the K10 -> K11 buffer and
// its atomics), the warp reduction of the lanes' partials (CS_BWD_RED_F64,
// cs_backward.cu) and the transmittance / colour sums / light from behind
// (CS_BWD_SP_F64).  Measured with any of the three in float32: 12-14 of 60k
// position gradients outside the bar; with all three in float64: none
// (profiles/r2_backward_precision.txt).
#ifndef CS_BWD_ACC_F64
#define CS_BWD_ACC_F64 1
#endif
#if CS_BWD_ACC_F64
typedef double gacc_t;
#else
typedef float gacc_t;
#endif
// The backward's transmittance / accumulated colour / light-from-behind
// S_k = (C - P_k) + T_end bg (divided by 1 - alpha >= 0.01): float64 when
// CS_BWD_SP_F64 (then the training forward keeps float64 colour sums, the
// same arithmetic the backward repeats), float32 otherwise.
#ifndef CS_BWD_SP_F64
#define CS_BWD_SP_F64 1
#endif
#if CS_BWD_SP_F64
typedef double bsp_t;
#else
typedef float bsp_t;
#endif

struct DevStats {     // device mirror of cs_frame_stats + scratch counters
  int64_t assembled;
  int64_t visible;
  int64_t skipped;
  int64_t pairs;
  int64_t fragments;
  int32_t n_segs;
  int32_t status;
  int64_t evals;         // blend (pixel, splat) evaluations executed (E)
  int64_t warp_hits;     // blend (box, splat) warp evaluations
  int64_t warp_hits_empty;  // ... where no live pixel passed the fast reject
  int64_t blend_max_item_cycles;  // longest blend work item (DIAG)
  int64_t blend_item_cycles;      // sum over blend work items (DIAG)
  int64_t blend_exact_hits;       // certified float32 blend (DIAG): hits decided in float64
  int64_t blend_floor_resolved;   // ... alpha-floor tests re-decided in float64
  int64_t blend_replays;          // ... transmittance replays
  int64_t pairs_eff;     // pairs actually processed (0 when the pair buffer overflowed)
  uint32_t tickets[16];  // chunk tickets for single-pass kernels, zeroed per frame
};


// Outputs of the projection kernel, indexed by assembled index (splat id);
// hot/rects/boxes/recs are written for visible splats only.
// 8-byte tile rectangle (tile coordinates < 2^16): K5/K6 gather it in depth
// order, so half the bytes of an int4 means half the gathered sectors' footprint.
__device__ __forceinline__ uint2 pack_rect(int x0, int x1, int y0, int y1) {
  return make_uint2((uint32_t)x0 | ((uint32_t)x1 << 16), (uint32_t)y0 | ((uint32_t)y1 << 16));
}
__device__ __forceinline__ int4 unpack_rect(uint2 r) {
  return make_int4((int)(r.x & 0xffffu), (int)(r.x >> 16), (int)(r.y & 0xffffu), (int)(r.y >> 16));
}

struct ProjOutputs {
  uint64_t* keys;    // float64 depth bits (~0 for culled Gaussians), for the exact run fix-up
  uint32_t* keys32;  // float32-rounded depth bits (~0 for culled): the radix-sorted key
  uint32_t* vals;    // splat id
  HotRec* hot;
  FastRec* fast;     // optional: the certified float32 blend's records (non-kept-state frames)
  uint2* rects;      // tile rectangle, 16-bit packed: (x0 | x1 << 16, y0 | y1 << 16)
  short4* boxes;     // copy of HotRec's cull box, dense (8 B)
  ProjRec* recs;     // optional (debug / dumps)
  const uint8_t* exclude;  // input, optional: rows culled as if absent (assignment renders)
  double log2_afl;         // log2(alpha_floor) (the FastRec floor thresholds), set by the host
  float ln_afl;            // logf(float(alpha_floor)) (the fast-reject threshold lthr), set by the host
  int mark_exact = 1;      // flagged splats' cull boxes carry kBoxExact (fast-blend frames only)
};

// K10 certified pre-reject (CS_BWD_FAST=1, off): a kept-state (training)
// forward also writes the FastRecs (without marking flagged boxes), and the
// blend backward skips a pixel's float64 re-evaluation of a hit whenever the
// FastRec's float32 power is below its certified floor threshold (P32 < Flo =>
// the float64 alpha is below alpha_floor, so the exact forward did not accept
// that fragment).  Parity-green (81/81 GPU tests) but measured slower: K10
// 1.886 -> 2.04 ms per iteration, 324 -> 308 it/s (profiles/r5e_bwd_fast_ab.txt;
// the extra 48-byte staging per hit and register pressure outweigh the
// float64 forms it skips -- the backward walks only up to each pixel's last
// accepted fragment, where few hits are sure rejects).
#ifndef CS_BWD_FAST
#define CS_BWD_FAST 0
#endif

// LoD scene tables on device (cs_lod.cu)
struct LodTables {
  const cs_cloud* clouds;      // [L*J] level-major
  const double* bmin;          // [J*3]
  const double* bmax;
  const double* intervals;     // [L*2] (lo, hi), nearest-first
  const uint8_t* occupied;     // [J]
  const Seg* all_segs;         // [L*J] level-major virtual concatenation (pointwise mode)
  int n_levels, n_blocks;
  int64_t total_all;
};

// blend kernel parameters (cs_blend.cu)
struct BlendParams {
  double bg[3];
  double alpha_floor, t_floor;
  int tile_size, width, height, ntx;
  uint32_t flags;
  // certified float32 blend: t_floor as float, the termination band
  // t_floor (1.01 en + 4u) = en * tfl_b + tfl_c, and 1.5 t_floor
  float tfl, tfl_b, tfl_c, tfl_far;
};

struct BlendState {  // per-pixel state kept for the backward pass
  double* final_t;      // (H*W) final transmittance
  int32_t* last;        // (H*W) list position one past the last accepted fragment
  double* color_acc;    // (H*W*3) sum of w*c (before the background term)
};

// ---------------------------------------------------------------------------
// blend helpers shared by the forward (cs_blend.cu) and backward (cs_backward.cu)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Bulk-copy staging (the blend's HotRec records): one cp.async.bulk per hit
// record completing on a per-warp mbarrier, instead of four 16-byte cp.async
// copies per record.  The barrier of a stage is armed by one arrive with the
// stage's expected byte count; the records' copies complete its transaction
// count; the warp waits on the stage's phase parity before reading.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n CS_MBAR_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra CS_MBAR_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// the warp's generic-proxy reads of a stage buffer are ordered before the
// async-proxy (bulk copy) writes that refill it
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// local pixel index (0..ts*ts-1) of thread `tid` of a 256-thread CTA, pixel slot q.  When the
// tile side is a multiple of 8, warps own 8x4 pixel boxes (box index
// warp + 8q, row-major over the tile's (ts/8) x (ts/4) boxes).
__device__ __forceinline__ int local_pixel(int tid, int q, int ts) {
  if ((ts & 7) == 0) {
    const int b = (tid >> 5) + 8 * q, l = tid & 31, nbx = ts >> 3;
    const int bx = b % nbx, by = b / nbx;
    return (by * 4 + (l >> 3)) * ts + bx * 8 + (l & 7);
  }
  return tid + q * 256;
}

// Blend work items are (tile, box) pairs: a box is 32 pixels of a tile --
// a kBoxW x kBoxH block when the tile side allows, else 32 consecutive
// row-major pixels.  box_pixel -> local pixel index (>= ts*ts: no pixel).
// The forward blends' warp box: CS_BOX_W x (32 / CS_BOX_W) pixels: 4 x 8 (tall) measured
// faster than 8 x 4 on the C3 flythrough (blend 0.749 -> 0.727 ms), 2 x 16 and
// 16 x 2 slower (0.850 / 0.936 ms; profiles/r4_build_flag_sweeps.txt)
#ifndef CS_BOX_W
#define CS_BOX_W 4
#endif
constexpr int kBoxW = CS_BOX_W, kBoxH = 32 / CS_BOX_W;
__host__ __device__ __forceinline__ int boxes_per_tile(int ts) {
  return (ts % kBoxW == 0 && ts % kBoxH == 0) ? (ts / kBoxW) * (ts / kBoxH) : (ts * ts + 31) / 32;
}
__device__ __forceinline__ int box_pixel(int b, int lane, int ts) {
  if (ts % kBoxW == 0 && ts % kBoxH == 0) {
    const int nbx = ts / kBoxW, bx = b % nbx, by = b / nbx;
    return (by * kBoxH + lane / kBoxW) * ts + bx * kBoxW + lane % kBoxW;
  }
  return b * 32 + lane;
}
// Two pixels per lane: 8x8 boxes, lane (x, y) of the upper 8x4 half and
// (x, y + 4) of the lower; tile sizes that are not multiples of 8 use
// row-major 64-pixel chunks (pixel j of the lane at 32 j + lane).
// two pixels per lane (the backward): a kBox2W x (64 / kBox2W) block, the
// lane's pixels 32 / kBox2W rows apart
#ifndef CS_BOX2_W
#define CS_BOX2_W 8
#endif
constexpr int kBox2W = CS_BOX2_W, kBox2H = 64 / CS_BOX2_W;
__host__ __device__ __forceinline__ int boxes_per_tile2(int ts) {
  return (ts % kBox2W == 0 && ts % kBox2H == 0) ? (ts / kBox2W) * (ts / kBox2H) : (ts * ts + 63) / 64;
}
__device__ __forceinline__ int box_pixel2(int b, int lane, int ts, int j) {
  if (ts % kBox2W == 0 && ts % kBox2H == 0) {
    const int nbx = ts / kBox2W, bx = b % nbx, by = b / nbx;
    return (by * kBox2H + lane / kBox2W + (32 / kBox2W) * j) * ts + bx * kBox2W + lane % kBox2W;
  }
  return b * 64 + 32 * j + lane;
}

// ---------------------------------------------------------------------------
// exp(x) for the blend's x = power in [lthr, 0] (lthr >= log(alpha_floor) - 1e-6
// > -745): x = (256 m + j) ln2/256 + r, |r| <= ln2/512,
// exp(x) = 2^m 2^(j/256) (1 + q(r)), q the degree-5 Taylor polynomial of
// exp(r) - 1 (truncation < 1e-19), 2^(j/256) = hi + lo from a 256-entry table
// in shared memory, result hi + (hi q + lo): ~0.5 ulp like a libm exp
// (tools/exp_check.cu).  Neither this, CUDA's exp() nor the reference's libm
// exp are bit-identical to each other; they differ only at exact alpha-floor
// / transmittance knife-edges.  The three non-trivial Taylor
// coefficients sit in the table block too, so kernels load them into
// registers once instead of re-materialising 64-bit immediates per call.
__constant__ double2 c_exp2_256[256] = {
    {1.0, 0.0}, {1.0027112750502025, -3.636615928692264e-17},
    {1.0054299011128027, 9.499186535455032e-17}, {1.0081558981184175, -3.252058756084308e-17},
    {1.0108892860517005, -1.5234778603368577e-17}, {1.0136300849514894, 9.283599768183568e-18},
    {1.016378314910953, -5.77217007319966e-17}, {1.019133996077738, 3.601904982259662e-17},
    {1.0218971486541166, 5.109225028973444e-17}, {1.0246677928971357, -7.56160786848778e-17},
    {1.0274459491187637, -4.9560741746453704e-17}, {1.030231637686041, 3.319830041080813e-17},
    {1.0330248790212284, 7.600838874027088e-18}, {1.0358256936019572, -7.806782391337636e-17},
    {1.0386341019613787, 5.996273788852511e-17}, {1.041450124688316, 3.784830480287576e-17},
    {1.0442737824274138, 8.551889705537965e-17}, {1.0471050958792898, 7.277077243104315e-17},
    {1.0499440858006872, 5.592937848127003e-17}, {1.0527907730046264, -9.629482899026936e-17},
    {1.0556451783605572, 1.759325738772092e-18}, {1.0585073227945128, -7.152651856637781e-17},
    {1.061377227289262, -1.1973537085365658e-17}, {1.0642549128844645, 5.0787541986112304e-17},
    {1.0671404006768237, -7.899853966841582e-17}, {1.0700337118202419, -9.937162711288919e-17},
    {1.0729348675259756, -3.839668843358824e-18}, {1.075843889062791, -1.0002716151144136e-17},
    {1.0787607977571199, -6.656660436056593e-17}, {1.0816856149932152, -4.782623902997086e-17},
    {1.0846183622133092, 3.166152845816346e-17}, {1.0875590609177697, 5.409349307820291e-18},
    {1.0905077326652577, -3.046782079812471e-17}, {1.0934643990728858, 1.441395814726921e-17},
    {1.0964290818163769, -5.919933484449316e-17}, {1.099401802630222, 7.170459599701923e-17},
    {1.102382583307841, 5.2660368715706944e-17}, {1.1053714457017412, 8.239288760500214e-17},
    {1.1083684117236787, -8.786813845180527e-17}, {1.1113735033448175, 5.563945026669698e-17},
    {1.1143867425958924, 1.0410278456845571e-16}, {1.1174081515673693, -7.97680590262822e-17},
    {1.1204377524096067, -6.201085906554179e-17}, {1.12347556733302, -9.699737588987043e-17},
    {1.1265216186082418, 5.165856758795457e-17}, {1.129575928566288, 6.712805858726257e-17},
    {1.1326385195987192, 3.237356166738e-17}, {1.1357094141578055, 5.066599926126156e-17},
    {1.1387886347566916, 8.912812676025408e-17}, {1.1418762039695616, 4.6510911775314124e-17},
    {1.1449721444318042, 4.6412898921700107e-17}, {1.148076478840179, 6.897740236627192e-17},
    {1.1511892299529827, 3.250710218863827e-17}, {1.154310420590216, 1.0417128946273266e-16},
    {1.1574400736337511, -9.1238712311344e-17}, {1.1605782120274988, -3.261040205417394e-17},
    {1.1637248587775775, 3.8292048369240935e-17}, {1.1668800369524817, -8.79187957999917e-17},
    {1.1700437696832502, -1.8477442017900047e-18}, {1.1732160801636373, -7.287562586584994e-17},
    {1.1763969916502812, 5.554203254218079e-17}, {1.1795865274628758, 1.009231277510039e-16},
    {1.182784710984341, 1.542975430079076e-17}, {1.1859915656609938, -9.209506835293106e-18},
    {1.189207115002721, 3.982015231465646e-17}, {1.1924313825831512, 4.3975514156097214e-17},
    {1.1956643920398273, 4.6166036704814814e-17}, {1.1989061670743806, -9.809193356008423e-17},
    {1.202156731452703, 6.644981499252301e-17}, {1.2054161090051239, -3.3572721932675296e-17},
    {1.2086843236265816, -4.746725945228984e-17}, {1.2119613992768012, -4.8906110775211184e-17},
    {1.215247359980469, -7.712630692681488e-17}, {1.2185422298274085, -9.006726958363838e-17},
    {1.2218460329727576, -1.0611021211402691e-16}, {1.2251587936371455, -8.903533814269983e-17},
    {1.22848053610687, -1.89878163130253e-17}, {1.2318112847340759, 7.38938247161005e-17},
    {1.2351510639369334, -1.0755244344307841e-16}, {1.2384998981998165, 2.7677020555739674e-17},
    {1.241857812073484, 4.658027591836937e-17}, {1.245224830175258, -4.6772404498467275e-17},
    {1.2486009771892048, -8.261810999021964e-17}, {1.2519862778663162, 4.8341671524698976e-17},
    {1.255380757024691, -6.7113898212968784e-18}, {1.2587844395497165, -8.421782587730599e-17},
    {1.2621973503942507, -3.0844648874738465e-17}, {1.2656195145788063, 4.2505770034508686e-17},
    {1.2690509571917332, 2.667932131342186e-18}, {1.2724917033894028, -1.0577916267212421e-17},
    {1.275941778396392, 9.91543024421429e-17}, {1.2794012075056693, -9.759095008356062e-17},
    {1.2828700160787783, 1.713594918243561e-17}, {1.2863482295460256, -3.416955706936182e-17},
    {1.2898358734066657, 8.949257530897592e-17}, {1.2933329732290895, -2.9745904431327516e-17},
    {1.2968395546510096, 2.5382502794888315e-17}, {1.3003556433796506, 5.678728102802217e-17},
    {1.3038812651919358, 8.647675598267871e-17}, {1.3074164459346773, -7.336645652878869e-17},
    {1.3109612115247644, -7.181536135519454e-17}, {1.3145155879493546, 2.2675433151045856e-17},
    {1.318079601266064, -5.4579558271491535e-17}, {1.3216532776031575, -2.4806382459130217e-17},
    {1.3252366431597413, -2.8587312100388614e-17}, {1.3288297242059544, 4.08908622391016e-17},
    {1.3324325470831615, -5.101586630916744e-17}, {1.3360451382041458, -5.891866356388801e-17},
    {1.339667524053303, 8.927282594831732e-17}, {1.3432997311868353, -5.802580890201438e-17},
    {1.3469417862329458, 3.224065101254679e-17}, {1.3505937158920345, -8.287110381462417e-17},
    {1.3542555469368927, 7.70094837980299e-17}, {1.3579273062129011, -9.529635744825189e-17},
    {1.3616090206382248, 1.533787661270668e-18}, {1.365300717204012, -1.0005363125974765e-16},
    {1.3690024229745905, 9.593797919118849e-17}, {1.3727141650876684, -4.495960595234841e-17},
    {1.3764359707545302, -6.898588935871801e-17}, {1.380167867260238, 1.0510314579969984e-16},
    {1.383909881963832, -6.770511658794786e-17}, {1.387662042298529, 8.422984274875415e-17},
    {1.3914243757719262, -4.9061748652889893e-17}, {1.3951969099662003, -9.329336224225497e-17},
    {1.3989796725383112, -9.614213209051323e-17}, {1.4027726912202048, -5.295783249407989e-17},
    {1.4065759938190154, 7.034914812136422e-18}, {1.4103896082172707, 4.166548728435062e-17},
    {1.4142135623730951, -9.667293313452913e-17}, {1.4180478843204152, 2.2744385421855295e-17},
    {1.4218926021691656, -1.6077828915890244e-17}, {1.4257477441054942, 9.880690758500607e-17},
    {1.42961333839197, -1.2031642489053655e-17}, {1.433489413367789, -5.802454243926826e-17},
    {1.4373759974489824, -4.2040340164675566e-17}, {1.4412731191286257, 5.602503650878986e-18},
    {1.4451808069770467, -3.0237581349939873e-17}, {1.449099089642035, -6.259405000819309e-17},
    {1.4530279958490526, -5.779948609396106e-17}, {1.4569675544014438, 5.648679453876998e-17},
    {1.460917794180647, -5.600377186075216e-17}, {1.4648787441464057, 9.530767543587157e-17},
    {1.4688504333369818, 8.465882756533628e-17}, {1.4728328908693675, 6.691774081940589e-17},
    {1.4768261459394993, -3.483994556892796e-17}, {1.4808302278224719, -9.686952102630619e-17},
    {1.4848451658727524, 1.0780086764407481e-16}, {1.488870989524397, 6.155367157742871e-17},
    {1.4929077282912648, 1.4192920154284036e-17}, {1.4969554117672355, -2.861663253899158e-17},
    {1.5010140696264256, -6.413767275790235e-17}, {1.5050837316234065, 7.074710613582846e-17},
    {1.5091644275934228, -1.016455327754295e-16}, {1.5132561874526098, 8.884497851338712e-17},
    {1.5173590411982147, -4.308699472043341e-17}, {1.5214730189088146, -5.9963876759456834e-18},
    {1.5255981507445384, -1.1024941712342561e-16}, {1.529734466947287, 3.7857921151572197e-17},
    {1.533881997840956, 8.875226844438446e-17}, {1.5380407738316568, 1.0174672351161359e-16},
    {1.5422108254079407, 7.949834809697621e-17}, {1.5463921831410214, 1.068396000565722e-16},
    {1.550584877685, -1.4600706590689385e-17}, {1.5547889397770887, -8.003161350116036e-17},
    {1.559004400237837, 3.7812070533575275e-17}, {1.5632312899713576, 7.484777645590734e-17},
    {1.567469639965553, -1.0352061768849722e-16}, {1.5717194812923414, -3.3429840046872e-17},
    {1.5759808451078865, -1.0136916471278304e-17}, {1.5802537626528246, -5.163402929554468e-17},
    {1.5845382652524937, -1.9337717034585703e-17}, {1.588834384317164, -5.9949501188244794e-18},
    {1.593142151342267, -1.0094406542311964e-16}, {1.597461597908627, 2.4868392796221e-17},
    {1.6017927556826934, -6.054917453527784e-17}, {1.606135656416771, -1.0354545288059995e-16},
    {1.6104903319492543, 2.4707192569797888e-17}, {1.6148568142048607, -7.316663399125123e-17},
    {1.6192351351948637, 2.0941334154229092e-17}, {1.6236253270173289, -3.584512851414475e-17},
    {1.6280274218573478, -6.712955084707084e-17}, {1.632441451987275, 9.852819230429993e-17},
    {1.6368674497669644, 7.698325071319876e-17}, {1.6413054476440063, -9.247568737640706e-17},
    {1.645755478153965, -1.0125679913674773e-16}, {1.6502175739206177, 9.133279588729904e-18},
    {1.6546917676561943, 9.643294303196029e-17}, {1.6591780921616162, -7.275545550823051e-17},
    {1.6636765803267364, 5.8909926967131e-17}, {1.6681872651305825, 4.269178019570615e-17},
    {1.6727101796415966, -5.476715964599563e-17}, {1.6772453570178785, 8.303949509950733e-17},
    {1.681792830507429, 8.199010020581497e-17}, {1.6863526334483934, -7.181463278358011e-17},
    {1.6909247992693053, -9.66967147439488e-17}, {1.6955093614893326, 7.238416872845167e-17},
    {1.7001063537185235, -8.0237193703977e-18}, {1.7047158096580513, -2.7288832847972816e-17},
    {1.709337763100463, -9.868779456632931e-17}, {1.713972247929926, 6.473975107753367e-17},
    {1.718619298122478, -1.851380418263111e-17}, {1.723278947746274, -9.5221238003938e-17},
    {1.7279512309618377, -1.0750981861204642e-16}, {1.732636182022311, -1.6980510743154155e-18},
    {1.7373338352737062, 3.164389299292957e-17}, {1.7420442251551564, -1.5259591189507888e-18},
    {1.746767386199169, -1.0752290483507515e-16}, {1.7515033530318782, -5.1244504205967247e-17},
    {1.7562521603732995, 2.960140695448873e-17}, {1.761013843037584, -7.943253125039228e-17},
    {1.7657884359332727, 9.461315018083268e-17}, {1.7705759740635547, 5.961794510040556e-17},
    {1.7753764925265212, 6.429731796556572e-17}, {1.7801900265154245, -5.2846272890916174e-17},
    {1.785016611318935, 1.5330400121031314e-17}, {1.789856282321401, -4.1543546606833504e-17},
    {1.7947090750031072, 1.8227458427912087e-17}, {1.7995750249405351, -2.526889233358898e-17},
    {1.804454167806624, -5.177222408793318e-17}, {1.809346539371032, -9.03264140245003e-17},
    {1.8142521755003989, -9.969531538920349e-17}, {1.8191711121586085, 7.402676901145839e-17},
    {1.8241033854070534, -1.0159627862277083e-16}, {1.8290490314048973, 6.889192908835696e-17},
    {1.8340080864093424, 3.283107224245627e-17}, {1.8389805867758937, 6.918969740272512e-18},
    {1.843966568958626, -5.939742026949965e-17}, {1.8489660695104508, 9.027580446261089e-17},
    {1.8539791250833855, 9.761887490727594e-17}, {1.8590057724288205, -9.528705461989941e-17},
    {1.864046048397789, 6.540912680620572e-17}, {1.8690999899412386, -9.938505214255067e-17},
    {1.8741676341103, -6.122763413004143e-17}, {1.8792490180565602, -1.6226315557835845e-17},
    {1.8843441790323345, -8.226593125533711e-17}, {1.8894531543909392, -9.005168285059127e-17},
    {1.8945759815869656, 3.4034035352165297e-17}, {1.8997126981765553, -3.8597397693785143e-17},
    {1.9048633418176741, 6.533857514718279e-17}, {1.9100279502703899, -5.90968800674406e-17},
    {1.9152065613971474, -1.0619946056195963e-16}, {1.9203992131630474, 7.116681540630314e-17},
    {1.925605943636125, -9.914963769693741e-17}, {1.930826790987627, 6.16714970616911e-17},
    {1.9360617934922943, 1.0332385960676326e-16}, {1.9413109895286405, -6.638029891621488e-17},
    {1.9465744175792332, 6.811022349533877e-17}, {1.9518521162309783, -2.199016969979351e-17},
    {1.9571441241754002, 8.960767791036668e-17}, {1.9624504802089273, 1.0976844000913547e-16},
    {1.9677712232331759, -1.0314928011531132e-16}, {1.9731063922552343, -7.451617863956037e-18},
    {1.978456026387951, 4.0388753109278167e-17}, {1.9838201648502194, -2.2034544123910627e-17},
    {1.9891988469672663, 8.2051326383692e-18}, {1.9945921121709402, 1.7909710352002645e-17}
};

struct ExpTable {
  double2 t[256];
};
#ifndef CS_EXP_REGCONST
#define CS_EXP_REGCONST 1
#endif
// The range-reduction constants and the 0.99 clamp, kept in registers (loaded
// through a volatile pointer) instead of being re-materialised as 64-bit
// immediates (two uniform moves each) at every use.
__constant__ double c_exp_consts[4] = {369.3299304675746,        // 256 / ln2
                                       -0.0027076061742263846,   // -(ln2/256), high 33 bits
                                       1.6409824502660487e-13,   // ln2/256, low part
                                       0.99};                    // alpha clamp (_kernels.py:59)
struct ExpCoef {
  double c3, c4, c5;  // 1/6, 1/24, 1/120
  double inv, hi, lo, clamp;
};

__device__ __forceinline__ ExpCoef load_exp_table(ExpTable* s_tab) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_tab->t[i] = c_exp2_256[i];
  ExpCoef c;
  // read through a volatile pointer so the values live in registers for the
  // whole kernel (the compiler cannot fold them back into immediates)
  volatile const double* vc = reinterpret_cast<volatile const double*>(&c_exp2_256[0]);
  const double one = vc[0];  // 2^0 = 1.0 exactly
  c.c3 = one / 6.0;
  c.c4 = one / 24.0;
  c.c5 = one / 120.0;
  if (CS_EXP_REGCONST) {
    volatile const double* vk = c_exp_consts;
    c.inv = vk[0]; c.hi = vk[1]; c.lo = vk[2]; c.clamp = vk[3];
  } else {
    c.inv = 369.3299304675746; c.hi = -0.0027076061742263846; c.lo = 1.6409824502660487e-13; c.clamp = 0.99;
  }
  return c;
}

__device__ __forceinline__ double exp_le0(double x, const ExpTable& T, const ExpCoef& c) {
  const double kd = rint(x * c.inv);                        // 256 / ln2
  double r = fma(kd, c.hi, x);                              // ln2/256, high 33 bits
  r = fma(kd, c.lo, r);                                     // ln2/256, low part
  double q = fma(r, c.c5, c.c4);
  q = fma(q, r, c.c3);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = q * r;                                               // exp(r) - 1
  const int k = (int)kd;
  const double2 t = T.t[k & 255];
  const double scale = __longlong_as_double((long long)((k >> 8) + 1023) << 52);  // 2^m, m = floor(k/256)
  return (t.x + fma(t.x, q, t.y)) * scale;
}

// grid of a persistent kernel: as many CTAs as are co-resident on all SMs
template <typename K>
static int persistent_grid(K kernel, int threads, size_t dyn_smem = 0) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, dyn_smem);
  return std::max(1, sms * std::max(1, per_sm));
}

// ---------------------------------------------------------------------------
// no-FMA float64 arithmetic in numpy order
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// numpy float64 -> int64 cast (x86 cvttsd2si: out of range / NaN -> INT64_MIN)
__device__ __forceinline__ int64_t np_to_i64(double x) {
  if (!(x >= -9223372036854775808.0 && x < 9223372036854775808.0)) return INT64_MIN;
  return (int64_t)x;
}
__device__ __forceinline__ int64_t clip_i64(int64_t v, int64_t lo, int64_t hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

// ---------------------------------------------------------------------------
// warp / block primitives

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if ((int)lane_id() >= o) v += n;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive scan of one value per thread; returns exclusive prefix,
// writes the block total.  `scratch` needs (blockDim/32 + 1) entries.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* scratch, T& total) {
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  T incl = warp_incl_scan(v);
  if (lane_id() == 31) scratch[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    T w = (int)lane_id() < nwarps ? scratch[lane_id()] : T(0);
    T wi = warp_incl_scan(w);
    if ((int)lane_id() < nwarps) scratch[lane_id()] = wi - w;
    if (lane_id() == 31) scratch[nwarps] = wi;
  }
  __syncthreads();
  T res = incl - v + scratch[warp];
  total = scratch[nwarps];
  __syncthreads();
  return res;
}

__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Decoupled look-back (single-pass chained scan).  Called by ALL lanes of
// warp 0 of the block owning `chunk` (chunks handed out in launch order by a
// ticket counter, so every predecessor is resident or finished).  Publishes
// the aggregate, walks back over predecessors 32 at a time and returns the
// exclusive prefix of this chunk; publishes the inclusive prefix.
__device__ __forceinline__ uint64_t lookback_exclusive(uint64_t* status, int64_t chunk,
                                                       uint64_t aggregate) {
  const uint32_t lane = lane_id();
  if (chunk == 0) {
    if (lane == 0) st_release_u64(&status[0], kFlagPre | aggregate);
    return 0;
  }
  if (lane == 0) st_release_u64(&status[chunk], kFlagAgg | aggregate);
  uint64_t exclusive = 0;
  int64_t pred = chunk - 1;
  while (true) {
    int64_t idx = pred - (int64_t)lane;
    uint64_t s = idx >= 0 ? ld_volatile_u64(&status[idx]) : (kFlagPre | 0ull);
    while (__any_sync(0xffffffffu, (s >> 62) == 0)) {
      if ((s >> 62) == 0) s = ld_volatile_u64(&status[idx]);
    }
    uint32_t pre_mask = __ballot_sync(0xffffffffu, (s >> 62) == 2);
    uint64_t v = s & kValMask;
    if (pre_mask) {
      int first = __ffs(pre_mask) - 1;
      uint64_t contrib = (int)lane <= first ? v : 0ull;
      exclusive += warp_sum(contrib);
      break;
    }
    exclusive += warp_sum(v);
    pred -= 32;
  }
  if (lane == 0) st_release_u64(&status[chunk], kFlagPre | (exclusive + aggregate));
  return exclusive;
}

// ---------------------------------------------------------------------------
// geometry loads (fp32 or fp64 quads)
struct Geom {
  double px, py, pz, op;
  double sx, sy, sz;
  double qw, qx, qy, qz;
};

__device__ __forceinline__ Geom load_geom(const cs_cloud& c, int64_t k) {
  Geom g;
  if (c.fp64) {
    const double2* p = reinterpret_cast<const double2*>(c.pos_op) + 2 * k;
    const double2* s = reinterpret_cast<const double2*>(c.scale) + 2 * k;
    const double2* q = reinterpret_cast<const double2*>(c.quat) + 2 * k;
    double2 p0 = __ldg(p), p1 = __ldg(p + 1), s0 = __ldg(s), s1 = __ldg(s + 1), q0 = __ldg(q),
            q1 = __ldg(q + 1);
    g.px = p0.x; g.py = p0.y; g.pz = p1.x; g.op = p1.y;
    g.sx = s0.x; g.sy = s0.y; g.sz = s1.x;
    g.qw = q0.x; g.qx = q0.y; g.qy = q1.x; g.qz = q1.y;
  } else {
    float4 p = __ldg(reinterpret_cast<const float4*>(c.pos_op) + k);
    float4 s = __ldg(reinterpret_cast<const float4*>(c.scale) + k);
    float4 q = __ldg(reinterpret_cast<const float4*>(c.quat) + k);
    g.px = p.x; g.py = p.y; g.pz = p.z; g.op = p.w;
    g.sx = s.x; g.sy = s.y; g.sz = s.z;
    g.qw = q.x; g.qx = q.y; g.qy = q.z; g.qz = q.w;
  }
  return g;
}

__device__ __forceinline__ void load_pos(const cs_cloud& c, int64_t k, double& x, double& y,
                                         double& z) {
  if (c.fp64) {
    const double2* p = reinterpret_cast<const double2*>(c.pos_op) + 2 * k;
    double2 p0 = __ldg(p), p1 = __ldg(p + 1);
    x = p0.x; y = p0.y; z = p1.x;
  } else {
    float4 p = __ldg(reinterpret_cast<const float4*>(c.pos_op) + k);
    x = p.x; y = p.y; z = p.z;
  }
}

// Upper-bound binary search over segment starts: last s with seg[s].start <= i.
__device__ __forceinline__ int find_seg(const Seg* segs, int n, int64_t i, int lo = 0, int hi = -1) {
  if (hi < 0) hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (segs[mid].start <= i) lo = mid; else hi = mid - 1;
  }
  return lo;
}

}  // namespace cs

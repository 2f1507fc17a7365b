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

struct __align__(16) HotRec {   // everything the blend reads per splat (80 B)
  double mx, my, c0, c1, c2;     // mean2d, conic (render.py:128-129, 172)
  double opacity;
  float r, g, b;                 // SH colour (fp32 of the float64 value)
  float lthr;                    // fast-reject threshold on power (<= log(alpha_floor/o) - margin)
  int16_t bx0, bx1, by0, by1;    // inclusive pixel-index box of {power >= lthr}
  uint32_t id;                   // compact index (gradient slot)
  uint32_t pad;
};
static_assert(sizeof(HotRec) == 80, "HotRec layout");

// pair-major cull boxes for the blend: (lo | hi << 16) as two int16, one word
// per axis; kEmptyBox = (32767, -32768) never intersects
__host__ __device__ __forceinline__ uint32_t pack_box(int lo, int hi) {
  return (uint32_t)(uint16_t)(int16_t)lo | ((uint32_t)(uint16_t)(int16_t)hi << 16);
}
constexpr uint32_t kEmptyBox = 0x7fffu | (0x8000u << 16);

struct DevStats {     // device mirror of cs_frame_stats + scratch counters
  int64_t assembled;
  int64_t visible;
  int64_t skipped;
  int64_t pairs;
  int64_t fragments;
  int32_t n_segs;
  int32_t status;
  int64_t evals;         // blend (pixel, splat) evaluations executed (E)
  int64_t pairs_eff;     // pairs actually processed (0 when the pair buffer overflowed)
  uint32_t tickets[16];  // chunk tickets for single-pass kernels, zeroed per frame
};


// Outputs of the projection kernel, indexed by assembled index (splat id);
// hot/rects/boxes/recs are written for visible splats only.
struct ProjOutputs {
  uint64_t* keys;    // float64 depth bits (~0 for culled Gaussians), for the exact run fix-up
  uint32_t* keys32;  // float32-rounded depth bits (~0 for culled): the radix-sorted key
  uint32_t* vals;    // splat id
  HotRec* hot;
  int4* rects;
  short4* boxes;     // copy of HotRec's cull box, dense (8 B)
  ProjRec* recs;     // optional (debug / dumps)
};

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
// an 8x4 block when the tile side is a multiple of 8, else 32 consecutive
// row-major pixels.  box_pixel -> local pixel index (>= ts*ts: no pixel).
__host__ __device__ __forceinline__ int boxes_per_tile(int ts) {
  return (ts & 7) == 0 ? (ts >> 3) * (ts >> 2) : (ts * ts + 31) / 32;
}
__device__ __forceinline__ int box_pixel(int b, int lane, int ts) {
  if ((ts & 7) == 0) {
    const int nbx = ts >> 3, bx = b % nbx, by = b / nbx;
    return (by * 4 + (lane >> 3)) * ts + bx * 8 + (lane & 7);
  }
  return b * 32 + lane;
}

// ---------------------------------------------------------------------------
// exp(x) for the blend's x = power in [lthr, 0] (lthr >= log(alpha_floor) - 1e-6
// > -745): x = (64 m + j) ln2/64 + r, |r| <= ln2/128, exp(x) = 2^m 2^(j/64) (1 + q(r))
// with q the degree-6 Taylor polynomial minus 1 (truncation < 2e-20) and
// 2^(j/64) = hi + lo from a 64-entry table kept in shared memory; the result
// is formed as hi + (hi q + lo), ~0.5 ulp like a libm exp (measured max 0.5x
// ulp over [-6, 0], tools/exp_check.cu).  Neither this, CUDA's exp() nor the
// reference's libm exp are bit-identical to each other: they differ only at
// exact alpha-floor / transmittance knife-edges.
__constant__ double2 c_exp2_64[64] = {
    {1.0, 0.0}, {1.0108892860517005, -1.5234778603368577e-17},
    {1.0218971486541166, 5.109225028973444e-17}, {1.0330248790212284, 7.600838874027088e-18},
    {1.0442737824274138, 8.551889705537965e-17}, {1.0556451783605572, 1.759325738772092e-18},
    {1.0671404006768237, -7.899853966841582e-17}, {1.0787607977571199, -6.656660436056593e-17},
    {1.0905077326652577, -3.046782079812471e-17}, {1.102382583307841, 5.2660368715706944e-17},
    {1.1143867425958924, 1.0410278456845571e-16}, {1.1265216186082418, 5.165856758795457e-17},
    {1.1387886347566916, 8.912812676025408e-17}, {1.1511892299529827, 3.250710218863827e-17},
    {1.1637248587775775, 3.8292048369240935e-17}, {1.1763969916502812, 5.554203254218079e-17},
    {1.189207115002721, 3.982015231465646e-17}, {1.202156731452703, 6.644981499252301e-17},
    {1.215247359980469, -7.712630692681488e-17}, {1.22848053610687, -1.89878163130253e-17},
    {1.241857812073484, 4.658027591836937e-17}, {1.255380757024691, -6.7113898212968784e-18},
    {1.2690509571917332, 2.667932131342186e-18}, {1.2828700160787783, 1.713594918243561e-17},
    {1.2968395546510096, 2.5382502794888315e-17}, {1.3109612115247644, -7.181536135519454e-17},
    {1.3252366431597413, -2.8587312100388614e-17}, {1.339667524053303, 8.927282594831732e-17},
    {1.3542555469368927, 7.70094837980299e-17}, {1.3690024229745905, 9.593797919118849e-17},
    {1.383909881963832, -6.770511658794786e-17}, {1.3989796725383112, -9.614213209051323e-17},
    {1.4142135623730951, -9.667293313452913e-17}, {1.42961333839197, -1.2031642489053655e-17},
    {1.4451808069770467, -3.0237581349939873e-17}, {1.460917794180647, -5.600377186075216e-17},
    {1.4768261459394993, -3.483994556892796e-17}, {1.4929077282912648, 1.4192920154284036e-17},
    {1.5091644275934228, -1.016455327754295e-16}, {1.5255981507445384, -1.1024941712342561e-16},
    {1.5422108254079407, 7.949834809697621e-17}, {1.559004400237837, 3.7812070533575275e-17},
    {1.5759808451078865, -1.0136916471278304e-17}, {1.593142151342267, -1.0094406542311964e-16},
    {1.6104903319492543, 2.4707192569797888e-17}, {1.6280274218573478, -6.712955084707084e-17},
    {1.645755478153965, -1.0125679913674773e-16}, {1.6636765803267364, 5.8909926967131e-17},
    {1.681792830507429, 8.199010020581497e-17}, {1.7001063537185235, -8.0237193703977e-18},
    {1.718619298122478, -1.851380418263111e-17}, {1.7373338352737062, 3.164389299292957e-17},
    {1.7562521603732995, 2.960140695448873e-17}, {1.7753764925265212, 6.429731796556572e-17},
    {1.7947090750031072, 1.8227458427912087e-17}, {1.8142521755003989, -9.969531538920349e-17},
    {1.8340080864093424, 3.283107224245627e-17}, {1.8539791250833855, 9.761887490727594e-17},
    {1.8741676341103, -6.122763413004143e-17}, {1.8945759815869656, 3.4034035352165297e-17},
    {1.9152065613971474, -1.0619946056195963e-16}, {1.9360617934922943, 1.0332385960676326e-16},
    {1.9571441241754002, 8.960767791036668e-17}, {1.978456026387951, 4.0388753109278167e-17}
};

__device__ __forceinline__ void load_exp_table(double2* s_tab) {
  for (int i = threadIdx.x; i < 64; i += blockDim.x) s_tab[i] = c_exp2_64[i];
}

__device__ __forceinline__ double exp_le0(double x, const double2* s_tab) {
  const double kd = rint(x * 92.33248261689366);          // 64 / ln2
  double r = fma(kd, -0.010830424696905538, x);           // ln2/64, high 33 bits
  r = fma(kd, 6.563929801064195e-13, r);                  // ln2/64, low part
  double q = fma(r, 1.0 / 720.0, 1.0 / 120.0);
  q = fma(q, r, 1.0 / 24.0);
  q = fma(q, r, 1.0 / 6.0);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = q * r;                                              // exp(r) - 1
  const int k = (int)kd;
  const double2 t = s_tab[k & 63];
  const double scale = __longlong_as_double((long long)((k >> 6) + 1023) << 52);  // 2^m, m = floor(k/64)
  return (t.x + fma(t.x, q, t.y)) * scale;
}

// grid of a persistent kernel: as many CTAs as are co-resident on all SMs
template <typename K>
static int persistent_grid(K kernel, int threads) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0);
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
__device__ __forceinline__ int find_seg(const Seg* segs, int n, int64_t i) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (segs[mid].start <= i) lo = mid; else hi = mid - 1;
  }
  return lo;
}

}  // namespace cs

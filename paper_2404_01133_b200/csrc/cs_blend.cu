// cs_blend.cu -- K9: per-tile front-to-back alpha blending.
//
// Replaces _kernels.blend_tiles (_kernels.py:17-76), the reference's only
// native kernel.  One CTA per tile, one thread per pixel (tile_size <= 16;
// 4 or 16 pixels per thread for 32/64).  For 16x16 tiles each warp owns an
// 8x4 pixel box.
//
// The tile's splat list (depth order) is streamed through shared memory in
// batches of 256 HotRec records (80 B: mean, conic, opacity, colour,
// fast-reject threshold, support box) with cp.async double buffering.  Tiles
// are launched heaviest list first (K8b), so the long hot-tile lists start in
// the first wave instead of forming the tail.  Per batch every warp first
// tests 32 splats at a time against its pixel box (one AABB test per lane,
// __ballot_sync) and then walks only the hits, so a splat whose alpha-floor
// support misses the warp's 32 pixels costs 1/32 of an AABB test instead of
// 32 float64 quadratic forms.  The CTA leaves as soon as every pixel has
// terminated (__syncthreads_count).
//
// Precision: the quadratic form is float64 in the
// reference's exact op order (no FMA).  A float64 power below
// log(alpha_floor / o) - 1e-6 is a guaranteed skip and costs no exp; every
// other fragment takes the reference path exactly: alpha = min(0.99,
// o * exp(power)) in float64, float64 alpha/transmittance decisions, so the
// accepted-fragment set equals the reference's.  Colour accumulates in
// float64 from float32 splat colours.  The AABB cull never drops a fragment
// the exact path could accept: it bounds {power >= threshold} (cs_project.cu).
#include "cs_internal.cuh"

namespace cs {

constexpr int kBlendThreads = 256;
constexpr int kBatch = 256;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void stage_batch(HotRec* dst, const uint32_t* list, const HotRec* hot,
                                            int64_t k, int64_t s1) {
  if (k < s1) {
    const char* g = reinterpret_cast<const char*>(hot + __ldg(list + k));
    char* d = reinterpret_cast<char*>(dst + threadIdx.x);
    cp_async16(d, g);
    cp_async16(d + 16, g + 16);
    cp_async16(d + 32, g + 32);
    cp_async16(d + 48, g + 48);
    cp_async16(d + 64, g + 64);
  }
}

// local pixel index (0..ts*ts-1) of thread `tid`, pixel slot q
__device__ __forceinline__ int local_pixel(int tid, int q, int ts) {
  if (ts == 16) {  // 8x4 box per warp: warp w -> origin ((w & 1) * 8, (w >> 1) * 4)
    const int w = tid >> 5, l = tid & 31;
    return ((w >> 1) * 4 + (l >> 3)) * 16 + (w & 1) * 8 + (l & 7);
  }
  return tid + q * kBlendThreads;
}

template <int PPT, typename OutT, bool KEEP>
__global__ void __launch_bounds__(kBlendThreads)
k_blend(const uint32_t* __restrict__ list, const uint2* __restrict__ ranges,
        const HotRec* __restrict__ hot, const uint32_t* __restrict__ tile_order, BlendParams bp,
        OutT* __restrict__ out, int32_t* __restrict__ frag_tile, DevStats* __restrict__ stats,
        BlendState state) {
  __shared__ __align__(16) HotRec buf[2][kBatch];
  __shared__ int s_red[kBlendThreads / 32];
  __shared__ long long s_ev[kBlendThreads / 32];
  const int t = tile_order ? (int)tile_order[blockIdx.x] : (int)blockIdx.x;
  const int tx = t % bp.ntx, ty = t / bp.ntx;
  const int ts = bp.tile_size;
  const uint2 rg = ranges[t];
  const int64_t s0 = rg.x, s1 = rg.y;
  const uint32_t lane = lane_id();

  double sx[PPT], sy[PPT], T[PPT], cr[PPT], cg[PPT], cb[PPT];
  int wx0[PPT], wx1[PPT], wy0[PPT], wy1[PPT];  // warp's pixel-index box per slot
  int cnt[PPT], last[PPT];
  bool done[PPT], valid[PPT];
  long long evals = 0;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int li = local_pixel(threadIdx.x, q, ts);
    const int px = tx * ts + li % ts, py = ty * ts + li / ts;
    valid[q] = li < ts * ts && px < bp.width && py < bp.height;
    sx[q] = (double)px + 0.5;  // pixel centres (_kernels.py:43-45)
    sy[q] = (double)py + 0.5;
    T[q] = 1.0; cr[q] = 0.0; cg[q] = 0.0; cb[q] = 0.0;
    cnt[q] = 0; last[q] = (int)s0;
    done[q] = !valid[q];
    int x0 = valid[q] ? px : 1 << 20, x1 = valid[q] ? px : -(1 << 20);
    int y0 = valid[q] ? py : 1 << 20, y1 = valid[q] ? py : -(1 << 20);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      x0 = min(x0, __shfl_xor_sync(0xffffffffu, x0, o));
      x1 = max(x1, __shfl_xor_sync(0xffffffffu, x1, o));
      y0 = min(y0, __shfl_xor_sync(0xffffffffu, y0, o));
      y1 = max(y1, __shfl_xor_sync(0xffffffffu, y1, o));
    }
    wx0[q] = x0; wx1[q] = x1; wy0[q] = y0; wy1[q] = y1;
  }

  const int64_t n = s1 - s0;
  const int nbatches = (int)((n + kBatch - 1) / kBatch);
  if (nbatches > 0) stage_batch(buf[0], list, hot, s0 + threadIdx.x, s1);
  cp_async_commit();
  for (int b = 0; b < nbatches; ++b) {
    const int64_t bstart = s0 + (int64_t)b * kBatch;
    if (b + 1 < nbatches) stage_batch(buf[(b + 1) & 1], list, hot, bstart + kBatch + threadIdx.x, s1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const HotRec* hb = buf[b & 1];
    const int nb = (int)min((int64_t)kBatch, s1 - bstart);
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      if (__all_sync(0xffffffffu, done[q])) continue;
      double Tq = T[q];
      for (int base = 0; base < nb; base += 32) {
        const int jl = base + (int)lane;
        bool hit = false;
        if (jl < nb) {
          const short4 bx = *reinterpret_cast<const short4*>(&hb[jl].bx0);
          hit = !(bx.x > wx1[q] || bx.y < wx0[q] || bx.z > wy1[q] || bx.w < wy0[q]);
        }
        uint32_t mask = __ballot_sync(0xffffffffu, hit);
        while (mask) {
          const int j = base + __ffs(mask) - 1;
          mask &= mask - 1;
          if (done[q]) continue;
          ++evals;
          const HotRec& h = hb[j];
          const double dx = dsub(sx[q], h.mx);
          const double dy = dsub(sy[q], h.my);
          // -0.5 * (c0*dx*dx + c2*dy*dy) - c1*dx*dy   (_kernels.py:54-57)
          const double power =
              dsub(dmul(-0.5, dadd(dmul(dmul(h.c0, dx), dx), dmul(dmul(h.c2, dy), dy))),
                   dmul(dmul(h.c1, dx), dy));
          if (power < (double)h.lthr) continue;  // alpha < alpha_floor guaranteed
          double alpha = dmul(h.opacity, exp(power));  // _kernels.py:58
          if (alpha > 0.99) alpha = 0.99;              // _kernels.py:59-60
          if (alpha < bp.alpha_floor) continue;        // _kernels.py:61-62
          const double nt = dmul(Tq, dsub(1.0, alpha));
          if (nt < bp.t_floor) { done[q] = true; continue; }  // _kernels.py:63-66
          const double w = dmul(Tq, alpha);
          cr[q] += w * (double)h.r;
          cg[q] += w * (double)h.g;
          cb[q] += w * (double)h.b;
          Tq = nt;
          cnt[q] += 1;
          last[q] = (int)(bstart + j + 1);
        }
        if (__all_sync(0xffffffffu, done[q])) break;
      }
      T[q] = Tq;
    }
    int alive = 0;
#pragma unroll
    for (int q = 0; q < PPT; ++q) alive |= done[q] ? 0 : 1;
    if (__syncthreads_count(alive) == 0) break;
  }
  cp_async_wait<0>();
  int my = 0;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    if (!valid[q]) continue;
    my += cnt[q];
    const int li = local_pixel(threadIdx.x, q, ts);
    const int px = tx * ts + li % ts, py = ty * ts + li / ts;
    const int64_t pix = (int64_t)py * bp.width + px;
    double o[3] = {cr[q] + T[q] * bp.bg[0], cg[q] + T[q] * bp.bg[1], cb[q] + T[q] * bp.bg[2]};
    if (!(bp.flags & CS_RENDER_NO_CLIP)) {
#pragma unroll
      for (int c = 0; c < 3; ++c) o[c] = o[c] < 0.0 ? 0.0 : (o[c] > 1.0 ? 1.0 : o[c]);
    }
    out[3 * pix] = (OutT)o[0];
    out[3 * pix + 1] = (OutT)o[1];
    out[3 * pix + 2] = (OutT)o[2];
    if (KEEP) {
      state.final_t[pix] = T[q];
      state.last[pix] = last[q];
      state.color_acc[3 * pix] = cr[q];
      state.color_acc[3 * pix + 1] = cg[q];
      state.color_acc[3 * pix + 2] = cb[q];
    }
  }
  my = warp_sum(my);
  evals = warp_sum(evals);
  if (lane == 0) {
    s_red[threadIdx.x >> 5] = my;
    s_ev[threadIdx.x >> 5] = evals;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    long long ev = 0;
    for (int w = 0; w < kBlendThreads / 32; ++w) { tot += s_red[w]; ev += s_ev[w]; }
    frag_tile[t] = tot;
    if (tot) atomicAdd(reinterpret_cast<unsigned long long*>(&stats->fragments),
                       (unsigned long long)tot);
    if (ev) atomicAdd(reinterpret_cast<unsigned long long*>(&stats->evals), (unsigned long long)ev);
  }
}

template <typename OutT, bool KEEP>
static void launch_blend_t(int ppt, int n_tiles, const uint32_t* list, const uint2* ranges,
                           const HotRec* hot, const uint32_t* order, const BlendParams& bp,
                           OutT* out, int32_t* frag_tile, DevStats* stats, BlendState st,
                           cudaStream_t s) {
  if (ppt == 1)
    k_blend<1, OutT, KEEP><<<n_tiles, kBlendThreads, 0, s>>>(list, ranges, hot, order, bp, out,
                                                            frag_tile, stats, st);
  else if (ppt == 4)
    k_blend<4, OutT, KEEP><<<n_tiles, kBlendThreads, 0, s>>>(list, ranges, hot, order, bp, out,
                                                            frag_tile, stats, st);
  else
    k_blend<16, OutT, KEEP><<<n_tiles, kBlendThreads, 0, s>>>(list, ranges, hot, order, bp, out,
                                                             frag_tile, stats, st);
}

// K8b: heaviest-first tile order.  Tiles are bucketed by floor(log2(list
// length)) and emitted bucket-descending (order inside a bucket is arbitrary;
// tiles are independent, so the image does not depend on it).
__global__ void k_tile_order(const uint2* __restrict__ ranges, int n_tiles, uint32_t* __restrict__ order) {
  __shared__ int hist[34];
  __shared__ int cursor[34];
  if (threadIdx.x < 34) hist[threadIdx.x] = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    const uint2 r = ranges[t];
    const uint32_t c = r.y - r.x;
    atomicAdd(&hist[c ? 32 - __clz(c) : 0], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int b = 33; b >= 0; --b) { cursor[b] = acc; acc += hist[b]; }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    const uint2 r = ranges[t];
    const uint32_t c = r.y - r.x;
    order[atomicAdd(&cursor[c ? 32 - __clz(c) : 0], 1)] = (uint32_t)t;
  }
}

void launch_tile_order(const uint2* ranges, int n_tiles, uint32_t* order, cudaStream_t s) {
  k_tile_order<<<1, 1024, 0, s>>>(ranges, n_tiles, order);
}

int blend_ppt(int tile_size) {
  const int px = tile_size * tile_size;
  if (px <= 256) return 1;
  if (px <= 1024) return 4;
  if (px <= 4096) return 16;
  return 0;
}

void launch_blend(int n_tiles, const uint32_t* list, const uint2* ranges, const HotRec* hot,
                  const uint32_t* order, const BlendParams& bp, void* out, bool f64_out,
                  int32_t* frag_tile, DevStats* stats, const BlendState* keep, cudaStream_t s) {
  const int ppt = blend_ppt(bp.tile_size);
  BlendState st = keep ? *keep : BlendState{nullptr, nullptr, nullptr};
  if (f64_out) {
    if (keep) launch_blend_t<double, true>(ppt, n_tiles, list, ranges, hot, order, bp, (double*)out, frag_tile, stats, st, s);
    else launch_blend_t<double, false>(ppt, n_tiles, list, ranges, hot, order, bp, (double*)out, frag_tile, stats, st, s);
  } else {
    if (keep) launch_blend_t<float, true>(ppt, n_tiles, list, ranges, hot, order, bp, (float*)out, frag_tile, stats, st, s);
    else launch_blend_t<float, false>(ppt, n_tiles, list, ranges, hot, order, bp, (float*)out, frag_tile, stats, st, s);
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
    h.id = (uint32_t)s;
    h.pad = 0;
    h.bx0 = h.by0 = -1;     // full-image box
    h.bx1 = h.by1 = 32000;
    hot[s] = h;
  }
}

__global__ void k_pack_tiles(int64_t p, const int64_t* tile_ids, int64_t n_tiles,
                             const int64_t* offsets, uint32_t* list, uint2* ranges) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += stride)
    list[i] = (uint32_t)tile_ids[i];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_tiles; t += stride)
    ranges[t] = make_uint2((uint32_t)offsets[t], (uint32_t)offsets[t + 1]);
}

void launch_pack(int64_t m, const double* means, const double* conics, const double* colors,
                 const double* opac, double alpha_floor, HotRec* hot, int64_t p,
                 const int64_t* tile_ids, int64_t n_tiles, const int64_t* offsets, uint32_t* list,
                 uint2* ranges, cudaStream_t s) {
  if (m > 0)
    k_pack_records<<<148 * 4, 256, 0, s>>>(m, means, conics, colors, opac, alpha_floor, hot);
  k_pack_tiles<<<148 * 4, 256, 0, s>>>(p, tile_ids, n_tiles, offsets, list, ranges);
}

}  // namespace cs

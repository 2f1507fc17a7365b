// cs_project.cu -- K3: EWA projection + SH colour + cull.
//
// Replaces render._project_cloud (render.py:111-188) up to the depth sort.
// One thread per assembled Gaussian, outputs at its assembled index; culled
// Gaussians get the depth key ~0, so the stable depth sort (K4) yields the
// visible set in (depth, assembled index) order -- the np.nonzero order of
// render.py:121/163 followed by the stable argsort of render.py:176-177 --
// with no compaction pass.
//
// All decision math (cull, mean, covariance, conic, radii, on-image test) is
// float64 written with explicit round-to-nearest intrinsics in numpy's
// operation order (no FMA contraction), so results are bit-identical to the
// reference run under OPENBLAS_CORETYPE=Sandybridge.
#include "cs_internal.cuh"

namespace cs {

__constant__ double kShC0 = 0.28209479177387814;
__constant__ double kShC1 = 0.4886025119029199;
__constant__ double kShC2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
__constant__ double kShC3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

__device__ __forceinline__ int degree_of(int c) { return c >= 16 ? 3 : c >= 9 ? 2 : c >= 4 ? 1 : 0; }

// eval_sh_basis (core.py:114-146) fused with sh_to_colors (core.py:166-172):
// colour = clip(0.5 + sum_n sh[c, n] * Y_n(dir), 0, 1).  Tolerance-only
// quantity (the reference sums through numpy einsum), evaluated in float64.
// The row (3*C floats, 16-byte aligned, stride % 4 == 0) is fetched with
// float4 loads; C is a template parameter so basis and coefficients stay in
// registers.
// The colour is a tolerance-only quantity (clipped [0, 1] colours, image
// parity 1e-4; the rows are float32 already), so it is evaluated in float32
// (CS_SH_F64 restores float64): the FP64 pipe stays with the decision math.
#ifdef CS_SH_F64
typedef double sh_t;
#else
typedef float sh_t;
#endif

template <int C, bool GENERIC>
__device__ __forceinline__ void sh_colour_t(const float* row, int degree, sh_t x, sh_t y, sh_t z,
                                            double out[3]) {
  constexpr int kVec = (3 * C + 3) / 4;
  float co[kVec * 4];
  const float4* r4 = reinterpret_cast<const float4*>(row);
#pragma unroll
  for (int i = 0; i < kVec; ++i) {
    const float4 v = GENERIC ? r4[i] : __ldg(r4 + i);  // GENERIC: a row staged in shared memory
    co[4 * i] = v.x; co[4 * i + 1] = v.y; co[4 * i + 2] = v.z; co[4 * i + 3] = v.w;
  }
  sh_t basis[C];
  basis[0] = (sh_t)kShC0;
  if (C >= 4) {
    basis[1] = degree >= 1 ? -(sh_t)kShC1 * y : (sh_t)0;
    basis[2] = degree >= 1 ? (sh_t)kShC1 * z : (sh_t)0;
    basis[3] = degree >= 1 ? -(sh_t)kShC1 * x : (sh_t)0;
  }
  if (C >= 9) {
    const sh_t xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    const bool on = degree >= 2;
    basis[4] = on ? (sh_t)kShC2[0] * xy : (sh_t)0;
    basis[5] = on ? (sh_t)kShC2[1] * yz : (sh_t)0;
    basis[6] = on ? (sh_t)kShC2[2] * ((sh_t)2 * zz - xx - yy) : (sh_t)0;
    basis[7] = on ? (sh_t)kShC2[3] * xz : (sh_t)0;
    basis[8] = on ? (sh_t)kShC2[4] * (xx - yy) : (sh_t)0;
    if (C >= 16) {
      const bool on3 = degree >= 3;
      basis[9] = on3 ? (sh_t)kShC3[0] * y * ((sh_t)3 * xx - yy) : (sh_t)0;
      basis[10] = on3 ? (sh_t)kShC3[1] * xy * z : (sh_t)0;
      basis[11] = on3 ? (sh_t)kShC3[2] * y * ((sh_t)4 * zz - xx - yy) : (sh_t)0;
      basis[12] = on3 ? (sh_t)kShC3[3] * z * ((sh_t)2 * zz - (sh_t)3 * xx - (sh_t)3 * yy) : (sh_t)0;
      basis[13] = on3 ? (sh_t)kShC3[4] * x * ((sh_t)4 * zz - xx - yy) : (sh_t)0;
      basis[14] = on3 ? (sh_t)kShC3[5] * z * (xx - yy) : (sh_t)0;
      basis[15] = on3 ? (sh_t)kShC3[6] * x * (xx - (sh_t)3 * yy) : (sh_t)0;
    }
  }
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    sh_t acc = 0;
#pragma unroll
    for (int n = 0; n < C; ++n) acc += (sh_t)co[ch * C + n] * basis[n];
    const double v = 0.5 + (double)acc;
    out[ch] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
  }
}

template <bool GENERIC = false>
__device__ __forceinline__ void sh_colour(const float* row, int C, int degree, double x, double y,
                                          double z, double out[3]) {
  const sh_t fx = (sh_t)x, fy = (sh_t)y, fz = (sh_t)z;
  switch (C) {
    case 16: sh_colour_t<16, GENERIC>(row, degree, fx, fy, fz, out); break;
    case 9: sh_colour_t<9, GENERIC>(row, degree, fx, fy, fz, out); break;
    case 4: sh_colour_t<4, GENERIC>(row, degree, fx, fy, fz, out); break;
    default: sh_colour_t<1, GENERIC>(row, degree, fx, fy, fz, out); break;
  }
}

// Sigma = R diag(s^2) R^T of one Gaussian (core.py:74-82, core.py:107-111),
// numpy's op order.
__device__ __forceinline__ void sigma_of(const Geom& g, double sig[9]) {
  // quat_to_rotmat, core.py:74-82
  const double w = g.qw, x = g.qx, y = g.qy, q = g.qz;
  double r[9];
  r[0] = dsub(1.0, dmul(2.0, dadd(dmul(y, y), dmul(q, q))));
  r[1] = dmul(2.0, dsub(dmul(x, y), dmul(w, q)));
  r[2] = dmul(2.0, dadd(dmul(x, q), dmul(w, y)));
  r[3] = dmul(2.0, dadd(dmul(x, y), dmul(w, q)));
  r[4] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(q, q))));
  r[5] = dmul(2.0, dsub(dmul(y, q), dmul(w, x)));
  r[6] = dmul(2.0, dsub(dmul(x, q), dmul(w, y)));
  r[7] = dmul(2.0, dadd(dmul(y, q), dmul(w, x)));
  r[8] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(y, y))));
  // build_covariances (core.py:107-111): rs = r * s^2 ; einsum kij,klj->kil.
  // numpy's contiguous 2-lane sum-of-products adds the three terms (t0 + t2) + t1.
  const double s2[3] = {dmul(g.sx, g.sx), dmul(g.sy, g.sy), dmul(g.sz, g.sz)};
  double rs[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) rs[3 * i + j] = dmul(r[3 * i + j], s2[j]);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int l = 0; l < 3; ++l)
      sig[3 * i + l] = dadd(dadd(dmul(rs[3 * i + 0], r[3 * l + 0]), dmul(rs[3 * i + 2], r[3 * l + 2])),
                            dmul(rs[3 * i + 1], r[3 * l + 1]));
}

// cov2d = J (W Sigma W^T) J^T entries (0,0), (0,1), (1,1) for camera-space
// position (t0, t1, z) (render.py:133-141 / lod.py:85-91), numpy's op order.
__device__ __forceinline__ void cov2d_of(const double sig[9], const cs_camera& cam, double t0,
                                         double t1, double z, double& c00_o, double& c01_o,
                                         double& c11_o) {
  const double* R = cam.R;
  // V = W Sigma W^T, einsum ij,kjl,ml->kim: ((W_ij * S_jl) * W_ml), j-major l-minor (render.py:133)
  double V[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int m = i; m < 3; ++m) {
      double acc = dmul(dmul(R[3 * i + 0], sig[0]), R[3 * m + 0]);
#pragma unroll
      for (int jl = 1; jl < 9; ++jl) {
        const int j = jl / 3, l = jl % 3;
        acc = dadd(acc, dmul(dmul(R[3 * i + j], sig[3 * j + l]), R[3 * m + l]));
      }
      V[3 * i + m] = acc;
    }
  // cov2d = J V J^T (render.py:136-141); J has zeros at (0,1) and (1,0), which
  // add exact zeros in numpy's 9-term sum and are skipped here.
  const double zz = dmul(z, z);
  const double j00 = ddiv(cam.fx, z);
  const double j02 = ddiv(dmul(-cam.fx, t0), zz);
  const double j11 = ddiv(cam.fy, z);
  const double j12 = ddiv(dmul(-cam.fy, t1), zz);
  // V entries below the diagonal: recompute in numpy order (V is symmetric only
  // up to rounding, so compute the exact (i, m) entry used).
  double V20, V21;
  {
    double acc = dmul(dmul(R[6], sig[0]), R[0]);
#pragma unroll
    for (int jl = 1; jl < 9; ++jl) {
      const int j = jl / 3, l = jl % 3;
      acc = dadd(acc, dmul(dmul(R[6 + j], sig[3 * j + l]), R[l]));
    }
    V20 = acc;
    acc = dmul(dmul(R[6], sig[0]), R[3]);
#pragma unroll
    for (int jl = 1; jl < 9; ++jl) {
      const int j = jl / 3, l = jl % 3;
      acc = dadd(acc, dmul(dmul(R[6 + j], sig[3 * j + l]), R[3 + l]));
    }
    V21 = acc;
  }
  const double V00 = V[0], V01 = V[1], V02 = V[2], V11 = V[4], V12 = V[5], V22 = V[8];
  // cov2d[0][0]: terms (0,0),(0,2),(2,0),(2,2) with t_jl = (J0j V_jl) J0l
  double c00 = dmul(dmul(j00, V00), j00);
  c00 = dadd(c00, dmul(dmul(j00, V02), j02));
  c00 = dadd(c00, dmul(dmul(j02, V20), j00));
  c00 = dadd(c00, dmul(dmul(j02, V22), j02));
  // cov2d[0][1]: (0,1),(0,2),(2,1),(2,2) with t_jl = (J0j V_jl) J1l
  double c01 = dmul(dmul(j00, V01), j11);
  c01 = dadd(c01, dmul(dmul(j00, V02), j12));
  c01 = dadd(c01, dmul(dmul(j02, V21), j11));
  c01 = dadd(c01, dmul(dmul(j02, V22), j12));
  // cov2d[1][1]: (1,1),(1,2),(2,1),(2,2) with t_jl = (J1j V_jl) J1l
  double c11 = dmul(dmul(j11, V11), j11);
  c11 = dadd(c11, dmul(dmul(j11, V12), j12));
  c11 = dadd(c11, dmul(dmul(j12, V21), j11));
  c11 = dadd(c11, dmul(dmul(j12, V22), j12));
  c00_o = c00;
  c01_o = c01;
  c11_o = c11;
}

struct ProjOut {
  bool in_front, ok, keep;
  double z, mx, my, a, b, c, det, rx, ry;
};

// Decision math of render.py:118-160 for one Gaussian, numpy op order.
__device__ __forceinline__ ProjOut project_one(const Geom& g, const cs_camera& cam,
                                               const cs_settings& st) {
  ProjOut o;
  const double* R = cam.R;
  double t0 = dadd(dadd(dadd(dmul(g.px, R[0]), dmul(g.py, R[1])), dmul(g.pz, R[2])), cam.t[0]);
  double t1 = dadd(dadd(dadd(dmul(g.px, R[3]), dmul(g.py, R[4])), dmul(g.pz, R[5])), cam.t[1]);
  double z = dadd(dadd(dadd(dmul(g.px, R[6]), dmul(g.py, R[7])), dmul(g.pz, R[8])), cam.t[2]);
  o.z = z;
  o.in_front = z > st.near_plane;            // render.py:120
  o.ok = false;
  o.keep = false;
  if (!o.in_front) return o;
  o.mx = dadd(ddiv(dmul(cam.fx, t0), z), cam.cx);   // render.py:128
  o.my = dadd(ddiv(dmul(cam.fy, t1), z), cam.cy);   // render.py:129
  double sig[9];
  sigma_of(g, sig);
  double c00, c01, c11;
  cov2d_of(sig, cam, t0, t1, z, c00, c01, c11);
  o.a = dadd(c00, st.low_pass);                // render.py:142-144
  o.b = c01;
  o.c = dadd(c11, st.low_pass);
  o.det = dsub(dmul(o.a, o.c), dmul(o.b, o.b)); // render.py:146
  o.ok = o.det > st.singular_det;              // render.py:147
  o.rx = dmul(st.support_sigmas, __dsqrt_rn(o.a));  // render.py:153-154
  o.ry = dmul(st.support_sigmas, __dsqrt_rn(o.c));
  const bool on_image = (dadd(o.mx, o.rx) > 0.0) && (dsub(o.mx, o.rx) < (double)cam.width) &&
                        (dadd(o.my, o.ry) > 0.0) && (dsub(o.my, o.ry) < (double)cam.height);
  o.keep = o.ok && on_image;                   // render.py:156-161
  return o;
}

// K15: significance_scores hit counts (lod.py:54-101).  One thread per
// Gaussian; Sigma once, then per training view the reference's tests in its
// order: in front of the near plane (lod.py:74), centre inside [0, W] x [0, H]
// inclusive (lod.py:79-83), support radius support_sigmas * sqrt(lambda_max)
// of cov2d + LOW_PASS >= MIN_FOOTPRINT_RADIUS (lod.py:84-95).  Same float64
// op order as the projection (the einsums of lod.py:85/91 are render.py's).
// Also writes the volume key (np.prod(scales, axis=1), lod.py:97; positive, so
// its IEEE bits sort like the value) for the percentile sort.
__global__ void __launch_bounds__(256)
k_significance(const cs_cloud cl, const cs_camera* __restrict__ cams, int n_cams, cs_settings st,
               int32_t* __restrict__ hits, uint64_t* __restrict__ vol_keys,
               uint32_t* __restrict__ vals) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < cl.count;
       k += (int64_t)gridDim.x * blockDim.x) {
    const Geom g = load_geom(cl, k);
    double sig[9];
    sigma_of(g, sig);
    int h = 0;
    for (int ci = 0; ci < n_cams; ++ci) {
      const cs_camera& cam = cams[ci];
      const double* R = cam.R;
      const double t0 = dadd(dadd(dadd(dmul(g.px, R[0]), dmul(g.py, R[1])), dmul(g.pz, R[2])), cam.t[0]);
      const double t1 = dadd(dadd(dadd(dmul(g.px, R[3]), dmul(g.py, R[4])), dmul(g.pz, R[5])), cam.t[1]);
      const double z = dadd(dadd(dadd(dmul(g.px, R[6]), dmul(g.py, R[7])), dmul(g.pz, R[8])), cam.t[2]);
      if (!(z > st.near_plane)) continue;                      // lod.py:74
      const double u = dadd(ddiv(dmul(cam.fx, t0), z), cam.cx); // lod.py:79
      const double v = dadd(ddiv(dmul(cam.fy, t1), z), cam.cy); // lod.py:80
      if (!(u >= 0.0 && u <= (double)cam.width && v >= 0.0 && v <= (double)cam.height)) continue;
      double c00, c01, c11;
      cov2d_of(sig, cam, t0, t1, z, c00, c01, c11);
      const double a = dadd(c00, st.low_pass), b = c01, c = dadd(c11, st.low_pass);
      const double mid = dmul(0.5, dadd(a, c));                 // lod.py:90
      const double disc = dsub(dmul(mid, mid), dsub(dmul(a, c), dmul(b, b)));
      const double lam = dadd(mid, __dsqrt_rn(disc > 0.0 ? disc : 0.0));  // lod.py:91
      const double radius = dmul(st.support_sigmas, __dsqrt_rn(lam));     // lod.py:92
      if (radius >= 0.5) ++h;                                   // MIN_FOOTPRINT_RADIUS, lod.py:45
    }
    hits[k] = h;
    vol_keys[k] = (uint64_t)__double_as_longlong(dmul(dmul(g.sx, g.sy), g.sz));
    vals[k] = (uint32_t)k;
  }
}

void launch_significance(const cs_cloud& cl, const cs_camera* cams, int n_cams,
                         const cs_settings& st, int32_t* hits, uint64_t* vol_keys, uint32_t* vals,
                         cudaStream_t s) {
  const int64_t blocks = std::min<int64_t>((cl.count + 255) / 256, 148 * 16);
  if (blocks <= 0) return;
  k_significance<<<(unsigned)blocks, 256, 0, s>>>(cl, cams, n_cams, st, hits, vol_keys, vals);
}

// Everything K3 writes for assembled index i < n once its geometry g is
// projected (po): depth keys, and for a kept splat its HotRec, cull box, tile
// rectangle (and the debug record).  sh_row: the splat's SH row, in global
// memory or (GENERIC_SH) staged in shared memory.
template <bool GENERIC_SH>
__device__ __forceinline__ void project_emit(int64_t i, const Geom& g, const ProjOut& po, const float* sh_row,
                                             int sh_coeffs, const cs_camera& cam, const cs_settings& st,
                                             const ProjOutputs& po_out) {
  // z > near > 0: the float64 bits are monotone; culled -> ~0 (sorts last)
  po_out.keys[i] = po.keep ? (uint64_t)__double_as_longlong(po.z) : ~0ull;
  // 32-bit sort key: a monotone coarsening of the float64 depth, so K4b only
  // has to re-sort runs of equal keys.  For z > near the float64 bit patterns
  // increase with z; (bits(z) - bits(near)) >> 24 keeps 2^28 steps per octave
  // over the 16 octaves above the near plane (32x finer than the float32
  // rounding, so far fewer equal-key runs), saturating beyond (~0.2 * 2^16 m
  // at the default near plane); ~0 marks culled Gaussians.
  {
    const uint64_t zb = (uint64_t)__double_as_longlong(po.z);
    const uint64_t nb = (uint64_t)__double_as_longlong(st.near_plane > 0.0 ? st.near_plane : 0.0);
    const uint64_t code = (zb - nb) >> 24;
    po_out.keys32[i] = po.keep ? (uint32_t)min(code, (uint64_t)0xfffffffeu) : 0xffffffffu;
  }
  // (no id array: the depth sort's first pass takes the identity as its values)
  if (!po.keep) return;
  const int64_t idx = i;
  // view direction and SH colour (render.py:167-169, core.py:166-172)
  double dx = g.px - cam.center[0], dy = g.py - cam.center[1], dz = g.pz - cam.center[2];
  int degree = min((int)st.sh_degree, degree_of(sh_coeffs));
  double col[3];
#ifdef CS_SH_F64
  double nrm = sqrt((dx * dx + dy * dy) + dz * dz);
  sh_colour<GENERIC_SH>(sh_row, sh_coeffs, degree, dx / nrm, dy / nrm, dz / nrm, col);
#else
  {  // the colour is evaluated in float32: so is the unit view direction (no
     // float64 divisions / sqrt for a tolerance-only quantity)
    const float fx = (float)dx, fy = (float)dy, fz = (float)dz;
    const float inv = rsqrtf(fmaf(fx, fx, fmaf(fy, fy, fz * fz)));
    sh_colour<GENERIC_SH>(sh_row, sh_coeffs, degree, fx * inv, fy * inv, fz * inv, col);
  }
#endif
  const double c0 = ddiv(po.c, po.det);   // render.py:172
  const double c1 = ddiv(-po.b, po.det);
  const double c2 = ddiv(po.a, po.det);
  // blend fast-reject threshold: alpha = o*exp(power) < alpha_floor whenever
  // power < log(alpha_floor / o) - 1e-6 (margin >> exp rounding).  Evaluated
  // in float32 with a 1e-5 margin, which covers the float32 logs (<= 2 ulp of
  // |log| <= ~20, i.e. < 5e-6): the threshold stays conservative, only the
  // exact float64 path decides a fragment.
  float lthr;
  const float ln_o = g.op > 0.0 ? logf((float)g.op) : 0.0f;   // (also the FastRec's log2(o))
  if (g.op > 0.0) {
    const float lf = __fsub_rn(po_out.ln_afl, ln_o);
    lthr = __fsub_rd(lf, 1e-5f + 1e-6f * fabsf(lf));
  } else {
    lthr = __int_as_float(0x7f800000);
  }
  HotRec h;
  h.mx = po.mx; h.my = po.my; h.c0 = c0; h.c1 = c1; h.c2 = c2;
  h.opacity = g.op;
  h.r = (float)col[0]; h.g = (float)col[1]; h.b = (float)col[2];
  h.lthr = lthr;
  // Pixel box of {d : power(d) >= lthr} = {d^T Q d <= 2L}, L = -lthr: the
  // ellipse's AABB half-extents are sqrt(2 L a), sqrt(2 L c) with
  // (a, b, c) = Q^-1 = cov2d + low pass; inflated (1e-4 relative + 1e-3 px)
  // to cover rounding of the float64 power.  Pixel px is inside when its
  // centre px + 0.5 lies in [mx - hx, mx + hx].
  const double L = -(double)lthr;
  short4 box = make_short4(32000, -1, 32000, -1);  // empty: never intersects
  if (L > 0.0) {
    // float32 square roots (relative error ~1e-7, inside the 1e-4 inflation)
    const double hx = (double)sqrtf((float)(2.0 * L * po.a)) * (1.0 + 1e-4) + 1e-3;
    const double hy = (double)sqrtf((float)(2.0 * L * po.c)) * (1.0 + 1e-4) + 1e-3;
    const double lim = 32000.0;
    box.x = (int16_t)fmin(fmax(ceil(po.mx - hx - 0.5), -1.0), lim);
    box.y = (int16_t)fmin(fmax(floor(po.mx + hx - 0.5), -1.0), lim);
    box.z = (int16_t)fmin(fmax(ceil(po.my - hy - 0.5), -1.0), lim);
    box.w = (int16_t)fmin(fmax(floor(po.my + hy - 0.5), -1.0), lim);
  }
  po_out.hot[idx] = h;
  if (po_out.fast) {
    bool exact;
    const FastRec f = make_fast_rec(po.mx, po.my, c0, c1, c2, g.op, ln_o, lthr, h.r, h.g, h.b, po.a, po.c,
                                    po_out.log2_afl, exact);
    po_out.fast[idx] = f;
    if (exact && po_out.mark_exact) box.x = (int16_t)kBoxExact;
  }
  po_out.boxes[idx] = box;
  // tile rectangle exactly as numpy (render.py:226-231): floor, astype(int64), clip
  {
    const int64_t ntx = (cam.width + st.tile_size - 1) / st.tile_size;
    const int64_t nty = (cam.height + st.tile_size - 1) / st.tile_size;
    const double ts = (double)st.tile_size;
    // x / ts for a power-of-two tile size is x * (1 / ts) exactly (both are
    // the correctly rounded x * 2^-k), so the division becomes a multiply
    const bool pow2 = (st.tile_size & (st.tile_size - 1)) == 0;
    const double its = pow2 ? __longlong_as_double((long long)(1024 - __ffs(st.tile_size)) << 52) : 0.0;
    auto div_ts = [&](double x) { return pow2 ? dmul(x, its) : ddiv(x, ts); };
    const int64_t tx0 = clip_i64(np_to_i64(floor(div_ts(dsub(dsub(po.mx, po.rx), 0.5)))), 0, ntx - 1);
    const int64_t tx1 = clip_i64(np_to_i64(floor(div_ts(dsub(dadd(po.mx, po.rx), 0.5)))), 0, ntx - 1);
    const int64_t ty0 = clip_i64(np_to_i64(floor(div_ts(dsub(dsub(po.my, po.ry), 0.5)))), 0, nty - 1);
    const int64_t ty1 = clip_i64(np_to_i64(floor(div_ts(dsub(dadd(po.my, po.ry), 0.5)))), 0, nty - 1);
    po_out.rects[idx] = pack_rect((int)tx0, (int)tx1, (int)ty0, (int)ty1);
  }
  if (po_out.recs) {  // debug / dump mode: the full _Projected record (render.py:89-108)
    ProjRec rec;
    rec.mx = po.mx; rec.my = po.my; rec.c0 = c0; rec.c1 = c1; rec.c2 = c2;
    rec.a = po.a; rec.b = po.b; rec.c = po.c; rec.rx = po.rx; rec.ry = po.ry;
    rec.opacity = g.op; rec.depth = po.z;
    rec.r = (float)col[0]; rec.g = (float)col[1]; rec.bl = (float)col[2]; rec.pad = 0;
    rec.src = i; rec.pad2 = 0;
    po_out.recs[idx] = rec;
  }
}


#ifndef CS_PROJ_THREADS
#define CS_PROJ_THREADS 256
#endif
#ifndef CS_PROJ_MINB
#define CS_PROJ_MINB 3
#endif
constexpr int kProjThreads = CS_PROJ_THREADS;
#ifndef CS_PROJ_STAGED
#define CS_PROJ_STAGED 1   // 0: one thread per Gaussian with direct global loads (A/B reference)
#endif

// Projection, one thread per assembled Gaussian, no compaction: every
// per-splat output is written at the Gaussian's assembled index i (its
// "splat id"), and a culled Gaussian gets the depth key ~0, which the stable
// depth sort (K4) moves behind every visible one.  So the sort's first M
// values are the visible splat ids in (depth, assembled index) order, and the
// kernel needs no block scan or cross-CTA look-back (LoD assembly already
// drops invisible blocks: ~97% of the assembled set is visible on C3).
__global__ void __launch_bounds__(kProjThreads, CS_PROJ_MINB)
k_project(const cs_cloud* __restrict__ clouds, const Seg* __restrict__ segs,
          DevStats* __restrict__ stats, cs_camera cam, cs_settings st,
          ProjOutputs po_out, const uint64_t* __restrict__ list) {
  const int64_t n = stats->assembled;
  const int64_t i = blockIdx.x * (int64_t)kProjThreads + threadIdx.x;
  const int64_t cta0 = blockIdx.x * (int64_t)kProjThreads;
  if (cta0 >= n) return;  // CTA-uniform
  // segment starts staged in shared memory (one coalesced load; n_segs <= L*J
  // is small), so the per-thread search costs no dependent global loads
  constexpr int kSmemSegs = 512;
  __shared__ int64_t s_start[kSmemSegs];
  const int n_segs = stats->n_segs;
  const bool smem_segs = n_segs <= kSmemSegs;
  if (smem_segs)
    for (int q = threadIdx.x; q < n_segs; q += kProjThreads) s_start[q] = segs[q].start;
  __syncthreads();
  ProjOut po;
  po.in_front = po.ok = po.keep = false;
  Geom g;
  int64_t local = 0;
  int cloud_id = 0;
  if (i < n) {
    int si = 0;
    if (smem_segs) {
      int hi = n_segs - 1;
      while (si < hi) {
        const int mid = (si + hi + 1) >> 1;
        if (s_start[mid] <= i) si = mid; else hi = mid - 1;
      }
    } else {
      si = find_seg(segs, n_segs, i);
    }
    const Seg sg = segs[si];
    cloud_id = sg.cloud;
    local = i - sg.start;
    if (cloud_id < 0) {  // pointwise list mode: packed (cloud << 40 | local)
      const uint64_t e = list[i];
      cloud_id = (int)(e >> 40);
      local = (int64_t)(e & ((1ull << 40) - 1));
    }
    g = load_geom(clouds[cloud_id], local);
    po = project_one(g, cam, st);
    // a row of the "rest" cloud of assign_b1 (partition.py:332-333): rendering
    // the full cloud with the excluded rows culled equals rendering
    // cloud.take(~mask) -- the kept rows keep their relative (index) order
    if (po_out.exclude && po_out.exclude[i]) po.in_front = po.ok = po.keep = false;
  }
  // skipped_singular: in front but det <= 1e-12 (render.py:146-148)
  const uint32_t kb = __ballot_sync(0xffffffffu, po.keep);
  const uint32_t sb = __ballot_sync(0xffffffffu, po.in_front && !po.ok);
  if (lane_id() == 0) {
    if (kb) atomicAdd(reinterpret_cast<unsigned long long*>(&stats->visible), (unsigned long long)__popc(kb));
    if (sb) atomicAdd(reinterpret_cast<unsigned long long*>(&stats->skipped), (unsigned long long)__popc(sb));
  }
  if (i >= n) return;
  const cs_cloud& cd = clouds[cloud_id];
  project_emit<false>(i, g, po, cd.sh + local * cd.sh_stride, cd.sh_coeffs, cam, st, po_out);
}

// K3, staged form (every source except the pointwise list): persistent CTAs
// walk 256-Gaussian tiles of the assembled index range.  A tile's inputs are
// contiguous runs of the level clouds (one run per (level, block) segment it
// touches), so thread 0 moves them into shared memory with cp.async.bulk
// copies completing on mbarriers -- the three float32 geometry quads per
// Gaussian double-buffered (tile t+1's copies are issued before tile t is
// computed), the SH rows single-buffered (tile t+1's issued once tile t's
// colours are done, landing while t+1's float64 projection math runs).  The
// global-load latency that stalled the one-thread-per-Gaussian kernel
// (long scoreboard, 34% of its stall samples at 35% occupancy) moves off
// the critical path.  Runs that cannot be staged (float64 quads, SH rows
// wider than 48 floats, more than kMaxPieces segments in a tile) fall back to
// per-thread global loads for those rows.
constexpr int kStPieces = 8;
constexpr int kStShFloats = 48;  // widest staged SH row (C = 16)

struct StPiece {
  int32_t row0, rows;      // tile-relative first row, row count
  int32_t cloud;           // descriptor index
  int32_t staged;          // 1: quads + SH in shared memory
  int64_t local0;          // first row inside the cloud
  int32_t sh_off;          // float offset of the piece's SH rows in s_sh
  int32_t pad;
};

__global__ void __launch_bounds__(kProjThreads, CS_PROJ_MINB)
k_project_staged(const cs_cloud* __restrict__ clouds, const Seg* __restrict__ segs,
                 DevStats* __restrict__ stats, cs_camera cam, cs_settings st,
                 ProjOutputs po_out, const uint64_t* __restrict__ list) {
  (void)list;
  // dynamic shared memory: geometry quads [2][3][kProjThreads] (pos_op, scale,
  // quat), then the SH rows of one tile (kProjThreads x kStShFloats floats)
  extern __shared__ __align__(128) unsigned char s_dyn[];
  float4 (*s_q)[3][kProjThreads] = reinterpret_cast<float4 (*)[3][kProjThreads]>(s_dyn);
  float* s_sh = reinterpret_cast<float*>(s_dyn + sizeof(float4) * 2 * 3 * kProjThreads);
  __shared__ __align__(8) uint64_t s_bar[3];                   // quads[0], quads[1], sh
  __shared__ StPiece s_pc[2][kStPieces];                       // per quad buffer
  __shared__ int s_npc[2];
  __shared__ int64_t s_start[256];
  const int64_t n = stats->assembled;
  const int n_segs = stats->n_segs;
  const bool smem_segs = n_segs <= 256;
  if (smem_segs)
    for (int q = threadIdx.x; q < n_segs; q += kProjThreads) s_start[q] = segs[q].start;
  if (threadIdx.x == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_init(&s_bar[2], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t n_tiles = (n + kProjThreads - 1) / kProjThreads;
  auto seg_of = [&](int64_t i) -> int {
    if (!smem_segs) return find_seg(segs, n_segs, i);
    int lo = 0, hi = n_segs - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_start[mid] <= i) lo = mid; else hi = mid - 1;
    }
    return lo;
  };
  // thread 0: the tile's pieces, and the bulk copies of their quads into buffer b
  auto issue_quads = [&](int64_t tile, int b) {
    const int64_t i0 = tile * kProjThreads, i1 = min(n, i0 + kProjThreads);
    int np = 0;
    uint32_t bytes = 0;
    int sh_off = 0;
    for (int si = seg_of(i0); si < n_segs && np < kStPieces; ++si) {
      const Seg sg = segs[si];
      const int64_t a = max(i0, sg.start), e = min(i1, sg.start + sg.count);
      if (a >= e) { if (sg.start >= i1) break; continue; }
      StPiece p;
      p.row0 = (int32_t)(a - i0);
      p.rows = (int32_t)(e - a);
      p.cloud = sg.cloud;
      p.local0 = a - sg.start;
      const cs_cloud& cd = clouds[sg.cloud];
      p.staged = (!cd.fp64 && cd.sh_stride <= kStShFloats) ? 1 : 0;
      p.sh_off = sh_off;   // fixed here: threads read it before issue_sh runs
      p.pad = 0;
      if (p.staged) sh_off += p.rows * cd.sh_stride;
      if (p.staged) {
        const uint32_t qb = (uint32_t)p.rows * 16u;
        const int64_t off = p.local0 * 16;
        bulk_copy_g2s(&s_q[b][0][p.row0], reinterpret_cast<const char*>(cd.pos_op) + off, qb, &s_bar[b]);
        bulk_copy_g2s(&s_q[b][1][p.row0], reinterpret_cast<const char*>(cd.scale) + off, qb, &s_bar[b]);
        bulk_copy_g2s(&s_q[b][2][p.row0], reinterpret_cast<const char*>(cd.quat) + off, qb, &s_bar[b]);
        bytes += 3 * qb;
      }
      s_pc[b][np++] = p;
      if (e >= i1) break;
    }
    s_npc[b] = np;
    mbar_arrive_expect_tx(&s_bar[b], bytes);
  };
  // thread 0: SH rows of the pieces in quad buffer b (after their pieces are known)
  auto issue_sh = [&](int b) {
    uint32_t bytes = 0;
    for (int k = 0; k < s_npc[b]; ++k) {
      const StPiece& p = s_pc[b][k];
      if (!p.staged) continue;
      const cs_cloud& cd = clouds[p.cloud];
      const uint32_t sb = (uint32_t)p.rows * (uint32_t)cd.sh_stride * 4u;
      bulk_copy_g2s(&s_sh[p.sh_off], cd.sh + p.local0 * cd.sh_stride, sb, &s_bar[2]);
      bytes += sb;
    }
    mbar_arrive_expect_tx(&s_bar[2], bytes);
  };
  uint32_t ph_q0 = 0, ph_q1 = 0, ph_sh = 0;
  int64_t tile = blockIdx.x;
  if (tile < n_tiles && threadIdx.x == 0) {
    issue_quads(tile, 0);
    issue_sh(0);
  }
  for (int it = 0; tile < n_tiles; ++it, tile += gridDim.x) {
    const int b = it & 1;
    const int64_t next = tile + gridDim.x;
    if (next < n_tiles && threadIdx.x == 0) issue_quads(next, b ^ 1);
    mbar_wait(&s_bar[b], b ? ph_q1 : ph_q0);
    if (b) ph_q1 ^= 1u; else ph_q0 ^= 1u;
    const int64_t i = tile * kProjThreads + threadIdx.x;
    const int r = (int)threadIdx.x;
    int pk = 0;
    const int np = s_npc[b];
    while (pk + 1 < np && s_pc[b][pk + 1].row0 <= r) ++pk;
    StPiece p = s_pc[b][pk];
    const bool live = i < n;
    if (live && r >= p.row0 + p.rows) {  // a row past the staged pieces: its own segment, global loads
      const int si = seg_of(i);
      const Seg sg = segs[si];
      p.row0 = r;
      p.rows = 1;
      p.cloud = sg.cloud;
      p.local0 = i - sg.start;
      p.staged = 0;
    }
    const int64_t local = p.local0 + (r - p.row0);
    ProjOut po;
    po.in_front = po.ok = po.keep = false;
    Geom g;
    if (live) {
      if (p.staged) {
        const float4 a = s_q[b][0][r], c = s_q[b][1][r], q = s_q[b][2][r];
        g.px = a.x; g.py = a.y; g.pz = a.z; g.op = a.w;
        g.sx = c.x; g.sy = c.y; g.sz = c.z;
        g.qw = q.x; g.qx = q.y; g.qy = q.z; g.qz = q.w;
      } else {
        g = load_geom(clouds[p.cloud], local);
      }
      po = project_one(g, cam, st);
      if (po_out.exclude && po_out.exclude[i]) po.in_front = po.ok = po.keep = false;
    }
    const uint32_t kb = __ballot_sync(0xffffffffu, po.keep);
    const uint32_t sb = __ballot_sync(0xffffffffu, po.in_front && !po.ok);
    if (lane_id() == 0) {
      if (kb) atomicAdd(reinterpret_cast<unsigned long long*>(&stats->visible), (unsigned long long)__popc(kb));
      if (sb) atomicAdd(reinterpret_cast<unsigned long long*>(&stats->skipped), (unsigned long long)__popc(sb));
    }
    mbar_wait(&s_bar[2], ph_sh);   // this tile's SH rows
    ph_sh ^= 1u;
    if (live) {
      const cs_cloud& cd = clouds[p.cloud];
      if (p.staged)
        project_emit<true>(i, g, po, &s_sh[p.sh_off + (r - p.row0) * cd.sh_stride], cd.sh_coeffs, cam, st, po_out);
      else
        project_emit<false>(i, g, po, cd.sh + local * cd.sh_stride, cd.sh_coeffs, cam, st, po_out);
    }
    fence_proxy_async_smem();   // this tile's shared-memory reads before the next copies
    __syncthreads();
    if (next < n_tiles && threadIdx.x == 0) issue_sh(b ^ 1);
  }
}

// Single-cloud source: one segment covering the whole cloud.
__global__ void k_setup_cloud(cs_cloud c, cs_cloud* clouds, Seg* segs, DevStats* stats) {
  clouds[0] = c;
  segs[0].start = 0;
  segs[0].count = c.count;
  segs[0].cloud = 0;
  segs[0].pad = 0;
  stats->n_segs = 1;
  stats->assembled = c.count;
}

const void* project_kernel() { return reinterpret_cast<const void*>(&k_project); }
const void* project_staged_kernel() { return reinterpret_cast<const void*>(&k_project_staged); }

void launch_project(const cs_cloud* d_clouds, const Seg* d_segs, DevStats* d_stats,
                    const cs_camera& cam, const cs_settings& st, int64_t capacity,
                    const ProjOutputs& out, const uint64_t* list, cudaStream_t s) {
  const int64_t blocks = (capacity + kProjThreads - 1) / kProjThreads;
  if (blocks == 0) return;
  if (!list && CS_PROJ_STAGED) {  // persistent, bulk-copy staged inputs
    constexpr size_t kDyn = sizeof(float4) * 2 * 3 * kProjThreads + sizeof(float) * kProjThreads * kStShFloats;
    static int grid = 0;
    if (grid == 0) {
      cudaFuncSetAttribute(k_project_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDyn);
      int dev = 0, sms = 0, per_sm = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_project_staged, kProjThreads, kDyn);
      grid = std::max(1, sms * std::max(1, per_sm));
    }
    k_project_staged<<<(unsigned)std::min<int64_t>(grid, blocks), kProjThreads, kDyn, s>>>(
        d_clouds, d_segs, d_stats, cam, st, out, list);
    return;
  }
  k_project<<<(unsigned)blocks, kProjThreads, 0, s>>>(d_clouds, d_segs, d_stats, cam, st, out, list);
}

void launch_setup_cloud(const cs_cloud& c, cs_cloud* d_clouds, Seg* d_segs, DevStats* d_stats,
                        cudaStream_t s) {
  k_setup_cloud<<<1, 1, 0, s>>>(c, d_clouds, d_segs, d_stats);
}

// ---------------------------------------------------------------------------
// core.py utilities on device (API mirror: build_covariances, sh_to_colors)

__global__ void k_build_covariances(int64_t n, const double* scales, const double* quats,
                                    double* out) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  Geom g;
  g.sx = scales[3 * k]; g.sy = scales[3 * k + 1]; g.sz = scales[3 * k + 2];
  g.qw = quats[4 * k]; g.qx = quats[4 * k + 1]; g.qy = quats[4 * k + 2]; g.qz = quats[4 * k + 3];
  const double w = g.qw, x = g.qx, y = g.qy, q = g.qz;
  double r[9];
  r[0] = dsub(1.0, dmul(2.0, dadd(dmul(y, y), dmul(q, q))));
  r[1] = dmul(2.0, dsub(dmul(x, y), dmul(w, q)));
  r[2] = dmul(2.0, dadd(dmul(x, q), dmul(w, y)));
  r[3] = dmul(2.0, dadd(dmul(x, y), dmul(w, q)));
  r[4] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(q, q))));
  r[5] = dmul(2.0, dsub(dmul(y, q), dmul(w, x)));
  r[6] = dmul(2.0, dsub(dmul(x, q), dmul(w, y)));
  r[7] = dmul(2.0, dadd(dmul(y, q), dmul(w, x)));
  r[8] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(y, y))));
  const double s2[3] = {dmul(g.sx, g.sx), dmul(g.sy, g.sy), dmul(g.sz, g.sz)};
  for (int i = 0; i < 3; ++i)
    for (int l = 0; l < 3; ++l)
      out[9 * k + 3 * i + l] =
          dadd(dadd(dmul(dmul(r[3 * i + 0], s2[0]), r[3 * l + 0]),
                    dmul(dmul(r[3 * i + 2], s2[2]), r[3 * l + 2])),
               dmul(dmul(r[3 * i + 1], s2[1]), r[3 * l + 1]));
}

__global__ void k_sh_to_colors(int64_t n, const double* sh, int C, const double* dirs, int degree,
                               double* out) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double x = dirs[3 * k], y = dirs[3 * k + 1], z = dirs[3 * k + 2];
  double basis[16];
  basis[0] = kShC0;
  if (degree >= 1) { basis[1] = -kShC1 * y; basis[2] = kShC1 * z; basis[3] = -kShC1 * x; }
  if (degree >= 2) {
    double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    basis[4] = kShC2[0] * xy; basis[5] = kShC2[1] * yz;
    basis[6] = kShC2[2] * (2.0 * zz - xx - yy); basis[7] = kShC2[3] * xz;
    basis[8] = kShC2[4] * (xx - yy);
    if (degree >= 3) {
      basis[9] = kShC3[0] * y * (3.0 * xx - yy);
      basis[10] = kShC3[1] * xy * z;
      basis[11] = kShC3[2] * y * (4.0 * zz - xx - yy);
      basis[12] = kShC3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
      basis[13] = kShC3[4] * x * (4.0 * zz - xx - yy);
      basis[14] = kShC3[5] * z * (xx - yy);
      basis[15] = kShC3[6] * x * (xx - 3.0 * yy);
    }
  }
  const int nb = (degree + 1) * (degree + 1);
  for (int ch = 0; ch < 3; ++ch) {
    double acc = 0.0;
    for (int m = 0; m < nb; ++m) acc += sh[(k * 3 + ch) * C + m] * basis[m];
    double v = 0.5 + acc;
    out[3 * k + ch] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
  }
}

void launch_build_covariances(int64_t n, const double* scales, const double* quats, double* out,
                              cudaStream_t s) {
  if (n <= 0) return;
  k_build_covariances<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, scales, quats, out);
}
void launch_sh_to_colors(int64_t n, const double* sh, int C, const double* dirs, int degree,
                         double* out, cudaStream_t s) {
  if (n <= 0) return;
  k_sh_to_colors<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, sh, C, dirs, degree, out);
}

}  // namespace cs

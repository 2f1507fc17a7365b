/*
 * cs_oracle.c -- CPU restatement of the citysplat rendering hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity *checker* for the CUDA
 * product in paper_2404_01133_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path never links, loads or calls anything under oracle/.
 *
 * Every function restates one reference function in the exact floating-point
 * operation order numpy / numba use (no FMA: build with -ffp-contract=off), so
 * that decision quantities (visible set, depth order, tile lists, LoD levels)
 * are bit-identical to the reference run under OPENBLAS_CORETYPE=Sandybridge
 * (SURVEY.md Appendix B).  Parity of this restatement is pinned against the
 * golden vectors in tests/golden/ produced by the reference itself
 * (tests/golden/make_golden.py).
 *
 * Reference files cited below live under /root/reference/pkg/src/citysplat/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  double R[9];      /* rotation_w2c, row-major */
  double t[3];      /* translation_w2c */
  double center[3]; /* camera_center = -R^T t as computed by the reference */
  double fx, fy, cx, cy;
  int64_t width, height;
} or_camera;

typedef struct {
  double background[3];
  double alpha_floor;
  double transmittance_floor;
  double near_plane;
  double support_sigmas; /* math.sqrt(2 ln(1/alpha_floor)), render.py:61-64 */
  double low_pass;       /* LOW_PASS = 0.3, render.py:33 */
  double singular_det;   /* _SINGULAR_DET = 1e-12, render.py:34 */
  int64_t sh_degree;
  int64_t tile_size;
} or_settings;

/* SH constants, core.py:35-52 */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

static inline double ld(const void* p, int f32, int64_t i) {
  return f32 ? (double)((const float*)p)[i] : ((const double*)p)[i];
}

/* numpy float64 -> int64 cast of an out-of-range value yields INT64_MIN on
 * x86 (cvttsd2si "integer indefinite"); np.clip then maps it to the low end.
 * render.py:228-231 relies on astype(np.int64) before clip. */
static inline int64_t np_to_i64(double x) {
  if (!(x >= -9223372036854775808.0 && x < 9223372036854775808.0)) return INT64_MIN;
  return (int64_t)x;
}
static inline int64_t clip_i64(int64_t v, int64_t lo, int64_t hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

/* eval_sh_basis, core.py:114-146 (band-major, same expression order). */
static void sh_basis(double x, double y, double z, int degree, double* out) {
  out[0] = SH_C0;
  if (degree >= 1) {
    out[1] = -SH_C1 * y;
    out[2] = SH_C1 * z;
    out[3] = -SH_C1 * x;
  }
  if (degree >= 2) {
    double xx = x * x, yy = y * y, zz = z * z;
    double xy = x * y, yz = y * z, xz = x * z;
    out[4] = SH_C2[0] * xy;
    out[5] = SH_C2[1] * yz;
    out[6] = SH_C2[2] * (2.0 * zz - xx - yy);
    out[7] = SH_C2[3] * xz;
    out[8] = SH_C2[4] * (xx - yy);
    if (degree >= 3) {
      out[9] = SH_C3[0] * y * (3.0 * xx - yy);
      out[10] = SH_C3[1] * xy * z;
      out[11] = SH_C3[2] * y * (4.0 * zz - xx - yy);
      out[12] = SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
      out[13] = SH_C3[4] * x * (4.0 * zz - xx - yy);
      out[14] = SH_C3[5] * z * (xx - yy);
      out[15] = SH_C3[6] * x * (xx - 3.0 * yy);
    }
  }
}

static int degree_of(int64_t c) { return c >= 16 ? 3 : c >= 9 ? 2 : c >= 4 ? 1 : 0; }

/*
 * _project_cloud, render.py:111-188, before the depth sort (render.py:176-177).
 * Outputs are written in ascending source order (the np.nonzero order of
 * render.py:121 / render.py:163); returns the visible count.  All geometric
 * math is float64 with numpy's elementwise order:
 *   t = P @ R^T + T          (dgemm under the Sandybridge pin: no FMA)   render.py:118
 *   Sigma = R diag(s^2) R^T  (einsum kij,klj->kil; numpy's 2-lane contiguous
 *                            sum-of-products adds terms as (t0 + t2) + t1)   core.py:107-111
 *   V = W Sigma W^T          (einsum ij,kjl,ml->kim, j-major l-minor)     render.py:133
 *   cov2d = J V J^T          (same 9-term order incl. zero terms)         render.py:141
 */
int64_t or_project(int64_t K, const void* pos, const void* opac, const void* scl,
                   const void* rot, int geom_f32, const void* sh, int sh_f32, int64_t C,
                   const or_camera* cam, const or_settings* st, double* means, double* conics,
                   double* covs, double* depths, double* colors, double* opacities,
                   double* radii, int64_t* source, int64_t* skipped_out, int nthreads) {
  const double* R = cam->R;
  const double* T = cam->t;
  int degree = (int)st->sh_degree;
  int sdeg = degree_of(C);
  if (sdeg < degree) degree = sdeg;
  int nb = (degree + 1) * (degree + 1);
  int64_t skipped = 0;
  uint8_t* keep = (uint8_t*)malloc((size_t)(K > 0 ? K : 1));
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  /* pass 1: cull decision (embarrassingly parallel) */
#pragma omp parallel for reduction(+ : skipped) schedule(static)
  for (int64_t k = 0; k < K; ++k) {
    double p0 = ld(pos, geom_f32, 3 * k), p1 = ld(pos, geom_f32, 3 * k + 1),
           p2 = ld(pos, geom_f32, 3 * k + 2);
    double t0 = ((p0 * R[0] + p1 * R[1]) + p2 * R[2]) + T[0];
    double t1 = ((p0 * R[3] + p1 * R[4]) + p2 * R[5]) + T[1];
    double z = ((p0 * R[6] + p1 * R[7]) + p2 * R[8]) + T[2];
    keep[k] = 0;
    if (!(z > st->near_plane)) continue; /* render.py:120 */
    double mx = cam->fx * t0 / z + cam->cx; /* render.py:128-129 */
    double my = cam->fy * t1 / z + cam->cy;
    /* quat_to_rotmat, core.py:74-82 */
    double w = ld(rot, geom_f32, 4 * k), x = ld(rot, geom_f32, 4 * k + 1),
           y = ld(rot, geom_f32, 4 * k + 2), zq = ld(rot, geom_f32, 4 * k + 3);
    double r[9];
    r[0] = 1.0 - 2.0 * (y * y + zq * zq);
    r[1] = 2.0 * (x * y - w * zq);
    r[2] = 2.0 * (x * zq + w * y);
    r[3] = 2.0 * (x * y + w * zq);
    r[4] = 1.0 - 2.0 * (x * x + zq * zq);
    r[5] = 2.0 * (y * zq - w * x);
    r[6] = 2.0 * (x * zq - w * y);
    r[7] = 2.0 * (y * zq + w * x);
    r[8] = 1.0 - 2.0 * (x * x + y * y);
    double s0 = ld(scl, geom_f32, 3 * k), s1 = ld(scl, geom_f32, 3 * k + 1),
           s2 = ld(scl, geom_f32, 3 * k + 2);
    double q0 = s0 * s0, q1 = s1 * s1, q2 = s2 * s2;
    double rs[9];
    for (int i = 0; i < 3; ++i) {
      rs[3 * i + 0] = r[3 * i + 0] * q0;
      rs[3 * i + 1] = r[3 * i + 1] * q1;
      rs[3 * i + 2] = r[3 * i + 2] * q2;
    }
    double sig[9];
    for (int i = 0; i < 3; ++i)
      for (int l = 0; l < 3; ++l)
        sig[3 * i + l] = (rs[3 * i + 0] * r[3 * l + 0] + rs[3 * i + 2] * r[3 * l + 2]) +
                         rs[3 * i + 1] * r[3 * l + 1];
    double V[9];
    for (int i = 0; i < 3; ++i)
      for (int m = 0; m < 3; ++m) {
        double acc = 0.0;
        int first = 1;
        for (int j = 0; j < 3; ++j)
          for (int l = 0; l < 3; ++l) {
            double term = (R[3 * i + j] * sig[3 * j + l]) * R[3 * m + l];
            if (first) { acc = term; first = 0; } else acc = acc + term;
          }
        V[3 * i + m] = acc;
      }
    double J[6] = {cam->fx / z, 0.0, -cam->fx * t0 / (z * z),
                   0.0, cam->fy / z, -cam->fy * t1 / (z * z)};
    double cv[4];
    for (int i = 0; i < 2; ++i)
      for (int m = 0; m < 2; ++m) {
        double acc = 0.0;
        int first = 1;
        for (int j = 0; j < 3; ++j)
          for (int l = 0; l < 3; ++l) {
            double term = (J[3 * i + j] * V[3 * j + l]) * J[3 * m + l];
            if (first) { acc = term; first = 0; } else acc = acc + term;
          }
        cv[2 * i + m] = acc;
      }
    double a = cv[0] + st->low_pass, b = cv[1], c = cv[3] + st->low_pass;
    double det = a * c - b * b;
    int ok = det > st->singular_det; /* render.py:146-148 */
    if (!ok) { skipped += 1; continue; }
    double rx = st->support_sigmas * sqrt(a), ry = st->support_sigmas * sqrt(c);
    int on_image = (mx + rx > 0.0) && (mx - rx < (double)cam->width) && (my + ry > 0.0) &&
                   (my - ry < (double)cam->height); /* render.py:156-160 */
    keep[k] = on_image ? 1 : 0;
  }
  /* pass 2: serial compaction in source order, recompute outputs */
  int64_t M = 0;
  for (int64_t k = 0; k < K; ++k)
    if (keep[k]) source[M++] = k;
#pragma omp parallel for schedule(static)
  for (int64_t o = 0; o < M; ++o) {
    int64_t k = source[o];
    double p0 = ld(pos, geom_f32, 3 * k), p1 = ld(pos, geom_f32, 3 * k + 1),
           p2 = ld(pos, geom_f32, 3 * k + 2);
    double t0 = ((p0 * R[0] + p1 * R[1]) + p2 * R[2]) + T[0];
    double t1 = ((p0 * R[3] + p1 * R[4]) + p2 * R[5]) + T[1];
    double z = ((p0 * R[6] + p1 * R[7]) + p2 * R[8]) + T[2];
    double mx = cam->fx * t0 / z + cam->cx;
    double my = cam->fy * t1 / z + cam->cy;
    double w = ld(rot, geom_f32, 4 * k), x = ld(rot, geom_f32, 4 * k + 1),
           y = ld(rot, geom_f32, 4 * k + 2), zq = ld(rot, geom_f32, 4 * k + 3);
    double r[9];
    r[0] = 1.0 - 2.0 * (y * y + zq * zq);
    r[1] = 2.0 * (x * y - w * zq);
    r[2] = 2.0 * (x * zq + w * y);
    r[3] = 2.0 * (x * y + w * zq);
    r[4] = 1.0 - 2.0 * (x * x + zq * zq);
    r[5] = 2.0 * (y * zq - w * x);
    r[6] = 2.0 * (x * zq - w * y);
    r[7] = 2.0 * (y * zq + w * x);
    r[8] = 1.0 - 2.0 * (x * x + y * y);
    double s0 = ld(scl, geom_f32, 3 * k), s1 = ld(scl, geom_f32, 3 * k + 1),
           s2 = ld(scl, geom_f32, 3 * k + 2);
    double q0 = s0 * s0, q1 = s1 * s1, q2 = s2 * s2;
    double rs[9];
    for (int i = 0; i < 3; ++i) {
      rs[3 * i + 0] = r[3 * i + 0] * q0;
      rs[3 * i + 1] = r[3 * i + 1] * q1;
      rs[3 * i + 2] = r[3 * i + 2] * q2;
    }
    double sig[9];
    for (int i = 0; i < 3; ++i)
      for (int l = 0; l < 3; ++l)
        sig[3 * i + l] = (rs[3 * i + 0] * r[3 * l + 0] + rs[3 * i + 2] * r[3 * l + 2]) +
                         rs[3 * i + 1] * r[3 * l + 1];
    double V[9];
    for (int i = 0; i < 3; ++i)
      for (int m = 0; m < 3; ++m) {
        double acc = 0.0;
        int first = 1;
        for (int j = 0; j < 3; ++j)
          for (int l = 0; l < 3; ++l) {
            double term = (R[3 * i + j] * sig[3 * j + l]) * R[3 * m + l];
            if (first) { acc = term; first = 0; } else acc = acc + term;
          }
        V[3 * i + m] = acc;
      }
    double J[6] = {cam->fx / z, 0.0, -cam->fx * t0 / (z * z),
                   0.0, cam->fy / z, -cam->fy * t1 / (z * z)};
    double cv[4];
    for (int i = 0; i < 2; ++i)
      for (int m = 0; m < 2; ++m) {
        double acc = 0.0;
        int first = 1;
        for (int j = 0; j < 3; ++j)
          for (int l = 0; l < 3; ++l) {
            double term = (J[3 * i + j] * V[3 * j + l]) * J[3 * m + l];
            if (first) { acc = term; first = 0; } else acc = acc + term;
          }
        cv[2 * i + m] = acc;
      }
    double a = cv[0] + st->low_pass, b = cv[1], c = cv[3] + st->low_pass;
    double det = a * c - b * b;
    means[2 * o] = mx;
    means[2 * o + 1] = my;
    conics[3 * o] = c / det; /* render.py:172 */
    conics[3 * o + 1] = -b / det;
    conics[3 * o + 2] = a / det;
    covs[3 * o] = a;
    covs[3 * o + 1] = b;
    covs[3 * o + 2] = c;
    depths[o] = z;
    radii[2 * o] = st->support_sigmas * sqrt(a);
    radii[2 * o + 1] = st->support_sigmas * sqrt(c);
    opacities[o] = ld(opac, geom_f32, k);
    /* view direction and SH colour, render.py:167-169 + core.py:166-172 */
    double dx = p0 - cam->center[0], dy = p1 - cam->center[1], dz = p2 - cam->center[2];
    double nrm = sqrt((dx * dx + dy * dy) + dz * dz);
    double basis[16];
    sh_basis(dx / nrm, dy / nrm, dz / nrm, degree, basis);
    for (int ch = 0; ch < 3; ++ch) {
      double acc = 0.0;
      for (int n = 0; n < nb; ++n) acc += ld(sh, sh_f32, (k * 3 + ch) * C + n) * basis[n];
      double v = 0.5 + acc;
      colors[3 * o + ch] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    }
  }
  free(keep);
  *skipped_out = skipped;
  return M;
}

/* Stable ascending argsort of positive float64 depths (np.argsort kind="stable",
 * render.py:176-177): LSD radix over the IEEE bit pattern, which is monotone
 * for non-negative doubles.  Ties keep input (= source) order. */
void or_depth_argsort(int64_t M, const double* depths, int64_t* order) {
  uint64_t* key = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(M > 0 ? M : 1));
  uint64_t* key2 = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(M > 0 ? M : 1));
  int64_t* idx2 = (int64_t*)malloc(sizeof(int64_t) * (size_t)(M > 0 ? M : 1));
  for (int64_t i = 0; i < M; ++i) {
    uint64_t b;
    memcpy(&b, &depths[i], 8);
    /* total order for IEEE doubles (handles negatives for generality) */
    key[i] = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    order[i] = i;
  }
  for (int pass = 0; pass < 8; ++pass) {
    int64_t cnt[257];
    memset(cnt, 0, sizeof(cnt));
    int sh = pass * 8;
    for (int64_t i = 0; i < M; ++i) cnt[((key[i] >> sh) & 255) + 1]++;
    if (cnt[1 + ((key[0] >> sh) & 255)] == M && M > 0) continue; /* constant digit */
    for (int d = 0; d < 256; ++d) cnt[d + 1] += cnt[d];
    for (int64_t i = 0; i < M; ++i) {
      int64_t p = cnt[(key[i] >> sh) & 255]++;
      key2[p] = key[i];
      idx2[p] = order[i];
    }
    memcpy(key, key2, sizeof(uint64_t) * (size_t)M);
    memcpy(order, idx2, sizeof(int64_t) * (size_t)M);
  }
  free(key);
  free(key2);
  free(idx2);
}

/* _bin_tiles rectangle + pair count, render.py:217-243.  rect = (tx0,tx1,ty0,ty1)
 * per splat (depth order).  Returns the pair total. */
int64_t or_tile_rects(int64_t M, const double* means, const double* radii, int64_t tile_size,
                      int64_t width, int64_t height, int64_t* rects) {
  int64_t ntx = (width + tile_size - 1) / tile_size;
  int64_t nty = (height + tile_size - 1) / tile_size;
  double ts = (double)tile_size;
  int64_t total = 0;
  for (int64_t s = 0; s < M; ++s) {
    double mx = means[2 * s], my = means[2 * s + 1];
    double rx = radii[2 * s], ry = radii[2 * s + 1];
    int64_t tx0 = clip_i64(np_to_i64(floor((mx - rx - 0.5) / ts)), 0, ntx - 1);
    int64_t tx1 = clip_i64(np_to_i64(floor((mx + rx - 0.5) / ts)), 0, ntx - 1);
    int64_t ty0 = clip_i64(np_to_i64(floor((my - ry - 0.5) / ts)), 0, nty - 1);
    int64_t ty1 = clip_i64(np_to_i64(floor((my + ry - 0.5) / ts)), 0, nty - 1);
    rects[4 * s] = tx0;
    rects[4 * s + 1] = tx1;
    rects[4 * s + 2] = ty0;
    rects[4 * s + 3] = ty1;
    total += (tx1 - tx0 + 1) * (ty1 - ty0 + 1);
  }
  return total;
}

/* Duplicate row-major over each rect (render.py:233-243) and stably group by
 * tile (render.py:245-248) with a counting sort, which is exactly the
 * np.argsort(kind="stable") + bincount/cumsum result. */
void or_bin_tiles(int64_t M, const int64_t* rects, int64_t width, int64_t tile_size,
                  int64_t n_tiles, int64_t* tile_ids, int64_t* offsets) {
  int64_t ntx = (width + tile_size - 1) / tile_size;
  memset(offsets, 0, sizeof(int64_t) * (size_t)(n_tiles + 1));
  for (int64_t s = 0; s < M; ++s)
    for (int64_t ty = rects[4 * s + 2]; ty <= rects[4 * s + 3]; ++ty)
      for (int64_t tx = rects[4 * s]; tx <= rects[4 * s + 1]; ++tx) offsets[ty * ntx + tx + 1]++;
  for (int64_t t = 0; t < n_tiles; ++t) offsets[t + 1] += offsets[t];
  int64_t* cursor = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_tiles > 0 ? n_tiles : 1));
  memcpy(cursor, offsets, sizeof(int64_t) * (size_t)n_tiles);
  for (int64_t s = 0; s < M; ++s)
    for (int64_t ty = rects[4 * s + 2]; ty <= rects[4 * s + 3]; ++ty)
      for (int64_t tx = rects[4 * s]; tx <= rects[4 * s + 1]; ++tx)
        tile_ids[cursor[ty * ntx + tx]++] = s;
  free(cursor);
}

/* _kernels.blend_tiles, _kernels.py:17-76, same loop nest and op order.
 * out (H,W,3) fully overwritten, fragments (T,) accepted counts.
 * Optional per-pixel outputs for the gradient oracle: final transmittance and
 * the list position one past the last accepted fragment. */
void or_blend_tiles(const int64_t* tile_ids, const int64_t* tile_offsets, int64_t n_tiles,
                    const double* means, const double* conics, const double* colors,
                    const double* opacities, const double* background, int64_t tile_size,
                    int64_t width, int64_t height, int64_t n_tiles_x, double alpha_floor,
                    double t_floor, double* out, int64_t* fragments, double* final_t,
                    int64_t* last_pos, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t t = 0; t < n_tiles; ++t) {
    int64_t tx = t % n_tiles_x, ty = t / n_tiles_x;
    int64_t x0 = tx * tile_size, y0 = ty * tile_size;
    int64_t x1 = x0 + tile_size < width ? x0 + tile_size : width;
    int64_t y1 = y0 + tile_size < height ? y0 + tile_size : height;
    int64_t s0 = tile_offsets[t], s1 = tile_offsets[t + 1];
    int64_t count = 0;
    for (int64_t py = y0; py < y1; ++py) {
      double sy = (double)py + 0.5;
      for (int64_t px = x0; px < x1; ++px) {
        double sx = (double)px + 0.5;
        double trans = 1.0, r = 0.0, g = 0.0, b = 0.0;
        int64_t last = s0;
        for (int64_t k = s0; k < s1; ++k) {
          int64_t s = tile_ids[k];
          double dx = sx - means[2 * s], dy = sy - means[2 * s + 1];
          double power = -0.5 * (conics[3 * s] * dx * dx + conics[3 * s + 2] * dy * dy) -
                         conics[3 * s + 1] * dx * dy;
          double alpha = opacities[s] * exp(power);
          if (alpha > 0.99) alpha = 0.99;
          if (alpha < alpha_floor) continue;
          double next_trans = trans * (1.0 - alpha);
          if (next_trans < t_floor) break;
          double w = trans * alpha;
          r += w * colors[3 * s];
          g += w * colors[3 * s + 1];
          b += w * colors[3 * s + 2];
          trans = next_trans;
          count += 1;
          last = k + 1;
        }
        int64_t o = (py * width + px) * 3;
        out[o] = r + trans * background[0];
        out[o + 1] = g + trans * background[1];
        out[o + 2] = b + trans * background[2];
        if (final_t) final_t[py * width + px] = trans;
        if (last_pos) last_pos[py * width + px] = last;
      }
    }
    fragments[t] = count;
  }
}

/* The accepted fragments of _kernels.blend_tiles (_kernels.py:46-72), per
 * pixel in blend order: the discrete decisions the gradient oracle
 * differentiates through (oracle/grad_oracle.py).  frag_splat == NULL: write
 * the per-pixel accepted count into pix_count.  Otherwise write each pixel's
 * accepted splat indices (into the depth-sorted arrays) at
 * frag_splat[frag_offsets[pixel] ...]. */
void or_blend_fragments(const int64_t* tile_ids, const int64_t* tile_offsets, int64_t n_tiles,
                        const double* means, const double* conics, const double* opacities,
                        int64_t tile_size, int64_t width, int64_t height, int64_t n_tiles_x,
                        double alpha_floor, double t_floor, int64_t* pix_count,
                        const int64_t* frag_offsets, int64_t* frag_splat, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t t = 0; t < n_tiles; ++t) {
    int64_t tx = t % n_tiles_x, ty = t / n_tiles_x;
    int64_t x0 = tx * tile_size, y0 = ty * tile_size;
    int64_t x1 = x0 + tile_size < width ? x0 + tile_size : width;
    int64_t y1 = y0 + tile_size < height ? y0 + tile_size : height;
    int64_t s0 = tile_offsets[t], s1 = tile_offsets[t + 1];
    for (int64_t py = y0; py < y1; ++py) {
      double sy = (double)py + 0.5;
      for (int64_t px = x0; px < x1; ++px) {
        double sx = (double)px + 0.5;
        double trans = 1.0;
        int64_t n = 0;
        const int64_t pix = py * width + px;
        for (int64_t k = s0; k < s1; ++k) {
          int64_t s = tile_ids[k];
          double dx = sx - means[2 * s], dy = sy - means[2 * s + 1];
          double power = -0.5 * (conics[3 * s] * dx * dx + conics[3 * s + 2] * dy * dy) -
                         conics[3 * s + 1] * dx * dy;
          double alpha = opacities[s] * exp(power);
          if (alpha > 0.99) alpha = 0.99;
          if (alpha < alpha_floor) continue;
          double next_trans = trans * (1.0 - alpha);
          if (next_trans < t_floor) break;
          if (frag_splat) frag_splat[frag_offsets[pix] + n] = s;
          ++n;
          trans = next_trans;
        }
        if (!frag_splat) pix_count[pix] = n;
      }
    }
  }
}

/* block_visible + select_level + decide_visibility + _screen_box,
 * lod.py:267-348.  Corner order x-major (lod.py:282-283); world_to_camera is
 * P @ R^T + t (core.py:376-377, no-FMA dgemm order under the pin); distance
 * is np.linalg.norm(...).min() (lod.py:284).
 * Returns 0, or -1 when no interval covers a visible block's distance
 * (select_level's ValueError, lod.py:321). level = -1 encodes None. */
int or_decide_visibility(int64_t n_blocks, const double* bmin, const double* bmax,
                         const uint8_t* occupied, int64_t n_int, const double* intervals,
                         const or_camera* cam, int64_t force_level, uint8_t* visible,
                         int64_t* level, double* distance, double* box, uint8_t* has_box) {
  const double* C = cam->center;
  for (int64_t j = 0; j < n_blocks; ++j) {
    visible[j] = 0;
    level[j] = -1;
    has_box[j] = 0;
    box[4 * j] = box[4 * j + 1] = box[4 * j + 2] = box[4 * j + 3] = 0.0;
    if (!occupied[j]) {
      distance[j] = INFINITY;
      continue;
    }
    const double* lo = bmin + 3 * j;
    const double* hi = bmax + 3 * j;
    int inside = 1;
    for (int a = 0; a < 3; ++a)
      if (!(C[a] >= lo[a] && C[a] <= hi[a])) inside = 0;
    int vis;
    double dist;
    double u[8], v[8], z[8];
    int any_behind = 0, all_behind = 1;
    for (int ci = 0; ci < 8; ++ci) {
      double px = (ci & 4) ? hi[0] : lo[0];
      double py = (ci & 2) ? hi[1] : lo[1];
      double pz = (ci & 1) ? hi[2] : lo[2];
      double t0 = ((px * cam->R[0] + py * cam->R[1]) + pz * cam->R[2]) + cam->t[0];
      double t1 = ((px * cam->R[3] + py * cam->R[4]) + pz * cam->R[5]) + cam->t[1];
      double t2 = ((px * cam->R[6] + py * cam->R[7]) + pz * cam->R[8]) + cam->t[2];
      z[ci] = t2;
      if (t2 <= 0.0) any_behind = 1; else all_behind = 0;
      u[ci] = cam->fx * t0 / t2 + cam->cx;
      v[ci] = cam->fy * t1 / t2 + cam->cy;
    }
    if (inside) {
      vis = 1;
      dist = 0.0;
    } else {
      dist = INFINITY;
      for (int ci = 0; ci < 8; ++ci) {
        double px = (ci & 4) ? hi[0] : lo[0];
        double py = (ci & 2) ? hi[1] : lo[1];
        double pz = (ci & 1) ? hi[2] : lo[2];
        double dx = px - C[0], dy = py - C[1], dz = pz - C[2];
        double d = sqrt((dx * dx + dy * dy) + dz * dz);
        if (d < dist) dist = d;
      }
      if (all_behind) vis = 0;
      else if (any_behind) vis = 1;
      else {
        double umin = u[0], umax = u[0], vmin = v[0], vmax = v[0];
        for (int ci = 1; ci < 8; ++ci) {
          if (u[ci] < umin) umin = u[ci];
          if (u[ci] > umax) umax = u[ci];
          if (v[ci] < vmin) vmin = v[ci];
          if (v[ci] > vmax) vmax = v[ci];
        }
        vis = (umax >= 0.0 && umin <= (double)cam->width && vmax >= 0.0 &&
               vmin <= (double)cam->height);
      }
    }
    distance[j] = dist;
    if (!vis) continue;
    visible[j] = 1;
    if (force_level >= 0) {
      level[j] = force_level;
    } else {
      int64_t lv = -1;
      for (int64_t i = 0; i < n_int; ++i)
        if (intervals[2 * i] <= dist && dist < intervals[2 * i + 1]) {
          lv = n_int - 1 - i;
          break;
        }
      if (lv < 0) return -1;
      level[j] = lv;
    }
    has_box[j] = 1;
    if (any_behind) {
      box[4 * j + 2] = (double)cam->width;
      box[4 * j + 3] = (double)cam->height;
    } else {
      double umin = u[0], umax = u[0], vmin = v[0], vmax = v[0];
      for (int ci = 1; ci < 8; ++ci) {
        if (u[ci] < umin) umin = u[ci];
        if (u[ci] > umax) umax = u[ci];
        if (v[ci] < vmin) vmin = v[ci];
        if (v[ci] > vmax) vmax = v[ci];
      }
      box[4 * j] = umin;
      box[4 * j + 1] = vmin;
      box[4 * j + 2] = umax;
      box[4 * j + 3] = vmax;
    }
  }
  return 0;
}

/* Pointwise ablation predicate, lod.py:378-390 + _select_levels lod.py:324-327:
 * keep[k] = (n-1 - (searchsorted(los, |p-C|, 'right') - 1)) == want. */
void or_pointwise_keep(int64_t K, const void* pos, int f32, const double* center, int64_t n_int,
                       const double* los, int64_t want, uint8_t* keep) {
  for (int64_t k = 0; k < K; ++k) {
    double dx = ld(pos, f32, 3 * k) - center[0];
    double dy = ld(pos, f32, 3 * k + 1) - center[1];
    double dz = ld(pos, f32, 3 * k + 2) - center[2];
    double d = sqrt((dx * dx + dy * dy) + dz * dz);
    int64_t i = 0;
    while (i < n_int && los[i] <= d) ++i; /* searchsorted side='right' */
    keep[k] = ((n_int - 1 - (i - 1)) == want) ? 1 : 0;
  }
}

/*
 * significance_scores hit counts, lod.py:54-101 (the per-view loop of
 * lod.py:71-95).  A view hits Gaussian k when its centre is in front of the
 * near plane (lod.py:74), projects inside [0, W] x [0, H] inclusive
 * (lod.py:81-83) and its support radius support_sigmas * sqrt(lambda_max of
 * cov2d + LOW_PASS) is >= MIN_FOOTPRINT_RADIUS = 0.5 px (lod.py:92-95).  The
 * covariance chain is the same numpy op order as _project_cloud (the einsums
 * of lod.py:85 / lod.py:91 are those of render.py:133 / render.py:141).
 * hits[k] counts views (the reference accumulates them in float64, exactly).
 */
void or_significance_hits(int64_t K, const void* pos, const void* scl, const void* rot,
                          int geom_f32, int64_t n_cams, const or_camera* cams,
                          const or_settings* st, int64_t* hits, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < K; ++k) {
    double p0 = ld(pos, geom_f32, 3 * k), p1 = ld(pos, geom_f32, 3 * k + 1),
           p2 = ld(pos, geom_f32, 3 * k + 2);
    double w = ld(rot, geom_f32, 4 * k), x = ld(rot, geom_f32, 4 * k + 1),
           y = ld(rot, geom_f32, 4 * k + 2), zq = ld(rot, geom_f32, 4 * k + 3);
    double r[9];
    r[0] = 1.0 - 2.0 * (y * y + zq * zq);
    r[1] = 2.0 * (x * y - w * zq);
    r[2] = 2.0 * (x * zq + w * y);
    r[3] = 2.0 * (x * y + w * zq);
    r[4] = 1.0 - 2.0 * (x * x + zq * zq);
    r[5] = 2.0 * (y * zq - w * x);
    r[6] = 2.0 * (x * zq - w * y);
    r[7] = 2.0 * (y * zq + w * x);
    r[8] = 1.0 - 2.0 * (x * x + y * y);
    double s0 = ld(scl, geom_f32, 3 * k), s1 = ld(scl, geom_f32, 3 * k + 1),
           s2 = ld(scl, geom_f32, 3 * k + 2);
    double q0 = s0 * s0, q1 = s1 * s1, q2 = s2 * s2;
    double rs[9], sig[9];
    for (int i = 0; i < 3; ++i) {
      rs[3 * i + 0] = r[3 * i + 0] * q0;
      rs[3 * i + 1] = r[3 * i + 1] * q1;
      rs[3 * i + 2] = r[3 * i + 2] * q2;
    }
    for (int i = 0; i < 3; ++i)
      for (int l = 0; l < 3; ++l)
        sig[3 * i + l] = (rs[3 * i + 0] * r[3 * l + 0] + rs[3 * i + 2] * r[3 * l + 2]) +
                         rs[3 * i + 1] * r[3 * l + 1];
    int64_t h = 0;
    for (int64_t ci = 0; ci < n_cams; ++ci) {
      const or_camera* cam = &cams[ci];
      const double* R = cam->R;
      const double* T = cam->t;
      double t0 = ((p0 * R[0] + p1 * R[1]) + p2 * R[2]) + T[0];
      double t1 = ((p0 * R[3] + p1 * R[4]) + p2 * R[5]) + T[1];
      double z = ((p0 * R[6] + p1 * R[7]) + p2 * R[8]) + T[2];
      if (!(z > st->near_plane)) continue;                 /* lod.py:74 */
      double u = cam->fx * t0 / z + cam->cx;                /* lod.py:79-80 */
      double v = cam->fy * t1 / z + cam->cy;
      int on_image = (u >= 0.0) && (u <= (double)cam->width) && (v >= 0.0) &&
                     (v <= (double)cam->height);            /* lod.py:81 */
      if (!on_image) continue;
      double V[9];
      for (int i = 0; i < 3; ++i)
        for (int m = 0; m < 3; ++m) {
          double acc = 0.0;
          int first = 1;
          for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l) {
              double term = (R[3 * i + j] * sig[3 * j + l]) * R[3 * m + l];
              if (first) { acc = term; first = 0; } else acc = acc + term;
            }
          V[3 * i + m] = acc;
        }
      double J[6] = {cam->fx / z, 0.0, -cam->fx * t0 / (z * z),
                     0.0, cam->fy / z, -cam->fy * t1 / (z * z)};
      double cv[4];
      for (int i = 0; i < 2; ++i)
        for (int m = 0; m < 2; ++m) {
          double acc = 0.0;
          int first = 1;
          for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l) {
              double term = (J[3 * i + j] * V[3 * j + l]) * J[3 * m + l];
              if (first) { acc = term; first = 0; } else acc = acc + term;
            }
          cv[2 * i + m] = acc;
        }
      double a = cv[0] + st->low_pass, b = cv[1], c = cv[3] + st->low_pass; /* lod.py:87-89 */
      double mid = 0.5 * (a + c);
      double disc = mid * mid - (a * c - b * b);
      double lam = mid + sqrt(disc > 0.0 ? disc : 0.0);    /* np.maximum(..., 0.0) */
      double radius = st->support_sigmas * sqrt(lam);
      if (radius >= 0.5) h += 1;                            /* MIN_FOOTPRINT_RADIUS */
    }
    hits[k] = h;
  }
}

/* normalize_position + contract + block_of_points, partition.py:110-169. */
void or_block_of_points(int64_t K, const void* pos, int f32, const double* pmin,
                        const double* pmax, int64_t nx, int64_t ny, int64_t nz, int64_t* out) {
  int64_t dims[3] = {nx, ny, nz};
  for (int64_t k = 0; k < K; ++k) {
    double ph[3], c[3];
    for (int a = 0; a < 3; ++a)
      ph[a] = 2.0 * (ld(pos, f32, 3 * k + a) - pmin[a]) / (pmax[a] - pmin[a]) - 1.0;
    double m = fabs(ph[0]);
    if (fabs(ph[1]) > m) m = fabs(ph[1]);
    if (fabs(ph[2]) > m) m = fabs(ph[2]);
    double safe = m > 1.0 ? m : 1.0;
    for (int a = 0; a < 3; ++a) c[a] = (m <= 1.0) ? ph[a] : (2.0 - 1.0 / safe) * ph[a] / safe;
    int64_t ib[3];
    for (int a = 0; a < 3; ++a) {
      ib[a] = clip_i64(np_to_i64(floor((c[a] + 2.0) / 4.0 * (double)dims[a])), 0, dims[a] - 1);
    }
    if (nz <= 1) ib[2] = 0;
    out[k] = ib[0] + nx * (ib[1] + ny * ib[2]);
  }
}

static double now_ms(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

/* Whole-frame CPU path (project -> depth sort -> bin -> blend) used for the
 * reported CPU baseline: rasterize_stats, render.py:252-280.  stage_ms gets
 * {project, sort, bin, blend}.  counts gets {visible, pairs, fragments, skipped}. */
int or_rasterize(int64_t K, const void* pos, const void* opac, const void* scl, const void* rot,
                 int geom_f32, const void* sh, int sh_f32, int64_t C, const or_camera* cam,
                 const or_settings* st, double* out, int64_t* counts, double* stage_ms,
                 int nthreads) {
  size_t k1 = (size_t)(K > 0 ? K : 1);
  double* means = malloc(sizeof(double) * 2 * k1);
  double* conics = malloc(sizeof(double) * 3 * k1);
  double* covs = malloc(sizeof(double) * 3 * k1);
  double* depths = malloc(sizeof(double) * k1);
  double* colors = malloc(sizeof(double) * 3 * k1);
  double* opac_o = malloc(sizeof(double) * k1);
  double* radii = malloc(sizeof(double) * 2 * k1);
  int64_t* source = malloc(sizeof(int64_t) * k1);
  int64_t skipped = 0;
  double t0 = now_ms();
  int64_t M = or_project(K, pos, opac, scl, rot, geom_f32, sh, sh_f32, C, cam, st, means, conics,
                         covs, depths, colors, opac_o, radii, source, &skipped, nthreads);
  double t1 = now_ms();
  int64_t* order = malloc(sizeof(int64_t) * (size_t)(M > 0 ? M : 1));
  or_depth_argsort(M, depths, order);
  size_t m1 = (size_t)(M > 0 ? M : 1);
  double* s_means = malloc(sizeof(double) * 2 * m1);
  double* s_conics = malloc(sizeof(double) * 3 * m1);
  double* s_colors = malloc(sizeof(double) * 3 * m1);
  double* s_opac = malloc(sizeof(double) * m1);
  double* s_radii = malloc(sizeof(double) * 2 * m1);
  for (int64_t i = 0; i < M; ++i) {
    int64_t s = order[i];
    s_means[2 * i] = means[2 * s];
    s_means[2 * i + 1] = means[2 * s + 1];
    s_radii[2 * i] = radii[2 * s];
    s_radii[2 * i + 1] = radii[2 * s + 1];
    for (int c = 0; c < 3; ++c) {
      s_conics[3 * i + c] = conics[3 * s + c];
      s_colors[3 * i + c] = colors[3 * s + c];
    }
    s_opac[i] = opac_o[s];
  }
  double t2 = now_ms();
  int64_t ts = st->tile_size;
  int64_t ntx = (cam->width + ts - 1) / ts, nty = (cam->height + ts - 1) / ts;
  int64_t n_tiles = ntx * nty;
  int64_t* rects = malloc(sizeof(int64_t) * 4 * m1);
  int64_t P = or_tile_rects(M, s_means, s_radii, ts, cam->width, cam->height, rects);
  int64_t* tile_ids = malloc(sizeof(int64_t) * (size_t)(P > 0 ? P : 1));
  int64_t* offsets = malloc(sizeof(int64_t) * (size_t)(n_tiles + 1));
  if (!tile_ids) return -2;
  or_bin_tiles(M, rects, cam->width, ts, n_tiles, tile_ids, offsets);
  double t3 = now_ms();
  int64_t* frags = malloc(sizeof(int64_t) * (size_t)n_tiles);
  or_blend_tiles(tile_ids, offsets, n_tiles, s_means, s_conics, s_colors, s_opac,
                 st->background, ts, cam->width, cam->height, ntx, st->alpha_floor,
                 st->transmittance_floor, out, frags, NULL, NULL, nthreads);
  double t4 = now_ms();
  int64_t F = 0;
  for (int64_t t = 0; t < n_tiles; ++t) F += frags[t];
  counts[0] = M;
  counts[1] = P;
  counts[2] = F;
  counts[3] = skipped;
  stage_ms[0] = t1 - t0;
  stage_ms[1] = t2 - t1;
  stage_ms[2] = t3 - t2;
  stage_ms[3] = t4 - t3;
  free(means); free(conics); free(covs); free(depths); free(colors); free(opac_o); free(radii);
  free(source); free(order); free(s_means); free(s_conics); free(s_colors); free(s_opac);
  free(s_radii); free(rects); free(tile_ids); free(offsets); free(frags);
  return 0;
}

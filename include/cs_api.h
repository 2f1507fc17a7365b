/*
 * cs_api.h -- C ABI of the B200-native CityGaussian rendering hot path.
 *
 * libcsgpu.so (built from paper_2404_01133_b200/csrc, sm_100a only) exports
 * exactly the functions declared here.  Signatures use plain pointers, sizes
 * and POD structs; no torch or CUDA types cross the boundary (streams are
 * passed as void* holding a cudaStream_t).  All device buffers passed in are
 * caller-owned; the context owns only its scratch workspace.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/citysplat/<file>:<line>).  INTEGRATION.md shows the
 * ctypes binding a citysplat maintainer would add.
 *
 * Return codes: 0 on success, negative on failure (CS_EINVAL, CS_ECUDA,
 * CS_ENOMEM, CS_ERANGE).  cs_last_error() returns a thread-local message.
 */
#ifndef CS_API_H
#define CS_API_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CS_OK 0
#define CS_EINVAL (-1)  /* -> ValueError (render.py:46-59, lod.py:314-321, lod.py:391-392) */
#define CS_ECUDA (-2)   /* -> RuntimeError */
#define CS_ENOMEM (-3)  /* -> MemoryError */
#define CS_ERANGE (-4)  /* select_level: no interval covers a distance (lod.py:321) */

/* Pinhole camera, core.py:339-377.  camera_center is passed as the reference
 * computes it (core.py:369-374) so LoD distances are bit-identical. */
typedef struct cs_camera {
  double R[9];      /* rotation_w2c, row-major */
  double t[3];      /* translation_w2c */
  double center[3]; /* camera_center */
  double fx, fy, cx, cy;
  int32_t width, height;
} cs_camera;

/* RenderSettings, render.py:37-64, plus the derived constants the reference
 * computes in Python (support_sigmas, LOW_PASS, _SINGULAR_DET) so the device
 * uses the identical float64 values. */
typedef struct cs_settings {
  double background[3];
  double alpha_floor;
  double transmittance_floor;
  double near_plane;
  double support_sigmas; /* sqrt(2 ln(1/alpha_floor)), render.py:61-64 */
  double low_pass;       /* 0.3, render.py:33 */
  double singular_det;   /* 1e-12, render.py:34 */
  int32_t sh_degree;
  int32_t tile_size;
} cs_settings;

/* One GaussianCloud (core.py:210-328) resident in HBM.  Geometry is stored
 * as 16-byte (fp32) or 32-byte (fp64) quads per Gaussian:
 *   pos_op = (x, y, z, opacity), scale = (sx, sy, sz, 0), quat = (w, x, y, z)
 * SH is fp32, channel-major (core.py:214-222): coefficient (c, n) of Gaussian
 * k at sh[k*sh_stride + c*sh_coeffs + n]; sh_stride >= 3*sh_coeffs, %4 == 0. */
typedef struct cs_cloud {
  const void* pos_op;
  const void* scale;
  const void* quat;
  const float* sh;
  int64_t count;
  int32_t sh_coeffs; /* 1, 4, 9 or 16 */
  int32_t sh_stride;
  int32_t fp64;      /* 1: geometry quads are double */
  int32_t reserved;
} cs_cloud;

/* Per-frame statistics (FrameStats, render.py:81-86, plus pipeline counts).
 * Written on the device by cs_render; read back only when asked. */
typedef struct cs_frame_stats {
  int64_t assembled;        /* AssembledSet.cloud.count (lod.py:395-401) */
  int64_t visible;          /* FrameStats.visible_splats */
  int64_t skipped_singular; /* FrameStats.skipped_singular */
  int64_t pairs;            /* tile pairs P (render.py:233-243) */
  int64_t fragments;        /* FrameStats.blended_fragments */
  int32_t n_segments;       /* (level, block) pieces concatenated */
  int32_t status;           /* bit0 pair-buffer overflow, bit1 CS_ERANGE */
  int64_t evals;            /* blend evaluations E (pixel x splat pairs walked; CS_RENDER_DIAG only) */
  int64_t warp_hits;        /* blend (8x4 pixel box, splat) pairs evaluated by a warp */
  int64_t warp_hits_empty;  /* ... of which no live pixel passed the alpha-floor test (CS_RENDER_DIAG only) */
  int64_t blend_max_item_cycles; /* longest blend work item (one pixel box), SM clocks (CS_RENDER_DIAG only) */
  int64_t blend_item_cycles;     /* sum over the blend's work items, SM clocks (CS_RENDER_DIAG only) */
  /* certified float32 blend (CS_RENDER_DIAG only): */
  int64_t blend_exact_hits;      /* (box, splat) hits of ill-conditioned splats decided in float64 */
  int64_t blend_floor_resolved;  /* fragments whose alpha-floor test fell inside the error bound (float64 re-decision) */
  int64_t blend_replays;         /* pixels whose termination test fell inside the error bound (float64 transmittance replay) */
} cs_frame_stats;

/* One block decision, VisibilityDecision (lod.py:255-264). level -1 = None. */
typedef struct cs_decision {
  double distance;
  double box[4];
  int32_t level;
  uint8_t visible;
  uint8_t has_box;
  uint8_t pad[2];
} cs_decision;

/* LodScene (lod.py:150-208) description for cs_lod_create.  All arrays are
 * host memory and are copied; cloud geometry stays where the caller put it. */
typedef struct cs_lod_desc {
  int32_t n_levels;
  int32_t n_blocks;
  const cs_cloud* clouds;     /* [n_levels * n_blocks], level-major (levels[L][j]) */
  const double* bounds_min;   /* [n_blocks * 3] world-space MAD bounds */
  const double* bounds_max;
  const double* intervals;    /* [n_levels * 2] (lo, hi), nearest-first */
} cs_lod_desc;

typedef struct cs_ctx cs_ctx;
typedef struct cs_lod cs_lod;

/* Frame sources */
#define CS_SRC_CLOUD 0     /* render one cloud: rasterize_stats(cloud, ...) */
#define CS_SRC_LOD_BLOCK 1 /* assemble_render_set(mode="block") then render */
#define CS_SRC_LOD_POINT 2 /* assemble_render_set(mode="pointwise") then render */

typedef struct cs_source {
  int32_t kind;
  int32_t force_level; /* -1 = None */
  cs_cloud cloud;      /* CS_SRC_CLOUD */
  const cs_lod* lod;   /* CS_SRC_LOD_* */
  /* CS_SRC_CLOUD only, optional (NULL): device uint8[cloud.count]; rows with a
   * nonzero byte are rendered as if absent -- the image of
   * cloud.take(nonzero(mask == 0)), the "rest" cloud of assign_b1
   * (partition.py:332-333), without materialising it */
  const uint8_t* exclude;
  /* CS_SRC_LOD_* only, optional (NULL = the render camera): the camera the LoD
   * selection runs for.  An AssembledSet (lod.py:351-401) is fixed by the
   * camera it was assembled for; rendering it from another camera must draw
   * that set, not re-select for the render camera. */
  const struct cs_camera* select_cam;
} cs_source;

/* cs_render flags */
#define CS_RENDER_SYNC 1u        /* synchronise, grow buffers and re-run on overflow */
#define CS_RENDER_F64_OUT 2u     /* out_rgb is double (compatibility tier) */
#define CS_RENDER_NO_CLIP 4u     /* leave the image unclipped */
#define CS_RENDER_KEEP_STATE 8u  /* internal: cs_render_train's kept state (cs_render rejects it) */
#define CS_RENDER_PROJECT_ONLY 16u /* stop after projection + depth order (cs_dump_projected) */
#define CS_RENDER_DEBUG 32u        /* also keep the full projected records (cs_dump_projected) */
#define CS_RENDER_DIAG 64u         /* also count evals and warp_hits_empty (blend diagnostics, slower) */

/* ---- context ----------------------------------------------------------- */
int cs_create(int device, cs_ctx** out);
void cs_destroy(cs_ctx* ctx);
const char* cs_last_error(void);
int cs_version(void);

/* ---- LoD scene (lod.py:150-208) ---------------------------------------- */
int cs_lod_create(cs_ctx* ctx, const cs_lod_desc* desc, cs_lod** out);
void cs_lod_destroy(cs_lod* lod);

/* decide_visibility (lod.py:330-348) incl. block_visible (lod.py:267-295),
 * _screen_box (lod.py:298-308) and select_level (lod.py:311-321).
 * out: host array [n_blocks].  Synchronous.  CS_ERANGE if select_level fails. */
int cs_decide_visibility(cs_ctx* ctx, const cs_lod* lod, const cs_camera* cam,
                         int32_t force_level, cs_decision* out_host, void* stream);

/* block_visible for n arbitrary boxes (lod.py:267-295); host in/out. */
int cs_block_visible(cs_ctx* ctx, int32_t n, const double* bmin, const double* bmax,
                     const cs_camera* cam, uint8_t* visible_out, double* distance_out,
                     void* stream);

/* select_level for n distances (lod.py:311-321); host in/out.
 * CS_EINVAL for a negative distance, CS_ERANGE if no interval covers one. */
int cs_select_level(cs_ctx* ctx, int32_t n, const double* distances, int32_t n_intervals,
                    const double* intervals, int32_t* level_out, void* stream);

/* ---- whole frame --------------------------------------------------------
 * rasterize_stats (render.py:252-280) of the source, with LoD selection +
 * assembly (lod.py:360-401) on device when src is a LoD source.
 * out_rgb: device (H, W, 3) float32 (or double with CS_RENDER_F64_OUT).
 * stats_host: optional; filled (after a sync) when non-NULL.
 * Without CS_RENDER_SYNC the call is fully asynchronous on `stream` and the
 * device-side stats can be read later with cs_frame_stats_get. */
int cs_render(cs_ctx* ctx, const cs_source* src, const cs_camera* cam, const cs_settings* st,
              void* out_rgb, uint32_t flags, cs_frame_stats* stats_host, void* stream);

/* Parameter gradients (device, float32, caller-allocated) for cs_render_backward,
 * laid out like the cloud's rows: positions (K,3), scales (K,3), rotations (K,4)
 * w.r.t. the raw (w,x,y,z) entering quat_to_rotmat, opacities (K) w.r.t. the
 * activated opacity, sh (K,3,C). */
typedef struct cs_grads {
  float* positions;
  float* scales;
  float* rotations;
  float* opacities;
  float* sh;
} cs_grads;

/* Training forward: rasterize_stats of one cloud (single-cloud source) that
 * keeps what its backward needs.  The frame's workspace (pair lists,
 * records, per-pixel transmittance / last fragment / colour) is handed to the
 * returned state, so other renders on the context -- further training
 * forwards for a multi-view loss, logging renders, graph replays -- use
 * other workspaces and never overwrite it.  flags: CS_RENDER_SYNC,
 * CS_RENDER_NO_CLIP.  Release with cs_state_release. */
typedef struct cs_state cs_state;
int cs_render_train(cs_ctx* ctx, const cs_source* src, const cs_camera* cam, const cs_settings* st,
                    float* out_rgb, uint32_t flags, cs_state** state_out, void* stream);
/* dL/dimage (device (H,W,3) float32) of that forward -> parameter gradients.
 * Waits for the forward to complete (not for the work after it) and fails
 * with CS_ENOMEM if the forward overflowed its pair buffer (the image and the
 * gradients of that step are invalid; the buffer is grown for the next one).
 * May be called more than once per state.  Not in the reference
 * (SPEC.md:76); semantics in SURVEY.md Appendix A. */
int cs_render_backward(cs_ctx* ctx, cs_state* state, const float* dl_dimg, const cs_grads* out,
                       void* stream);
void cs_state_release(cs_state* state);

/* Per-stage CUDA-event timing of the next max_frames cs_render calls on this
 * context; cs_timing_end returns per-stage sums in ms over the frames timed:
 * [select, project, depth_sort, gather_scan, duplicate, tile_sort, ranges, blend]. */
int cs_timing_begin(cs_ctx* ctx, int32_t max_frames);
int cs_timing_end(cs_ctx* ctx, double* stage_ms, int32_t* frames);

/* Frame graphs (no reference counterpart; B200 launch path): an asynchronous
 * cs_render (no SYNC/DEBUG/DIAG/KEEP_STATE flag, no stats, no timing) whose
 * source, settings, resolution, output, stream and buffer capacities repeat
 * is captured once into a CUDA graph and replayed with only the camera
 * parameters patched.  Returns the number of graphs cached by the context
 * (diagnostics); set CS_NO_GRAPH in the environment to disable. */
int cs_frame_graphs(cs_ctx* ctx);

/* Stats of the last frame (synchronises the stream). */
int cs_frame_stats_get(cs_ctx* ctx, cs_frame_stats* out, void* stream);

/* Synchronise `stream` and report CS_ENOMEM if an asynchronous frame on this
 * context overflowed its tile-pair buffer (that frame rendered incompletely;
 * the buffers are grown).  Every cs_render / cs_render_train call performs
 * the same (non-synchronising) check on entry, so an overflow is never
 * silent: it fails the frame's next call at the latest. */
int cs_check(cs_ctx* ctx, void* stream);

/* Golden-intermediate dumps of the last frame, host destinations.
 * cs_dump_projected mirrors render._Projected (render.py:89-108): arrays in
 * depth order; source = index into the assembled cloud.
 * cs_dump_tiles mirrors render._bin_tiles (render.py:217-249): tile_ids
 * (indices into the depth-sorted splats) and CSR offsets [n_tiles+1]. */
int cs_dump_projected(cs_ctx* ctx, double* means, double* conics, double* covs, double* depths,
                      double* colors, double* opacities, double* radii, int64_t* source,
                      void* stream);
int cs_dump_tiles(cs_ctx* ctx, int64_t* tile_ids, int64_t* offsets, void* stream);
/* Assembled-order (segment) table of the last LoD frame:
 * per piece (cloud index = level*n_blocks + block, count). */
int cs_dump_segments(cs_ctx* ctx, int32_t* cloud_index, int64_t* count, int32_t max_n,
                     int32_t* n_out, void* stream);
/* Assembled order of the last pointwise frame (lod.py:378-390): packed
 * (cloud_index << 40 | row) per assembled Gaussian. */
int cs_dump_assembled_list(cs_ctx* ctx, uint64_t* packed, int64_t max_n, int64_t* n_out,
                           void* stream);

/* ---- the reference's native kernel, one for one --------------------------
 * _kernels.blend_tiles (_kernels.py:17-76) with the same argument list; all
 * arrays are DEVICE pointers, same dtypes and shapes as the numba kernel. */
int cs_blend_tiles(cs_ctx* ctx, const int64_t* tile_ids, const int64_t* tile_offsets,
                   int64_t n_tiles, const double* means, const double* conics,
                   const double* colors, const double* opacities, int64_t n_splats,
                   const double* background, int32_t tile_size, int32_t width, int32_t height,
                   int32_t n_tiles_x, double alpha_floor, double t_floor, double* out,
                   int64_t* fragments, void* stream);

/* ---- utilities used by the API mirror (core.py) -------------------------- */
/* build_covariances (core.py:107-111): n quats (w,x,y,z) + scales -> 3x3. */
int cs_build_covariances(cs_ctx* ctx, int64_t n, const double* scales, const double* quats,
                         double* out, void* stream);
/* sh_to_colors (core.py:166-172): sh (n,3,C) f64, dirs (n,3) -> colors (n,3). */
int cs_sh_to_colors(cs_ctx* ctx, int64_t n, const double* sh, int32_t coeffs,
                    const double* dirs, int32_t degree, double* out, void* stream);

/* ---- block training (the reference has no backward) ---
 * Training loss of metrics.py:121-125, (1-lam)*L1 + lam*(1-SSIM) with the
 * valid-region 11x11 Gaussian-window SSIM of metrics.py:70-95, and its
 * gradient.  img, ref, grad_out: device (H,W,3) float32; loss_out: device
 * double[1].  H, W >= 11 (metrics.py:80-81), else CS_EINVAL. */
int cs_training_loss(cs_ctx* ctx, const float* img, const float* ref, int32_t height,
                     int32_t width, double lam, double* loss_out, float* grad_out, void* stream);
/* Adam hyper-parameters (torch.optim.Adam semantics, bias-corrected; step is
 * the 1-based step count after this update).  Learning rates per parameter
 * group; the manifest scales (partition.py:45-50) are applied by the caller. */
typedef struct cs_adam_hparams {
  float lr_position, lr_scale, lr_rotation, lr_opacity, lr_sh;
  float beta1, beta2, eps;
  int32_t step;
  int32_t reserved;
} cs_adam_hparams;
/* One Adam step of a block's raw parameters with the PLY activations
 * (ply.py:108-123: exp scale, sigmoid opacity, normalised quaternion).
 * geom: device (K,11) float32 rows (16-byte aligned, as are the moments, sh, sh moments, grads->rotations, grads->sh and the quads) [x,y,z, log s0..2, q w,x,y,z (raw), logit o];
 * geom_m/geom_v its Adam moments; sh (K,3C) float32 and its moments.
 * grads: cs_render_backward's output for the activated parameters.
 * Writes the activated (K,4) float32 quads pos_op/scale/quat that a cs_cloud
 * with sh_stride = 3C (C = 4 or 16) reads for the next forward. */
int cs_block_adam(cs_ctx* ctx, int64_t K, int32_t sh_coeffs, float* geom, float* geom_m,
                  float* geom_v, float* sh, float* sh_m, float* sh_v, const cs_grads* grads,
                  const cs_adam_hparams* hp, float* pos_op, float* scale, float* quat,
                  void* stream);
/* The activated quads of geom without an update (first forward). */
int cs_block_activate(cs_ctx* ctx, int64_t K, const float* geom, float* pos_op, float* scale,
                      float* quat, void* stream);
/* ---- fusion (partition.py:570-587) ---------------------------------------
 * Block membership of n positions: normalize_position (partition.py:110-114)
 * -> contract (partition.py:117-126) -> block_of_points (partition.py:161-169).
 * positions: device, fp32 (f32=1) or fp64 xyz triples.  out: device int32. */
int cs_block_of_points(cs_ctx* ctx, int64_t n, const void* positions, int32_t f32,
                       const double* p_min, const double* p_max, int32_t nx, int32_t ny,
                       int32_t nz, int32_t* out, void* stream);
/* Stable compaction of the rows of one block cloud that still belong to block j
 * (the keep mask of fuse, partition.py:582-585): writes kept row indices
 * (device int64, ascending) and the count (device int64). */
int cs_fuse_filter(cs_ctx* ctx, int64_t n, const void* positions, int32_t f32,
                   const double* p_min, const double* p_max, int32_t nx, int32_t ny, int32_t nz,
                   int32_t block, int64_t* kept_idx, int64_t* kept_count, void* stream);

/* ---- LoD generation (lod.py:54-248) -------------------
 * significance_scores (lod.py:54-101): per-Gaussian training-view hit count x
 * opacity x percentile-clamped volume^0.1.  cams: HOST array of n_cams views.
 * scores: device double[count]; hits: device int32[count] or NULL. */
int cs_significance(cs_ctx* ctx, const cs_cloud* cloud, const cs_camera* cams, int32_t n_cams,
                    const cs_settings* st, double* scores, int32_t* hits, void* stream);
/* _priority (lod.py:114-116): indices by descending score, ties -> lower index.
 * scores: device double[n]; order: device int32[n]. */
int cs_priority(cs_ctx* ctx, int64_t n, const double* scores, int32_t* order, void* stream);
/* build_lod's kept rows (lod.py:222-234): level L (rates coarsest first, HOST)
 * keeps the top _keep_count(rate_L, n) of `order`, grouped by block in
 * ascending block id, ascending row inside a block.  rows: device
 * int32[n_levels * n] (level L at offset L*n); counts: HOST int64
 * [n_levels * n_blocks].  Synchronises `stream`. */
int cs_lod_rows(cs_ctx* ctx, int64_t n, const int32_t* order, const int32_t* membership,
                int32_t n_blocks, const double* rates, int32_t n_levels, int32_t* rows,
                int64_t* counts, void* stream);
/* mad_bounds (lod.py:130-147) of every block's members (membership: device
 * int32[count]); blocks without members get zero bounds (lod.py:236-240).
 * bmin/bmax: HOST double[n_blocks * 3].  Synchronises `stream`. */
int cs_mad_bounds(cs_ctx* ctx, const cs_cloud* cloud, const int32_t* membership, int32_t n_blocks,
                  double n_mad, double* bmin, double* bmax, void* stream);
/* GaussianCloud.take(rows).with_sh_degree (core.py): copies the geometry quads
 * of `rows` and the first dst->sh_coeffs SH coefficients per channel into the
 * caller-allocated dst (same fp64 flag; dst->count is ignored, n rows written). */
int cs_gather_cloud(cs_ctx* ctx, const cs_cloud* src, const int32_t* rows, int64_t n,
                    const cs_cloud* dst, void* stream);

/* ---- training-data assignment (partition.py:172-439) ----
 * bounds_contain(contract(normalize_position(p)), lo, hi) (partition.py:110-126,
 * 172-181) for n points (device xyz, fp32 or fp64, stride 3 floats or 4 = the
 * pos_op quads of a cs_cloud); p_min = p_max = NULL: the points are already
 * contracted (BlockGrid.contracted).  mask: device uint8[n] or NULL; count:
 * HOST int64 (synchronises `stream`) or NULL. */
int cs_bounds_contain(cs_ctx* ctx, int64_t n, const void* positions, int32_t f32, int32_t stride,
                      const double* p_min, const double* p_max, const double* lo, const double* hi,
                      uint8_t* mask, int64_t* count, void* stream);
/* metrics.ssim (metrics.py:70-96) of two device (H, W, 3) float32 images with
 * the reference's 11x11 window (HOST double[121]).  acc4: device double[4];
 * acc4[3] receives the SSIM (acc4[0..2] per-channel sums).  Asynchronous. */
int cs_ssim(cs_ctx* ctx, const float* img_a, const float* img_b, int32_t height, int32_t width,
            const double* window, double* acc4, void* stream);

/* ---- measurement --------------------------------------------------------------
 * Dense DFMA throughput of this device (TFLOP/s, 2 flops per DFMA), measured
 * with CUDA events: the FP64 roofline denominator of the blend.
 * Synchronises `stream`. */
int cs_measure_fp64_peak(cs_ctx* ctx, double* tflops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CS_API_H */

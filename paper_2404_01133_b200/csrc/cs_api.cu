// cs_api.cu -- C ABI (include/cs_api.h): context, workspace and the frame
// pipeline K1..K9 on one stream with no host round trip.
//
//   K1  lod_select / pointwise      (lod.py:330-401)            cs_lod.cu
//   K3  project + cull              (render.py:111-172)         cs_project.cu
//   K4  depth radix sort, 64-bit    (render.py:176-177)         cs_sort.cu
//   K5  rank gather + pair scan     (render.py:178-188,226-236) cs_bin.cu
//   K6  pair duplication            (render.py:237-243)         cs_bin.cu
//   K7  tile radix sort             (render.py:245)             cs_sort.cu
//   K8  tile ranges                 (render.py:247-248)         cs_bin.cu
//   K9  blend                       (_kernels.py:17-76)         cs_blend.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <cstdlib>
#include <string>
#include <vector>

#include "cs_internal.cuh"

namespace cs {
// cs_project.cu
void launch_project(const cs_cloud* d_clouds, const Seg* d_segs, DevStats* d_stats,
                    const cs_camera& cam, const cs_settings& st, int64_t capacity,
                    const ProjOutputs& out, const uint64_t* list, cudaStream_t s);
void launch_setup_cloud(const cs_cloud& c, cs_cloud* d_clouds, Seg* d_segs, DevStats* d_stats,
                        cudaStream_t s);
void launch_build_covariances(int64_t n, const double* scales, const double* quats, double* out,
                              cudaStream_t s);
void launch_sh_to_colors(int64_t n, const double* sh, int C, const double* dirs, int degree,
                         double* out, cudaStream_t s);
// cs_lod.cu
void launch_lod_select(const LodTables& T, const cs_camera& cam, int force_level,
                       cs_decision* dec, Seg* segs, DevStats* stats, cudaStream_t s);
void launch_pointwise(const LodTables& T, const cs_camera& cam, int force_level, uint64_t* status,
                      uint64_t* list, Seg* segs, DevStats* stats, cudaStream_t s);
void launch_block_visible(int n, const double* bmin, const double* bmax, const cs_camera& cam,
                          uint8_t* vis, double* dist, cudaStream_t s);
void launch_select_level(int n, const double* d, int ni, const double* iv, int32_t* out,
                         cudaStream_t s);
// cs_sort.cu
size_t radix_status_words(int64_t capacity, int key_bytes);
template <typename K>
int radix_sort(K* k0, uint32_t* v0, K* k1, uint32_t* v1, const int64_t* n_dev, int64_t capacity,
               int begin_bit, int end_bit, uint32_t* hist, uint32_t* status, uint32_t* tickets,
               cudaStream_t s, bool hist_ready = false, bool identity_vals = false);
// cs_depth.cu
void launch_fix_depth_runs(const uint32_t* k32_sorted, uint32_t* order, const uint64_t* k64,
                           const DevStats* stats, int64_t capacity, void* ctl_mem,
                           uint32_t* long_runs, uint32_t long_cap, uint32_t* scratch,
                           cudaStream_t s);
size_t fix_ctl_bytes();
int64_t fix_long_cap(int64_t capacity);
// cs_train.cu
void launch_training_loss(const float* img, const float* ref, int H, int W, double lam,
                          float* maps, double* acc, double* loss, float* grad, cudaStream_t s);
void launch_block_adam(int64_t K, int C, float* geom, float* gm, float* gv, float* sh, float* shm,
                       float* shv, const cs_grads& g, const cs_adam_hparams& h, float4* pos_op,
                       float4* scale, float4* quat, cudaStream_t s);
void launch_activate_geom(int64_t K, const float* geom, float4* pos_op, float4* scale, float4* quat,
                          cudaStream_t s);
// cs_bin.cu
int64_t bin_chunks(int64_t capacity);
const void* lod_select_kernel();
const void* project_kernel();
const void* project_staged_kernel();
int64_t bin_status_words(int64_t capacity);
void launch_bin_pairs(const uint32_t* order, const uint2* rects, DevStats* stats, int64_t pair_cap,
                      int64_t capacity, uint64_t* status, int ntx, uint32_t* keys, uint32_t* vals,
                      uint32_t* hist, int key_bits, bool emit, int64_t* host_overflow,
                      cudaStream_t s);


void launch_tile_ranges(const uint32_t* keys, const uint32_t* vals, const short4* boxes,
                        const int64_t* n_pairs, uint2* ranges, uint32_t* bxs, uint32_t* bys,
                        cudaStream_t s);
void launch_dump_projected(const uint32_t* order, const ProjRec* recs, const DevStats* stats,
                           double* means, double* conics, double* covs, double* depths,
                           double* colors, double* opac, double* radii, int64_t* src,
                           cudaStream_t s);
void launch_dump_tiles(const uint32_t* order, const uint32_t* vals, const uint2* ranges,
                       const DevStats* stats, int n_tiles, int64_t* rank_of, int64_t* tile_ids,
                       int64_t* offsets, cudaStream_t s);
// cs_blend.cu
int blend_ppt(int tile_size);
void launch_tile_order(const uint2* ranges, int n_tiles, uint32_t* order, cudaStream_t s);
void launch_blend(int n_tiles, const uint32_t* list, const uint32_t* bxs, const uint32_t* bys,
                  const uint2* ranges, const HotRec* hot, const FastRec* fast, const uint32_t* order,
                  const BlendParams& bp, void* out, bool f64_out, int32_t* frag_tile,
                  DevStats* stats, const BlendState* keep, cudaStream_t s);
void launch_pack(int64_t m, const double* means, const double* conics, const double* colors,
                 const double* opac, double alpha_floor, HotRec* hot, int64_t p,
                 const int64_t* tile_ids, int64_t n_tiles, const int64_t* offsets, uint32_t* list,
                 uint32_t* bxs, uint32_t* bys, uint2* ranges, cudaStream_t s);
// cs_fuse.cu
void launch_block_of_points(int64_t n, const void* pos, int f32, const double* pmin,
                            const double* pmax, int nx, int ny, int nz, int32_t* out,
                            cudaStream_t s);
void launch_fuse_filter(int64_t n, const void* pos, int f32, const double* pmin, const double* pmax,
                        int nx, int ny, int nz, int block, uint64_t* status, uint32_t* ticket,
                        int64_t* kept, int64_t* kept_count, cudaStream_t s);
// cs_backward.cu
void launch_blend_bwd(int n_tiles, const uint32_t* list, const uint32_t* bxs, const uint32_t* bys,
                      const uint2* ranges, const HotRec* hot, const FastRec* fast, const uint32_t* order,
                      const cs_settings& st, int width, int height, int ntx, const float* dl_dimg,
                      const BlendState& state, uint32_t* ticket, gacc_t* grads, int64_t cap,
                      cudaStream_t s);
void launch_project_bwd(const cs_cloud& cl, const uint64_t* depth_keys, const cs_camera& cam,
                        const cs_settings& st, const gacc_t* grads, int64_t cap, const cs_grads& out,
                        cudaStream_t s);
cudaError_t significance_run(const cs_cloud& cl, const cs_camera* cams_host, int n_cams,
                             const cs_settings& st, double* scores, int32_t* hits_out,
                             cudaStream_t s);
cudaError_t priority_run(int64_t K, const double* scores, int32_t* order, cudaStream_t s);
cudaError_t lod_rows_run(int64_t K, const int32_t* order, const int32_t* membership, int n_blocks,
                         const int64_t* keep, int n_levels, int32_t* rows_out, int64_t* counts_dev,
                         cudaStream_t s);
cudaError_t mad_bounds_run(const cs_cloud& cl, const int32_t* membership, int n_blocks,
                           double n_mad, double* bmin_dev, double* bmax_dev, int64_t* cnt_host,
                           cudaStream_t s);
void launch_gather_cloud(const cs_cloud& src, const int32_t* rows, int64_t n, const cs_cloud& dst,
                         cudaStream_t s);
void launch_bounds_contain(int64_t n, const void* pos, int f32, int stride, const double* pmin,
                           const double* pmax, const double* lo, const double* hi, uint8_t* mask,
                           unsigned long long* count, cudaStream_t s);
cudaError_t ssim_run(const float* a, const float* b, int H, int W, const double* window,
                     double* acc4, cudaStream_t s);
cudaError_t fp64_peak_run(double* tflops, cudaStream_t s);
}  // namespace cs

using namespace cs;

static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CS_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      if (e_ == cudaErrorMemoryAllocation)                                                 \
        return fail(CS_ENOMEM, "%s: %s", #call, cudaGetErrorString(e_));                   \
      return fail(CS_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
    }                                                                                      \
  } while (0)

#define CS_CHECK_LAUNCH() CS_CUDA(cudaGetLastError())

// A growable device buffer.
// Bumped whenever any device buffer is (re)allocated or freed: part of the
// frame-graph key, so a captured frame never replays with a stale pointer.
static std::atomic<uint64_t> g_buf_generation{1};

struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    g_buf_generation++;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t b = std::max<size_t>(want, 256);
    cudaError_t e = cudaMalloc(&p, b);
    if (e == cudaSuccess) bytes = b;
    return e;
  }
  void release() {
    if (p) {
      g_buf_generation++;
      cudaFree(p);
    }
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const { return reinterpret_cast<T*>(p); }
};

struct cs_lod {
  cs_ctx* ctx = nullptr;
  uint64_t serial = 0;  // unique per scene (frame-graph cache key)
  int n_levels = 0, n_blocks = 0;
  std::vector<cs_cloud> clouds;
  std::vector<int64_t> counts;
  int64_t max_assembled = 0;
  int64_t total_all = 0;
  DBuf d_clouds, d_bmin, d_bmax, d_int, d_occ, d_allsegs;
  LodTables tables() const {
    LodTables T;
    T.clouds = d_clouds.as<cs_cloud>();
    T.bmin = d_bmin.as<double>();
    T.bmax = d_bmax.as<double>();
    T.intervals = d_int.as<double>();
    T.occupied = d_occ.as<uint8_t>();
    T.all_segs = d_allsegs.as<Seg>();
    T.n_levels = n_levels;
    T.n_blocks = n_blocks;
    T.total_all = total_all;
    return T;
  }
};

// The buffers one frame writes and its backward reads (pair lists, HotRecs,
// depth keys, tile ranges, per-pixel blend state, stats).  A context renders
// into its current workspace; cs_render_train hands the workspace to a
// cs_state (held until cs_state_release), and the next frame switches to a
// free workspace, so any number of renders may run between a training
// forward and its backward without touching the state the backward reads.
struct Ws {
  DBuf stats, clouds1, segs, dec;
  DBuf st_gather, st_pw, st_sort, hist, sort_tickets;
  DBuf keysA, valsA, keysB, valsB, recs;
  DBuf k32A, k32B, long_runs, fix_ctl;          // K4 32-bit depth sort + K4b run fix-up
  DBuf hot, fast, boxes, rects, tile_order;
  DBuf pkA, pvA, pkB, pvB, ranges, frag_tile, pw_list;
  DBuf st_t, st_last, st_acc;
  int64_t cap_vis = 0, cap_pairs = 0, cap_pw = 0, cap_tiles = 0;
  bool held = false;  // owned by a cs_state
  // last frame bookkeeping (for dumps / backward)
  const uint32_t* last_order = nullptr;
  bool last_debug = false;
  const uint32_t* last_list = nullptr;
  const uint32_t* last_bxs = nullptr;  // pair-major cull boxes of the last frame
  const uint32_t* last_bys = nullptr;
  const uint2* last_ranges = nullptr;
  int last_tiles = 0;
  int last_width = 0, last_height = 0;
  void release() {
    DBuf* all[] = {&stats, &clouds1, &segs, &dec, &st_gather, &st_pw, &st_sort, &hist, &sort_tickets,
                   &keysA, &valsA, &keysB, &valsB, &recs, &k32A, &k32B, &long_runs, &fix_ctl, &hot,
                   &fast, &boxes, &rects, &tile_order, &pkA, &pvA, &pkB, &pvB, &ranges, &frag_tile, &pw_list,
                   &st_t, &st_last, &st_acc};
    for (DBuf* b : all) b->release();
  }
};

struct cs_ctx {
  int device = 0;
  std::mutex mu;  // one frame at a time per context (contexts are per thread/stream)
  std::vector<Ws*> ws_all;   // every workspace of this context
  Ws* ws = nullptr;          // the one the next frame renders into
  Ws* last = nullptr;        // the one the last frame rendered into (dumps, stats)
  DBuf st_fuse, fuse_ticket;
  DBuf scratch1, scratch2, scratch3, scratch4;  // API utilities
  DBuf gacc;                                    // per-rank blend-backward partials
  DBuf loss_maps, loss_acc;                     // cs_training_loss workspace
  cs_frame_stats* h_stats = nullptr;            // pinned
  // pair-buffer overflow of an asynchronous frame, written by k_bin_pairs into
  // mapped pinned memory: [0] pairs the frame needed, [1] its frame serial
  volatile int64_t* h_overflow = nullptr;
  int64_t* d_overflow = nullptr;
  int64_t serial = 0;        // frames rendered on this context
  // frame graph (see cs_render): the last eligible call's key, and the
  // captured, instantiated frame for it with the camera-carrying kernel nodes
  struct FrameKey {
    cs_source src;
    cs_settings st;
    uint64_t lod_serial;
    int width, height;
    uint32_t flags;
    void* out;
    cudaStream_t stream;
    const void* ws;
    int64_t cap_vis, cap_pairs, cap_pw, cap_tiles;
    uint64_t buf_generation;
  };
  struct CamNode {
    cudaGraphNode_t node;
    cudaKernelNodeParams params;
    std::vector<void*> args;
    int cam_arg;
  };
  struct FrameGraph {
    FrameKey key;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::vector<CamNode> cam_nodes;
  };
  std::vector<FrameGraph> graphs;   // most recent last (double-buffered outputs: 2 keys)
  std::vector<FrameKey> seen;       // recent eligible keys (capture on the second sighting)
  std::vector<FrameKey> uncapturable;  // keys whose capture failed (never retried)
  cudaStream_t capture_stream = nullptr;
  cs_camera graph_cam{};
  // per-stage CUDA-event timing (cs_timing_begin/end)
  bool timing_on = false;
  int timing_max = 0, timing_frame = 0;
  std::vector<cudaEvent_t> tev;
};

// A training forward's kept state (cs_render_train): its workspace, the
// frame's geometry, and an event + pinned status word that tell the backward
// whether the forward completed without a pair-buffer overflow.
struct cs_state {
  cs_ctx* ctx = nullptr;
  Ws* ws = nullptr;
  int64_t count = 0;      // rows of the rendered cloud
  int width = 0, height = 0;
  cs_camera cam{};
  cs_settings st{};
  cs_cloud cloud{};
  cudaEvent_t done = nullptr;
  int32_t* h_status = nullptr;  // pinned: DevStats.status after the forward
  int64_t* h_pairs = nullptr;   // pinned: DevStats.pairs after the forward
};

static constexpr int kStages = 8;  // select, project, depth sort, gather+scan, duplicate,
                                   // tile sort, ranges, blend
static void mark(cs_ctx* c, int stage, cudaStream_t s) {
  if (c->timing_on && c->timing_frame < c->timing_max)
    cudaEventRecord(c->tev[(size_t)c->timing_frame * (kStages + 1) + stage], s);
}

extern "C" {

int cs_version(void) { return 1; }
const char* cs_last_error(void) { return g_err.c_str(); }

static int ws_init(Ws* w) {
  if (w->stats.ensure(sizeof(DevStats)) || w->hist.ensure(sizeof(uint32_t) * 256 * 8) ||
      w->sort_tickets.ensure(sizeof(uint32_t) * 16) || w->clouds1.ensure(sizeof(cs_cloud)))
    return fail(CS_ENOMEM, "frame workspace");
  return CS_OK;
}

// The workspace the next frame renders into: the current one unless a
// cs_state holds it, then a free one (new workspaces start from the current
// pair capacity, so a training loop does not re-learn its sizes).
static int frame_ws(cs_ctx* c, Ws** out) {
  if (c->ws && !c->ws->held) { *out = c->ws; return CS_OK; }
  for (Ws* w : c->ws_all)
    if (!w->held) { c->ws = w; *out = w; return CS_OK; }
  Ws* w = new Ws();
  c->ws_all.push_back(w);
  int rc = ws_init(w);
  if (rc) return rc;
  if (c->ws) w->cap_pairs = c->ws->cap_pairs;
  c->ws = w;
  *out = w;
  return CS_OK;
}

int cs_create(int device, cs_ctx** out) {
  if (!out) return fail(CS_EINVAL, "out is NULL");
  int n = 0;
  CS_CUDA(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(CS_EINVAL, "device %d not present (%d)", device, n);
  CS_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  CS_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(CS_EINVAL, "libcsgpu is built for sm_100a; device %d is sm_%d%d", device,
                prop.major, prop.minor);
  cs_ctx* c = new cs_ctx();
  c->device = device;
  CS_CUDA(cudaMallocHost(&c->h_stats, sizeof(cs_frame_stats)));
  void* ov = nullptr;
  CS_CUDA(cudaHostAlloc(&ov, 2 * sizeof(int64_t), cudaHostAllocMapped));
  c->h_overflow = reinterpret_cast<volatile int64_t*>(ov);
  c->h_overflow[0] = c->h_overflow[1] = 0;
  CS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->d_overflow), ov, 0));
  Ws* w = nullptr;
  int rc = frame_ws(c, &w);
  if (rc) return rc;
  if (c->fuse_ticket.ensure(sizeof(uint32_t) * 4) != cudaSuccess) return fail(CS_ENOMEM, "tk");
  *out = c;
  return CS_OK;
}

void cs_destroy(cs_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (Ws* w : c->ws_all) {
    w->release();
    delete w;
  }
  DBuf* all[] = {&c->st_fuse, &c->fuse_ticket, &c->gacc, &c->loss_maps, &c->loss_acc,
                 &c->scratch1, &c->scratch2, &c->scratch3, &c->scratch4};
  for (DBuf* b : all) b->release();
  if (c->h_stats) cudaFreeHost(c->h_stats);
  if (c->h_overflow) cudaFreeHost(const_cast<int64_t*>(c->h_overflow));
  for (cudaEvent_t e : c->tev) cudaEventDestroy(e);
  for (auto& g : c->graphs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
  }
  if (c->capture_stream) cudaStreamDestroy(c->capture_stream);
  delete c;
}

// ---------------------------------------------------------------------------
// LoD scene

int cs_lod_create(cs_ctx* ctx, const cs_lod_desc* d, cs_lod** out) {
  if (!ctx || !d || !out) return fail(CS_EINVAL, "NULL argument");
  if (d->n_levels <= 0 || d->n_blocks <= 0) return fail(CS_EINVAL, "empty LoD scene");
  CS_CUDA(cudaSetDevice(ctx->device));
  cs_lod* L = new cs_lod();
  L->ctx = ctx;
  static std::atomic<uint64_t> next_serial{1};
  L->serial = next_serial++;
  L->n_levels = d->n_levels;
  L->n_blocks = d->n_blocks;
  const int LJ = d->n_levels * d->n_blocks;
  L->clouds.assign(d->clouds, d->clouds + LJ);
  L->counts.resize(LJ);
  std::vector<Seg> allsegs(LJ);
  int64_t start = 0;
  for (int i = 0; i < LJ; ++i) {
    const cs_cloud& c = L->clouds[i];
    if (c.count < 0 || (c.count > 0 && (!c.pos_op || !c.scale || !c.quat || !c.sh)))
      return fail(CS_EINVAL, "cloud %d: bad descriptor", i);
    if (c.count > 0 && (c.sh_stride < 3 * c.sh_coeffs || (c.sh_stride & 3)))
      return fail(CS_EINVAL, "cloud %d: sh_stride %d", i, c.sh_stride);
    L->counts[i] = c.count;
    allsegs[i].start = start;
    allsegs[i].count = c.count;
    allsegs[i].cloud = i;
    allsegs[i].pad = 0;
    start += c.count;
  }
  L->total_all = start;
  std::vector<uint8_t> occ(d->n_blocks);
  for (int j = 0; j < d->n_blocks; ++j) {
    occ[j] = L->counts[(d->n_levels - 1) * d->n_blocks + j] > 0;  // LodScene.occupied (lod.py:207-208)
    int64_t mx = 0;
    for (int l = 0; l < d->n_levels; ++l) mx = std::max(mx, L->counts[l * d->n_blocks + j]);
    L->max_assembled += mx;
  }
  if (L->d_clouds.ensure(sizeof(cs_cloud) * LJ) || L->d_bmin.ensure(sizeof(double) * 3 * d->n_blocks) ||
      L->d_bmax.ensure(sizeof(double) * 3 * d->n_blocks) ||
      L->d_int.ensure(sizeof(double) * 2 * d->n_levels) || L->d_occ.ensure(d->n_blocks) ||
      L->d_allsegs.ensure(sizeof(Seg) * LJ))
    return fail(CS_ENOMEM, "lod tables");
  CS_CUDA(cudaMemcpy(L->d_clouds.p, L->clouds.data(), sizeof(cs_cloud) * LJ, cudaMemcpyHostToDevice));
  CS_CUDA(cudaMemcpy(L->d_bmin.p, d->bounds_min, sizeof(double) * 3 * d->n_blocks, cudaMemcpyHostToDevice));
  CS_CUDA(cudaMemcpy(L->d_bmax.p, d->bounds_max, sizeof(double) * 3 * d->n_blocks, cudaMemcpyHostToDevice));
  CS_CUDA(cudaMemcpy(L->d_int.p, d->intervals, sizeof(double) * 2 * d->n_levels, cudaMemcpyHostToDevice));
  CS_CUDA(cudaMemcpy(L->d_occ.p, occ.data(), d->n_blocks, cudaMemcpyHostToDevice));
  CS_CUDA(cudaMemcpy(L->d_allsegs.p, allsegs.data(), sizeof(Seg) * LJ, cudaMemcpyHostToDevice));
  *out = L;
  return CS_OK;
}

void cs_lod_destroy(cs_lod* L) {
  if (!L) return;
  cudaSetDevice(L->ctx->device);
  cudaDeviceSynchronize();
  L->d_clouds.release(); L->d_bmin.release(); L->d_bmax.release(); L->d_int.release();
  L->d_occ.release(); L->d_allsegs.release();
  delete L;
}

static int ensure_frame_buffers(Ws* w, int64_t cap_vis, int n_segs, int n_blocks,
                                int n_tiles, int64_t cap_pw) {
  cap_vis = std::max<int64_t>(cap_vis, 1);
  if (w->segs.ensure(sizeof(Seg) * std::max(n_segs, 1)) ||
      w->dec.ensure(sizeof(cs_decision) * std::max(n_blocks, 1)))
    return fail(CS_ENOMEM, "segment tables");
  if (cap_vis > w->cap_vis) {
    int64_t cap = std::max<int64_t>(cap_vis, w->cap_vis + w->cap_vis / 2);
    if (cap >= (1ll << 30)) return fail(CS_EINVAL, "more than 2^30 assembled Gaussians");
    const int64_t chunks = (cap + 255) / 256 + 1;
    if (w->st_gather.ensure(8 * std::max<int64_t>(chunks, bin_status_words(cap))) ||
        w->keysA.ensure(8 * cap) || w->keysB.ensure(8 * cap) || w->valsA.ensure(4 * cap) ||
        w->k32A.ensure(4 * cap) || w->k32B.ensure(4 * cap) ||
        w->long_runs.ensure(4 * fix_long_cap(cap)) || w->fix_ctl.ensure(fix_ctl_bytes()) ||
        w->valsB.ensure(4 * cap) || w->hot.ensure(sizeof(HotRec) * cap) ||
        w->rects.ensure(8 * cap) || w->boxes.ensure(8 * cap))
      return fail(CS_ENOMEM, "visible-splat buffers (%lld)", (long long)cap);
    w->cap_vis = cap;
    // the pair capacity follows the visible capacity (8 pairs per splat): a
    // frame of a larger cloud never starts from a smaller cloud's pair buffer
    w->cap_pairs = std::max<int64_t>(w->cap_pairs, std::max<int64_t>(1 << 20, 8 * cap));
  }
  if (w->cap_pairs == 0) w->cap_pairs = std::max<int64_t>(1 << 20, 8 * w->cap_vis);
  if (w->cap_pairs >= (1ll << 30)) w->cap_pairs = (1ll << 30) - 1;
  if (w->pkA.ensure(4 * w->cap_pairs) || w->pvA.ensure(4 * w->cap_pairs) ||
      w->pkB.ensure(4 * w->cap_pairs) || w->pvB.ensure(4 * w->cap_pairs))
    return fail(CS_ENOMEM, "pair buffers (%lld)", (long long)w->cap_pairs);
  const size_t sw = std::max(radix_status_words(w->cap_vis, 8), radix_status_words(w->cap_pairs, 4));
  if (w->st_sort.ensure(4 * sw)) return fail(CS_ENOMEM, "sort status");
  if (n_tiles > w->cap_tiles) {
    if (w->ranges.ensure(sizeof(uint2) * n_tiles) || w->frag_tile.ensure(4 * n_tiles) ||
        w->tile_order.ensure(4 * (n_tiles + 2 * 34 * 16)))  // + launch_tile_order's scratch
      return fail(CS_ENOMEM, "tile buffers");
    w->cap_tiles = n_tiles;
  }
  if (cap_pw > 0 && cap_pw > w->cap_pw) {
    if (w->pw_list.ensure(8 * cap_pw) || w->st_pw.ensure(8 * ((cap_pw + 255) / 256 + 1)))
      return fail(CS_ENOMEM, "pointwise buffers");
    w->cap_pw = cap_pw;
  }
  return CS_OK;
}

static int validate(const cs_camera* cam, const cs_settings* st) {
  if (!cam || !st) return fail(CS_EINVAL, "camera/settings NULL");
  if (cam->width <= 0 || cam->height <= 0) return fail(CS_EINVAL, "image dimensions must be positive");
  if (cam->width > 32000 || cam->height > 32000) return fail(CS_EINVAL, "images are limited to 32000 px per side");
  if (st->tile_size < 8) return fail(CS_EINVAL, "tile_size must be at least 8");
  if (blend_ppt(st->tile_size) == 0) return fail(CS_EINVAL, "tile_size > 64 not supported");
  if (st->sh_degree < 0 || st->sh_degree > 3) return fail(CS_EINVAL, "sh_degree must be 0..3");
  if (!(st->alpha_floor > 0.0 && st->alpha_floor < 1.0)) return fail(CS_EINVAL, "alpha_floor");
  if (!(st->transmittance_floor > 0.0 && st->transmittance_floor < 1.0))
    return fail(CS_EINVAL, "transmittance_floor");
  if (!(st->near_plane > 0.0)) return fail(CS_EINVAL, "near_plane must be positive");
  return CS_OK;
}

static int bits_for(int64_t n) {
  int b = 1;
  while ((1ll << b) < n) ++b;
  return b;
}

// One pass of the whole pipeline into workspace w (no sync).
static int render_once(cs_ctx* c, Ws* w, const cs_source* src, const cs_camera* cam,
                       const cs_settings* st, void* out, uint32_t flags, cudaStream_t s) {
  const int ts = st->tile_size;
  const int ntx = (cam->width + ts - 1) / ts, nty = (cam->height + ts - 1) / ts;
  const int n_tiles = ntx * nty;
  int64_t cap_vis = 0, cap_pw = 0;
  int n_segs = 1, n_blocks = 1;
  const cs_lod* L = src->lod;
  if (src->kind == CS_SRC_CLOUD) {
    const cs_cloud& cl = src->cloud;
    if (cl.count < 0 || (cl.count > 0 && (!cl.pos_op || !cl.scale || !cl.quat || !cl.sh)))
      return fail(CS_EINVAL, "bad cloud descriptor");
    if (cl.count > 0 && (cl.sh_stride < 3 * cl.sh_coeffs || (cl.sh_stride & 3)))
      return fail(CS_EINVAL, "bad sh_stride");
    cap_vis = cl.count;
  } else {
    if (!L) return fail(CS_EINVAL, "LoD source without scene");
    if (src->exclude) return fail(CS_EINVAL, "exclude masks apply to single-cloud sources only");
    n_segs = L->n_levels * L->n_blocks;
    n_blocks = L->n_blocks;
    if (src->kind == CS_SRC_LOD_BLOCK) {
      cap_vis = src->force_level >= 0 ? 0 : L->max_assembled;
      if (src->force_level >= 0) {
        if (src->force_level >= L->n_levels) return fail(CS_EINVAL, "force_level out of range");
        for (int j = 0; j < L->n_blocks; ++j) cap_vis += L->counts[src->force_level * L->n_blocks + j];
      }
    } else if (src->kind == CS_SRC_LOD_POINT) {
      cap_vis = L->total_all;
      cap_pw = L->total_all;
    } else {
      return fail(CS_EINVAL, "unknown source kind %d", src->kind);
    }
  }
  int rc = ensure_frame_buffers(w, cap_vis, n_segs, n_blocks, n_tiles, cap_pw);
  if (rc) return rc;
  c->last = w;
  ++c->serial;
  // the LoD selection camera: an AssembledSet keeps the camera it was
  // assembled for (lod.py:360-401), which may differ from the render camera
  const cs_camera& scam = src->select_cam ? *src->select_cam : *cam;
  DevStats* stats = w->stats.as<DevStats>();
  const bool timed = !(flags & CS_RENDER_PROJECT_ONLY);
  if (timed) mark(c, 0, s);
  CS_CUDA(cudaMemsetAsync(stats, 0, sizeof(DevStats), s));
  const cs_cloud* clouds = nullptr;
  const uint64_t* list = nullptr;
  if (src->kind == CS_SRC_CLOUD) {
    launch_setup_cloud(src->cloud, w->clouds1.as<cs_cloud>(), w->segs.as<Seg>(), stats, s);
    clouds = w->clouds1.as<cs_cloud>();
  } else if (src->kind == CS_SRC_LOD_BLOCK) {
    launch_lod_select(L->tables(), scam, src->force_level, w->dec.as<cs_decision>(),
                      w->segs.as<Seg>(), stats, s);
    clouds = L->d_clouds.as<cs_cloud>();
  } else {
    CS_CUDA(cudaMemsetAsync(w->st_pw.p, 0, 8 * ((cap_pw + 255) / 256 + 1), s));
    launch_pointwise(L->tables(), scam, src->force_level, w->st_pw.as<uint64_t>(),
                     w->pw_list.as<uint64_t>(), w->segs.as<Seg>(), stats, s);
    clouds = L->d_clouds.as<cs_cloud>();
    list = w->pw_list.as<uint64_t>();
  }
  CS_CHECK_LAUNCH();
  if (timed) mark(c, 1, s);
  const int64_t cap = std::max<int64_t>(cap_vis, 1);
  const bool debug = (flags & (CS_RENDER_DEBUG | CS_RENDER_PROJECT_ONLY)) != 0;
  if (debug && w->recs.ensure(sizeof(ProjRec) * w->cap_vis)) return fail(CS_ENOMEM, "debug records");
  // the certified float32 blend's records (frames without kept state)
  const bool fast_blend = !(flags & CS_RENDER_KEEP_STATE);
  // kept-state frames write them too for the backward's certified pre-reject
  const bool want_fast = fast_blend || CS_BWD_FAST;
  if (want_fast && w->fast.ensure(sizeof(FastRec) * w->cap_vis)) return fail(CS_ENOMEM, "blend records");
  ProjOutputs po{w->keysA.as<uint64_t>(), w->k32A.as<uint32_t>(), w->valsA.as<uint32_t>(),
                 w->hot.as<HotRec>(), want_fast ? w->fast.as<FastRec>() : nullptr,
                 w->rects.as<uint2>(), w->boxes.as<short4>(),
                 debug ? w->recs.as<ProjRec>() : nullptr,
                 src->kind == CS_SRC_CLOUD ? src->exclude : nullptr, std::log2(st->alpha_floor),
                 std::log((float)st->alpha_floor), fast_blend ? 1 : 0};
  launch_project(clouds, w->segs.as<Seg>(), stats, *cam, *st, cap, po, list, s);
  w->last_debug = debug;
  CS_CHECK_LAUNCH();
  if (timed) mark(c, 2, s);
  // K4: global depth order over the assembled set: stable 32-bit radix sort of
  // the float32-rounded depth (culled Gaussians carry ~0 and land behind the M
  // visible ones), then K4b re-sorts runs of equal float32 depth by (float64
  // depth, splat id) -- the exact stable argsort of render.py:176-177.
  const int which = radix_sort<uint32_t>(w->k32A.as<uint32_t>(), w->valsA.as<uint32_t>(),
                                         w->k32B.as<uint32_t>(), w->valsB.as<uint32_t>(),
                                         &stats->assembled, cap, 0, 32, w->hist.as<uint32_t>(),
                                         w->st_sort.as<uint32_t>(), w->sort_tickets.as<uint32_t>(), s, false,
                                         /*identity_vals=*/true);
  if (which < 0) return fail(CS_EINVAL, "depth sort: identity values need 8-bit digits");
  CS_CHECK_LAUNCH();
  uint32_t* order = which ? w->valsB.as<uint32_t>() : w->valsA.as<uint32_t>();
  const uint32_t* k32s = which ? w->k32B.as<uint32_t>() : w->k32A.as<uint32_t>();
  launch_fix_depth_runs(k32s, order, w->keysA.as<uint64_t>(), stats, cap, w->fix_ctl.p,
                        w->long_runs.as<uint32_t>(), (uint32_t)fix_long_cap(cap),
                        w->keysB.as<uint32_t>(), s);
  CS_CHECK_LAUNCH();
  if (timed) mark(c, 3, s);
  // K5+K6: pair counts in depth order, scanned, and the pairs emitted in one
  // pass (also counts the tile sort's digit histograms, so K7 skips its
  // counting pass)
  CS_CUDA(cudaMemsetAsync(w->st_gather.p, 0, 8 * (bin_chunks(cap) + 1), s));
  const bool project_only = (flags & CS_RENDER_PROJECT_ONLY) != 0;
  launch_bin_pairs(order, w->rects.as<uint2>(), stats, w->cap_pairs, cap,
                   w->st_gather.as<uint64_t>(), ntx, w->pkA.as<uint32_t>(), w->pvA.as<uint32_t>(),
                   bits_for(n_tiles) <= 24 ? w->hist.as<uint32_t>() : nullptr, bits_for(n_tiles),
                   !project_only, c->d_overflow, s);
  CS_CHECK_LAUNCH();
  if (timed) mark(c, 4, s);
  if (project_only) {
    w->last_order = order;
    w->last_list = nullptr;
    return CS_OK;
  }
  mark(c, 5, s);
  // K7: stable sort by tile id only (ceil(log2 T) bits)
  const int which2 = radix_sort<uint32_t>(w->pkA.as<uint32_t>(), w->pvA.as<uint32_t>(),
                                          w->pkB.as<uint32_t>(), w->pvB.as<uint32_t>(),
                                          &stats->pairs_eff, w->cap_pairs, 0, bits_for(n_tiles),
                                          w->hist.as<uint32_t>(), w->st_sort.as<uint32_t>(),
                                          w->sort_tickets.as<uint32_t>() + 8, s,
                                          /*hist_ready=*/bits_for(n_tiles) <= 24);
  CS_CHECK_LAUNCH();
  const uint32_t* tkeys = which2 ? w->pkB.as<uint32_t>() : w->pkA.as<uint32_t>();
  const uint32_t* tvals = which2 ? w->pvB.as<uint32_t>() : w->pvA.as<uint32_t>();
  mark(c, 6, s);
  // K8: tile ranges
  CS_CUDA(cudaMemsetAsync(w->ranges.p, 0, sizeof(uint2) * n_tiles, s));
  // the sort's other (key, value) buffers are free now: they take the pair-major boxes
  uint32_t* bxs = which2 ? w->pkA.as<uint32_t>() : w->pkB.as<uint32_t>();
  uint32_t* bys = which2 ? w->pvA.as<uint32_t>() : w->pvB.as<uint32_t>();
  launch_tile_ranges(tkeys, tvals, w->boxes.as<short4>(), &stats->pairs_eff, w->ranges.as<uint2>(), bxs, bys, s);
  CS_CHECK_LAUNCH();
  mark(c, 7, s);
  // K9: blend
  BlendParams bp;
  for (int i = 0; i < 3; ++i) bp.bg[i] = st->background[i];
  bp.alpha_floor = st->alpha_floor;
  bp.t_floor = st->transmittance_floor;
  bp.tile_size = ts;
  bp.width = cam->width;
  bp.height = cam->height;
  bp.ntx = ntx;
  bp.flags = flags;
  BlendState keep{nullptr, nullptr, nullptr};
  const int64_t npx = (int64_t)cam->width * cam->height;
  if (flags & CS_RENDER_KEEP_STATE) {
    if (w->st_t.ensure(8 * npx) || w->st_last.ensure(4 * npx) || w->st_acc.ensure(24 * npx))
      return fail(CS_ENOMEM, "blend state");
    keep = BlendState{w->st_t.as<double>(), w->st_last.as<int32_t>(), w->st_acc.as<double>()};
  }
  launch_tile_order(w->ranges.as<uint2>(), n_tiles, w->tile_order.as<uint32_t>(), s);
  CS_CHECK_LAUNCH();
  launch_blend(n_tiles, tvals, bxs, bys, w->ranges.as<uint2>(), w->hot.as<HotRec>(),
               fast_blend ? w->fast.as<FastRec>() : nullptr, w->tile_order.as<uint32_t>(),
               bp, out, (flags & CS_RENDER_F64_OUT) != 0, w->frag_tile.as<int32_t>(), stats,
               (flags & CS_RENDER_KEEP_STATE) ? &keep : nullptr, s);
  CS_CHECK_LAUNCH();
  mark(c, 8, s);
  if (c->timing_on && c->timing_frame < c->timing_max) ++c->timing_frame;
  w->last_order = order;
  w->last_list = tvals;
  w->last_bxs = bxs;
  w->last_bys = bys;
  w->last_ranges = w->ranges.as<uint2>();
  w->last_tiles = n_tiles;
  w->last_width = cam->width;
  w->last_height = cam->height;
  return CS_OK;
}

static_assert(offsetof(DevStats, blend_max_item_cycles) == offsetof(cs_frame_stats, blend_max_item_cycles) &&
                  offsetof(DevStats, blend_replays) == offsetof(cs_frame_stats, blend_replays) &&
                  sizeof(cs_frame_stats) == offsetof(DevStats, pairs_eff),
              "DevStats must lead with the cs_frame_stats layout");
static int fetch_stats(cs_ctx* c, Ws* w, cudaStream_t s) {
  // DevStats and cs_frame_stats share the leading layout
  if (!w) return fail(CS_EINVAL, "no frame rendered on this context");
  CS_CUDA(cudaMemcpyAsync(c->h_stats, w->stats.p, sizeof(cs_frame_stats), cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaStreamSynchronize(s));
  return CS_OK;
}

// An asynchronous frame that overflowed its pair buffer (k_bin_pairs wrote the
// pair count it needed into mapped host memory) is reported by the next call
// on the context: the buffers of every workspace grow to fit, and the call
// fails with CS_ENOMEM -- that frame's image is background-only and must be
// re-rendered.  Never silent.
static int check_overflow(cs_ctx* c) {
  const int64_t need = c->h_overflow[0];
  if (!need) return CS_OK;
  const int64_t cap = c->h_overflow[1];
  c->h_overflow[0] = 0;
  c->h_overflow[1] = 0;
  const int64_t grow = std::min<int64_t>((1ll << 30) - 1, need + need / 4 + 1024);
  for (Ws* w : c->ws_all) w->cap_pairs = std::max(w->cap_pairs, grow);
  if (need >= (1ll << 30))
    return fail(CS_ENOMEM, "an earlier asynchronous frame needed %lld tile pairs (> 2^30)", (long long)need);
  return fail(CS_ENOMEM,
              "an earlier asynchronous frame on this context overflowed its pair buffer (%lld pairs > "
              "%lld) and rendered incompletely; the buffers have been grown -- render it again",
              (long long)need, (long long)cap);
}

// Frame graphs.  A frame is ~18 kernels and ~10 memsets whose sizes all live
// in device memory, so it is graph-capturable; only the camera differs
// between the frames of a flythrough, and it reaches the device solely as a
// kernel parameter of K1 (k_lod_select) and K3 (k_project).  When two
// consecutive asynchronous calls share everything but the camera pose (same
// source, settings, resolution, output, stream, workspace and buffer
// capacities), the frame is captured once on a private stream and
// instantiated; later calls patch the two camera parameters with
// cudaGraphExecKernelNodeSetParams and launch the graph on the caller's
// stream -- the same kernels on the same buffers, without per-kernel launch
// gaps.  Synchronous, stats, debug, diagnostics, kept-state, timed and
// separate-selection-camera frames always take the direct path.
static bool graph_eligible(const cs_ctx* c, const cs_source* src, uint32_t flags,
                           const cs_frame_stats* stats_host) {
  const uint32_t direct = CS_RENDER_SYNC | CS_RENDER_DEBUG | CS_RENDER_PROJECT_ONLY | CS_RENDER_DIAG |
                          CS_RENDER_KEEP_STATE;
  if (std::getenv("CS_NO_GRAPH")) return false;
  return !(flags & direct) && !stats_host && !c->timing_on && !src->select_cam &&
         (src->kind == CS_SRC_LOD_BLOCK || src->kind == CS_SRC_CLOUD);
}

static cs_ctx::FrameKey frame_key(const cs_ctx* c, const Ws* w, const cs_source* src, const cs_camera* cam,
                                  const cs_settings* st, void* out, uint32_t flags, cudaStream_t s) {
  cs_ctx::FrameKey k;
  std::memset(&k, 0, sizeof(k));
  std::memcpy(&k.src, src, sizeof(cs_source));
  std::memcpy(&k.st, st, sizeof(cs_settings));
  k.lod_serial = src->kind == CS_SRC_CLOUD ? 0 : src->lod->serial;
  k.width = cam->width;
  k.height = cam->height;
  k.flags = flags;
  k.out = out;
  k.stream = s;
  k.ws = w;
  k.cap_vis = w->cap_vis; k.cap_pairs = w->cap_pairs; k.cap_pw = w->cap_pw; k.cap_tiles = w->cap_tiles;
  k.buf_generation = g_buf_generation.load();
  return k;
}

static bool same_key(const cs_ctx::FrameKey& a, const cs_ctx::FrameKey& b) {
  return std::memcmp(&a, &b, sizeof(a)) == 0;
}

constexpr size_t kMaxGraphs = 4;

// Capture the frame into a graph.  The frame itself was already rendered on
// the caller's stream, so any failure here only means "stay on the direct
// path": the key is remembered as uncapturable and the call succeeds.
static int capture_graph(cs_ctx* c, Ws* w, const cs_source* src, const cs_camera* cam, const cs_settings* st,
                         void* out, uint32_t flags, const cs_ctx::FrameKey& key) {
  auto give_up = [&](cudaGraph_t g) {
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    c->uncapturable.push_back(key);
    if (c->uncapturable.size() > 16) c->uncapturable.erase(c->uncapturable.begin());
    g_err.clear();
    return CS_OK;
  };
  if (!c->capture_stream &&
      cudaStreamCreateWithFlags(&c->capture_stream, cudaStreamNonBlocking) != cudaSuccess)
    return give_up(nullptr);
  if (cudaStreamBeginCapture(c->capture_stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return give_up(nullptr);
  const int64_t serial = c->serial;
  const int rc = render_once(c, w, src, cam, st, out, flags, c->capture_stream);
  c->serial = serial;
  cudaGraph_t g = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(c->capture_stream, &g);
  if (rc || ce != cudaSuccess || !g) return give_up(g);
  cs_ctx::FrameGraph fg;
  fg.key = key;
  fg.graph = g;
  size_t n = 0;
  if (cudaGraphGetNodes(g, nullptr, &n) != cudaSuccess) return give_up(g);
  std::vector<cudaGraphNode_t> nodes(n);
  if (cudaGraphGetNodes(g, nodes.data(), &n) != cudaSuccess) return give_up(g);
  const void* f_sel = lod_select_kernel();
  const void* f_proj = project_kernel();
  const void* f_proj2 = project_staged_kernel();
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nd, &t) != cudaSuccess) return give_up(g);
    if (t != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeParams p;
    if (cudaGraphKernelNodeGetParams(nd, &p) != cudaSuccess) return give_up(g);
    // argument index of the cs_camera (k_lod_select(T, cam, ...),
    // k_project(clouds, segs, stats, cam, ...)) and the argument count
    int cam_arg = -1, n_args = 0;
    if (p.func == f_sel) { cam_arg = 1; n_args = 6; }
    if (p.func == f_proj || p.func == f_proj2) { cam_arg = 3; n_args = 7; }
    if (cam_arg < 0) continue;
    cs_ctx::CamNode cn;
    cn.node = nd;
    cn.params = p;
    cn.args.assign(p.kernelParams, p.kernelParams + n_args);
    cn.cam_arg = cam_arg;
    fg.cam_nodes.push_back(cn);
  }
  if (fg.cam_nodes.empty() || cudaGraphInstantiate(&fg.exec, g, 0) != cudaSuccess) return give_up(g);
  if (c->graphs.size() >= kMaxGraphs) {
    cudaGraphExecDestroy(c->graphs.front().exec);
    cudaGraphDestroy(c->graphs.front().graph);
    c->graphs.erase(c->graphs.begin());
  }
  c->graphs.push_back(std::move(fg));
  return CS_OK;
}

static int replay_graph(cs_ctx* c, cs_ctx::FrameGraph& fg, const cs_camera* cam, cudaStream_t s) {
  c->graph_cam = *cam;
  for (cs_ctx::CamNode& cn : fg.cam_nodes) {
    cn.args[cn.cam_arg] = &c->graph_cam;
    cudaKernelNodeParams p = cn.params;
    p.kernelParams = cn.args.data();
    CS_CUDA(cudaGraphExecKernelNodeSetParams(fg.exec, cn.node, &p));
  }
  CS_CUDA(cudaGraphLaunch(fg.exec, s));
  c->last = reinterpret_cast<Ws*>(const_cast<void*>(fg.key.ws));
  ++c->serial;
  return CS_OK;
}

int cs_frame_graphs(cs_ctx* c) { return c ? (int)c->graphs.size() : 0; }

// The frame pipeline with its overflow handling; KEEP_STATE is internal
// (cs_render_train).
static int render_frame(cs_ctx* c, Ws* w, const cs_source* src, const cs_camera* cam, const cs_settings* st,
                        void* out, uint32_t flags, cs_frame_stats* stats_host, cudaStream_t s) {
  int rc;
  if (graph_eligible(c, src, flags, stats_host)) {
    const cs_ctx::FrameKey key = frame_key(c, w, src, cam, st, out, flags, s);
    for (cs_ctx::FrameGraph& fg : c->graphs)
      if (same_key(key, fg.key)) return replay_graph(c, fg, cam, s);
    rc = render_once(c, w, src, cam, st, out, flags, s);
    if (rc) return rc;
    // capture on the second sighting of a key whose buffers are already sized
    const cs_ctx::FrameKey after = frame_key(c, w, src, cam, st, out, flags, s);
    bool seen = false, bad = false;
    for (const cs_ctx::FrameKey& k : c->seen) seen |= same_key(k, after);
    for (const cs_ctx::FrameKey& k : c->uncapturable) bad |= same_key(k, after);
    if (seen && !bad && same_key(after, key)) return capture_graph(c, w, src, cam, st, out, flags, after);
    c->seen.push_back(after);
    if (c->seen.size() > kMaxGraphs) c->seen.erase(c->seen.begin());
    return CS_OK;
  }
  for (int attempt = 0; attempt < 4; ++attempt) {
    rc = render_once(c, w, src, cam, st, out, flags, s);
    if (rc) return rc;
    if (!(flags & CS_RENDER_SYNC) && !stats_host) return CS_OK;
    rc = fetch_stats(c, w, s);
    if (rc) return rc;
    if (c->h_stats->status & 2) return fail(CS_ERANGE, "no interval covers a block distance");
    if (!(c->h_stats->status & 1)) {
      if (stats_host) *stats_host = *c->h_stats;
      return CS_OK;
    }
    // this frame overflowed (and was synchronised): its own report is handled here
    c->h_overflow[0] = 0;
    c->h_overflow[1] = 0;
    if (!(flags & CS_RENDER_SYNC)) {
      if (stats_host) *stats_host = *c->h_stats;
      w->cap_pairs = std::min<int64_t>((1ll << 30) - 1, c->h_stats->pairs + c->h_stats->pairs / 4 + 1024);
      return fail(CS_ENOMEM, "pair buffer overflow (%lld pairs > %lld); the buffer has been grown",
                  (long long)c->h_stats->pairs, (long long)w->cap_pairs);
    }
    // grow the pair buffers to the observed count and re-run
    w->cap_pairs = std::min<int64_t>((1ll << 30) - 1, c->h_stats->pairs + c->h_stats->pairs / 4 + 1024);
    if (c->h_stats->pairs >= (1ll << 30)) return fail(CS_ENOMEM, "more than 2^30 tile pairs");
  }
  return fail(CS_ECUDA, "pair buffer did not converge");
}

int cs_render(cs_ctx* c, const cs_source* src, const cs_camera* cam, const cs_settings* st,
              void* out, uint32_t flags, cs_frame_stats* stats_host, void* stream) {
  if (!c || !src || !out) return fail(CS_EINVAL, "NULL argument");
  int rc = validate(cam, st);
  if (rc) return rc;
  if (flags & CS_RENDER_KEEP_STATE)
    return fail(CS_EINVAL, "kept-state forwards go through cs_render_train");
  std::lock_guard<std::mutex> lock(c->mu);
  CS_CUDA(cudaSetDevice(c->device));
  rc = check_overflow(c);
  if (rc) return rc;
  Ws* w = nullptr;
  rc = frame_ws(c, &w);
  if (rc) return rc;
  return render_frame(c, w, src, cam, st, out, flags, stats_host, (cudaStream_t)stream);
}

int cs_render_train(cs_ctx* c, const cs_source* src, const cs_camera* cam, const cs_settings* st,
                    float* out_rgb, uint32_t flags, cs_state** state_out, void* stream) {
  if (!c || !src || !out_rgb || !state_out) return fail(CS_EINVAL, "NULL argument");
  *state_out = nullptr;
  int rc = validate(cam, st);
  if (rc) return rc;
  if (src->kind != CS_SRC_CLOUD) return fail(CS_EINVAL, "training renders take a single-cloud source");
  if (src->exclude) return fail(CS_EINVAL, "training renders take no exclude mask");
  if (flags & ~(uint32_t)(CS_RENDER_SYNC | CS_RENDER_NO_CLIP))
    return fail(CS_EINVAL, "cs_render_train accepts CS_RENDER_SYNC and CS_RENDER_NO_CLIP only");
  std::lock_guard<std::mutex> lock(c->mu);
  CS_CUDA(cudaSetDevice(c->device));
  rc = check_overflow(c);
  if (rc) return rc;
  Ws* w = nullptr;
  rc = frame_ws(c, &w);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  rc = render_frame(c, w, src, cam, st, out_rgb, flags | CS_RENDER_KEEP_STATE, nullptr, s);
  if (rc) return rc;
  cs_state* S = new cs_state();
  S->ctx = c;
  S->ws = w;
  S->count = src->cloud.count;
  S->width = cam->width;
  S->height = cam->height;
  S->cam = *cam;
  S->st = *st;
  S->cloud = src->cloud;
  if (cudaMallocHost(&S->h_status, 16) != cudaSuccess ||
      cudaEventCreateWithFlags(&S->done, cudaEventDisableTiming) != cudaSuccess) {
    if (S->h_status) cudaFreeHost(S->h_status);
    delete S;
    return fail(CS_ENOMEM, "state");
  }
  S->h_pairs = reinterpret_cast<int64_t*>(S->h_status + 2);
  DevStats* d = w->stats.as<DevStats>();
  CS_CUDA(cudaMemcpyAsync(S->h_status, &d->status, 4, cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaMemcpyAsync(S->h_pairs, &d->pairs, 8, cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaEventRecord(S->done, s));
  w->held = true;
  *state_out = S;
  return CS_OK;
}

void cs_state_release(cs_state* S) {
  if (!S) return;
  {
    std::lock_guard<std::mutex> lock(S->ctx->mu);
    cudaSetDevice(S->ctx->device);
    // the backward (or anything else) reading the workspace was enqueued on some
    // stream: the next frame into it is ordered after it only by the caller's
    // stream discipline, so wait for the forward's completion at least
    if (S->done) cudaEventSynchronize(S->done);
    S->ws->held = false;
  }
  if (S->done) cudaEventDestroy(S->done);
  if (S->h_status) cudaFreeHost(S->h_status);
  delete S;
}

int cs_render_backward(cs_ctx* c, cs_state* S, const float* dl_dimg, const cs_grads* out,
                       void* stream) {
  if (!c || !S || !out || !dl_dimg) return fail(CS_EINVAL, "NULL argument");
  if (S->ctx != c) return fail(CS_EINVAL, "state belongs to another context");
  std::lock_guard<std::mutex> lock(c->mu);
  CS_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  // The forward's own pair-buffer status: wait for the forward (the loss
  // kernels enqueued after it keep the GPU busy meanwhile) and refuse to
  // differentiate an incomplete frame.
  CS_CUDA(cudaEventSynchronize(S->done));
  if (*S->h_status & 1) {
    Ws* w = S->ws;
    w->cap_pairs = std::min<int64_t>((1ll << 30) - 1, *S->h_pairs + *S->h_pairs / 4 + 1024);
    c->h_overflow[0] = 0;
    c->h_overflow[1] = 0;
    return fail(CS_ENOMEM,
                "the training forward overflowed its pair buffer (%lld pairs); its image and "
                "gradients are invalid -- the buffer has been grown, repeat the step",
                (long long)*S->h_pairs);
  }
  Ws* w = S->ws;
  const cs_cloud& cl = S->cloud;
  const int64_t cap = w->cap_vis;
  if (c->gacc.ensure(sizeof(gacc_t) * 9 * cap)) return fail(CS_ENOMEM, "gradient partials");
  CS_CUDA(cudaMemsetAsync(c->gacc.p, 0, sizeof(gacc_t) * 9 * cap, s));
  const int ts = S->st.tile_size;
  const int ntx = (S->width + ts - 1) / ts;
  BlendState state{w->st_t.as<double>(), w->st_last.as<int32_t>(), w->st_acc.as<double>()};
  launch_blend_bwd(w->last_tiles, w->last_list, w->last_bxs, w->last_bys, w->last_ranges,
                   w->hot.as<HotRec>(), CS_BWD_FAST ? w->fast.as<FastRec>() : nullptr,
                   w->tile_order.as<uint32_t>(), S->st, S->width,
                   S->height, ntx, dl_dimg, state, &w->stats.as<DevStats>()->tickets[5],
                   c->gacc.as<gacc_t>(), cap, s);
  CS_CHECK_LAUNCH();
  // K11 writes every row (zeros for the culled ones): no clear of the outputs.
  // The forward's per-splat float64 depth keys (~0 = culled) are still in keysA.
  launch_project_bwd(cl, w->keysA.as<uint64_t>(), S->cam, S->st, c->gacc.as<gacc_t>(), cap, *out, s);
  CS_CHECK_LAUNCH();
  return CS_OK;
}

int cs_check(cs_ctx* c, void* stream) {
  if (!c) return fail(CS_EINVAL, "NULL argument");
  CS_CUDA(cudaSetDevice(c->device));
  CS_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  std::lock_guard<std::mutex> lock(c->mu);
  return check_overflow(c);
}

int cs_training_loss(cs_ctx* c, const float* img, const float* ref, int32_t height, int32_t width,
                     double lam, double* loss_out, float* grad_out, void* stream) {
  if (!c || !img || !ref || !loss_out || !grad_out) return fail(CS_EINVAL, "NULL argument");
  if (height < 11 || width < 11) return fail(CS_EINVAL, "images must be at least 11x11 for ssim");
  if (!(lam >= 0.0 && lam <= 1.0)) return fail(CS_EINVAL, "lam must be in [0, 1]");
  std::lock_guard<std::mutex> lock(c->mu);
  CS_CUDA(cudaSetDevice(c->device));
  const size_t maps = (size_t)9 * (height - 10) * (((width - 10) + 3) & ~3);  // row pitch mult. of 4
  if (c->loss_maps.ensure(4 * maps) || c->loss_acc.ensure(16)) return fail(CS_ENOMEM, "loss maps");
  launch_training_loss(img, ref, height, width, lam, c->loss_maps.as<float>(),
                       c->loss_acc.as<double>(), loss_out, grad_out, (cudaStream_t)stream);
  CS_CHECK_LAUNCH();
  return CS_OK;
}

int cs_block_adam(cs_ctx* c, int64_t K, int32_t sh_coeffs, float* geom, float* geom_m,
                  float* geom_v, float* sh, float* sh_m, float* sh_v, const cs_grads* grads,
                  const cs_adam_hparams* hp, float* pos_op, float* scale, float* quat,
                  void* stream) {
  if (!c || !grads || !hp || K < 0) return fail(CS_EINVAL, "bad argument");
  if (K > 0 && (!geom || !geom_m || !geom_v || !sh || !sh_m || !sh_v || !pos_op || !scale || !quat))
    return fail(CS_EINVAL, "NULL buffer");
  if (sh_coeffs != 1 && sh_coeffs != 4 && sh_coeffs != 9 && sh_coeffs != 16)
    return fail(CS_EINVAL, "sh_coeffs must be 1, 4, 9 or 16");
  if (hp->step < 1) return fail(CS_EINVAL, "step must be >= 1");
  auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (K > 0 && !(a16(geom) && a16(geom_m) && a16(geom_v) && a16(grads->rotations) && a16(pos_op) &&
                 a16(scale) && a16(quat) && a16(sh) && a16(sh_m) && a16(sh_v) && a16(grads->sh)))
    return fail(CS_EINVAL, "geom, SH, moments, rotation/SH gradients and quads must be 16-byte aligned");
  CS_CUDA(cudaSetDevice(c->device));
  launch_block_adam(K, sh_coeffs, geom, geom_m, geom_v, sh, sh_m, sh_v, *grads, *hp,
                    reinterpret_cast<float4*>(pos_op), reinterpret_cast<float4*>(scale),
                    reinterpret_cast<float4*>(quat), (cudaStream_t)stream);
  CS_CHECK_LAUNCH();
  return CS_OK;
}

int cs_block_activate(cs_ctx* c, int64_t K, const float* geom, float* pos_op, float* scale,
                      float* quat, void* stream) {
  if (!c || K < 0 || (K > 0 && (!geom || !pos_op || !scale || !quat)))
    return fail(CS_EINVAL, "bad argument");
  CS_CUDA(cudaSetDevice(c->device));
  launch_activate_geom(K, geom, reinterpret_cast<float4*>(pos_op), reinterpret_cast<float4*>(scale),
                       reinterpret_cast<float4*>(quat), (cudaStream_t)stream);
  CS_CHECK_LAUNCH();
  return CS_OK;
}

int cs_timing_begin(cs_ctx* c, int32_t max_frames) {
  if (!c || max_frames <= 0) return fail(CS_EINVAL, "bad argument");
  CS_CUDA(cudaSetDevice(c->device));
  const size_t need = (size_t)max_frames * (kStages + 1);
  while (c->tev.size() < need) {
    cudaEvent_t e;
    CS_CUDA(cudaEventCreate(&e));
    c->tev.push_back(e);
  }
  c->timing_max = max_frames;
  c->timing_frame = 0;
  c->timing_on = true;
  return CS_OK;
}

int cs_timing_end(cs_ctx* c, double* stage_ms, int32_t* frames) {
  if (!c || !stage_ms || !frames) return fail(CS_EINVAL, "NULL argument");
  CS_CUDA(cudaSetDevice(c->device));
  c->timing_on = false;
  for (int k = 0; k < kStages; ++k) stage_ms[k] = 0.0;
  for (int f = 0; f < c->timing_frame; ++f) {
    cudaEvent_t* e = &c->tev[(size_t)f * (kStages + 1)];
    CS_CUDA(cudaEventSynchronize(e[kStages]));
    for (int k = 0; k < kStages; ++k) {
      float ms = 0.f;
      CS_CUDA(cudaEventElapsedTime(&ms, e[k], e[k + 1]));
      stage_ms[k] += ms;
    }
  }
  *frames = c->timing_frame;
  return CS_OK;
}

int cs_frame_stats_get(cs_ctx* c, cs_frame_stats* out, void* stream) {
  if (!c || !out) return fail(CS_EINVAL, "NULL argument");
  CS_CUDA(cudaSetDevice(c->device));
  int rc = fetch_stats(c, c->last, (cudaStream_t)stream);
  if (rc) return rc;
  *out = *c->h_stats;
  return CS_OK;
}

int cs_dump_projected(cs_ctx* c, double* means, double* conics, double* covs, double* depths,
                      double* colors, double* opacities, double* radii, int64_t* source,
                      void* stream) {
  if (!c || !c->last || !c->last->last_order) return fail(CS_EINVAL, "no frame rendered");
  if (!c->last->last_debug) return fail(CS_EINVAL, "last frame was not rendered in debug mode");
  CS_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  int rc = fetch_stats(c, c->last, s);
  if (rc) return rc;
  const int64_t M = c->h_stats->visible;
  if (M == 0) return CS_OK;
  const size_t b = sizeof(double) * M;
  if (c->scratch1.ensure(b * 15 + 8 * M)) return fail(CS_ENOMEM, "dump");
  double* base = c->scratch1.as<double>();
  double *dm = base, *dc = dm + 2 * M, *dv = dc + 3 * M, *dd = dv + 3 * M, *dcol = dd + M,
         *dop = dcol + 3 * M, *dr = dop + M;
  int64_t* ds = reinterpret_cast<int64_t*>(dr + 2 * M);
  launch_dump_projected(c->last->last_order, c->last->recs.as<ProjRec>(), c->last->stats.as<DevStats>(), dm, dc, dv,
                        dd, dcol, dop, dr, ds, s);
  CS_CHECK_LAUNCH();
  struct { void* h; void* d; size_t n; } cp[] = {
      {means, dm, 2 * b}, {conics, dc, 3 * b}, {covs, dv, 3 * b}, {depths, dd, b},
      {colors, dcol, 3 * b}, {opacities, dop, b}, {radii, dr, 2 * b}, {source, ds, 8 * (size_t)M}};
  for (auto& x : cp)
    if (x.h) CS_CUDA(cudaMemcpyAsync(x.h, x.d, x.n, cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaStreamSynchronize(s));
  return CS_OK;
}

int cs_dump_tiles(cs_ctx* c, int64_t* tile_ids, int64_t* offsets, void* stream) {
  if (!c || !c->last || !c->last->last_list) return fail(CS_EINVAL, "no frame rendered");
  CS_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  int rc = fetch_stats(c, c->last, s);
  if (rc) return rc;
  const int64_t P = c->h_stats->pairs;
  const int64_t NA = c->h_stats->assembled;  // rank_of is indexed by splat id (assembled index)
  if (c->scratch2.ensure(8 * (P + c->last->last_tiles + 1 + NA))) return fail(CS_ENOMEM, "dump");
  int64_t* dt = c->scratch2.as<int64_t>();
  int64_t* doff = dt + P;
  int64_t* rank_of = doff + c->last->last_tiles + 1;
  launch_dump_tiles(c->last->last_order, c->last->last_list, c->last->last_ranges, c->last->stats.as<DevStats>(),
                    c->last->last_tiles, rank_of, dt, doff, s);
  CS_CHECK_LAUNCH();
  if (tile_ids && P) CS_CUDA(cudaMemcpyAsync(tile_ids, dt, 8 * P, cudaMemcpyDeviceToHost, s));
  if (offsets) CS_CUDA(cudaMemcpyAsync(offsets, doff, 8 * (c->last->last_tiles + 1), cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaStreamSynchronize(s));
  return CS_OK;
}

int cs_dump_segments(cs_ctx* c, int32_t* cloud_index, int64_t* count, int32_t max_n,
                     int32_t* n_out, void* stream) {
  if (!c) return fail(CS_EINVAL, "NULL ctx");
  CS_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  int rc = fetch_stats(c, c->last, s);
  if (rc) return rc;
  const int n = std::min<int>(c->h_stats->n_segments, max_n);
  std::vector<Seg> h(std::max(n, 1));
  if (n) CS_CUDA(cudaMemcpyAsync(h.data(), c->last->segs.p, sizeof(Seg) * n, cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < n; ++i) {
    cloud_index[i] = h[i].cloud;
    count[i] = h[i].count;
  }
  *n_out = n;
  return CS_OK;
}

int cs_dump_assembled_list(cs_ctx* c, uint64_t* packed, int64_t max_n, int64_t* n_out,
                           void* stream) {
  if (!c || !packed || !n_out) return fail(CS_EINVAL, "NULL argument");
  CS_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  int rc = fetch_stats(c, c->last, s);
  if (rc) return rc;
  const int64_t n = std::min<int64_t>(c->h_stats->assembled, max_n);
  if (n > 0 && c->last->pw_list.p)
    CS_CUDA(cudaMemcpyAsync(packed, c->last->pw_list.p, 8 * n, cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaStreamSynchronize(s));
  *n_out = n;
  return CS_OK;
}

// ---------------------------------------------------------------------------
// LoD API mirror

int cs_decide_visibility(cs_ctx* c, const cs_lod* L, const cs_camera* cam, int32_t force_level,
                         cs_decision* out_host, void* stream) {
  if (!c || !L || !cam || !out_host) return fail(CS_EINVAL, "NULL argument");
  std::lock_guard<std::mutex> lock(c->mu);
  CS_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  Ws* w = nullptr;
  int rc = frame_ws(c, &w);
  if (rc) return rc;
  rc = ensure_frame_buffers(w, 1, L->n_levels * L->n_blocks, L->n_blocks, 1, 0);
  if (rc) return rc;
  c->last = w;
  DevStats* stats = w->stats.as<DevStats>();
  CS_CUDA(cudaMemsetAsync(stats, 0, sizeof(DevStats), s));
  launch_lod_select(L->tables(), *cam, force_level, w->dec.as<cs_decision>(), w->segs.as<Seg>(),
                    stats, s);
  CS_CHECK_LAUNCH();
  CS_CUDA(cudaMemcpyAsync(out_host, w->dec.p, sizeof(cs_decision) * L->n_blocks,
                          cudaMemcpyDeviceToHost, s));
  rc = fetch_stats(c, w, s);
  if (rc) return rc;
  if (c->h_stats->status & 2) return fail(CS_ERANGE, "no interval covers a block distance");
  return CS_OK;
}

int cs_block_visible(cs_ctx* c, int32_t n, const double* bmin, const double* bmax,
                     const cs_camera* cam, uint8_t* vis, double* dist, void* stream) {
  if (!c || !cam || n < 0) return fail(CS_EINVAL, "bad argument");
  if (n == 0) return CS_OK;
  std::lock_guard<std::mutex> lock(c->mu);
  CS_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (c->scratch3.ensure(64 * (size_t)n)) return fail(CS_ENOMEM, "scratch");
  double* db = c->scratch3.as<double>();
  double* dmax = db + 3 * n;
  double* dd = dmax + 3 * n;
  uint8_t* dv = reinterpret_cast<uint8_t*>(dd + n);
  CS_CUDA(cudaMemcpyAsync(db, bmin, 24 * (size_t)n, cudaMemcpyHostToDevice, s));
  CS_CUDA(cudaMemcpyAsync(dmax, bmax, 24 * (size_t)n, cudaMemcpyHostToDevice, s));
  launch_block_visible(n, db, dmax, *cam, dv, dd, s);
  CS_CHECK_LAUNCH();
  CS_CUDA(cudaMemcpyAsync(vis, dv, n, cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaMemcpyAsync(dist, dd, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaStreamSynchronize(s));
  return CS_OK;
}

int cs_select_level(cs_ctx* c, int32_t n, const double* d, int32_t ni, const double* iv,
                    int32_t* out, void* stream) {
  if (!c || n < 0 || ni <= 0) return fail(CS_EINVAL, "bad argument");
  if (n == 0) return CS_OK;
  std::lock_guard<std::mutex> lock(c->mu);
  CS_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (c->scratch4.ensure(8 * (size_t)n + 16 * (size_t)ni + 4 * (size_t)n)) return fail(CS_ENOMEM, "scratch");
  double* dd = c->scratch4.as<double>();
  double* div = dd + n;
  int32_t* dout = reinterpret_cast<int32_t*>(div + 2 * ni);
  CS_CUDA(cudaMemcpyAsync(dd, d, 8 * (size_t)n, cudaMemcpyHostToDevice, s));
  CS_CUDA(cudaMemcpyAsync(div, iv, 16 * (size_t)ni, cudaMemcpyHostToDevice, s));
  launch_select_level(n, dd, ni, div, dout, s);
  CS_CHECK_LAUNCH();
  CS_CUDA(cudaMemcpyAsync(out, dout, 4 * (size_t)n, cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < n; ++i) {
    if (out[i] == -2) return fail(CS_EINVAL, "distance must be nonnegative");
    if (out[i] == -1) return fail(CS_ERANGE, "no interval covers distance %g", d[i]);
  }
  return CS_OK;
}

// ---------------------------------------------------------------------------
// reference-kernel mirror and core utilities

int cs_blend_tiles(cs_ctx* c, const int64_t* tile_ids, const int64_t* tile_offsets,
                   int64_t n_tiles, const double* means, const double* conics,
                   const double* colors, const double* opacities, int64_t n_splats,
                   const double* background, int32_t tile_size, int32_t width, int32_t height,
                   int32_t n_tiles_x, double alpha_floor, double t_floor, double* out,
                   int64_t* fragments, void* stream) {
  if (!c || !tile_offsets || !out || !fragments || !background)
    return fail(CS_EINVAL, "NULL argument");
  if (tile_size < 8 || blend_ppt(tile_size) == 0) return fail(CS_EINVAL, "tile_size");
  std::lock_guard<std::mutex> lock(c->mu);
  CS_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  int64_t P = 0;
  CS_CUDA(cudaMemcpyAsync(&P, tile_offsets + n_tiles, 8, cudaMemcpyDeviceToHost, s));
  double bg[3];
  CS_CUDA(cudaMemcpyAsync(bg, background, 24, cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaStreamSynchronize(s));
  const int64_t m = std::max<int64_t>(n_splats, 1);
  Ws* w = nullptr;
  int rc = frame_ws(c, &w);
  if (rc) return rc;
  if (c->scratch1.ensure(sizeof(HotRec) * m) ||
      c->scratch2.ensure(12 * std::max<int64_t>(P, 1) + sizeof(uint2) * n_tiles + 4 * n_tiles + 8))
    return fail(CS_ENOMEM, "blend scratch");
  HotRec* hot = c->scratch1.as<HotRec>();
  uint32_t* list = c->scratch2.as<uint32_t>();
  uint32_t* pbx = list + std::max<int64_t>(P, 1);
  uint32_t* pby = pbx + std::max<int64_t>(P, 1);
  uint2* ranges = reinterpret_cast<uint2*>(pby + std::max<int64_t>(P, 1));
  // keep uint2 8-byte aligned
  ranges = reinterpret_cast<uint2*>((reinterpret_cast<uintptr_t>(ranges) + 7) & ~uintptr_t(7));
  int32_t* ftile = reinterpret_cast<int32_t*>(ranges + n_tiles);
  launch_pack(n_splats, means, conics, colors, opacities, alpha_floor, hot, P, tile_ids,
              n_tiles, tile_offsets, list, pbx, pby, ranges, s);
  CS_CHECK_LAUNCH();
  CS_CUDA(cudaMemsetAsync(w->stats.p, 0, sizeof(DevStats), s));
  BlendParams bp;
  for (int i = 0; i < 3; ++i) bp.bg[i] = bg[i];
  bp.alpha_floor = alpha_floor;
  bp.t_floor = t_floor;
  bp.tile_size = tile_size;
  bp.width = width;
  bp.height = height;
  bp.ntx = n_tiles_x;
  bp.flags = CS_RENDER_NO_CLIP;
  launch_blend((int)n_tiles, list, pbx, pby, ranges, hot, nullptr, nullptr, bp, out, true, ftile, w->stats.as<DevStats>(),
               nullptr, s);
  CS_CHECK_LAUNCH();
  // fragments: int32 per tile -> int64
  std::vector<int32_t> h(n_tiles);
  std::vector<int64_t> h64(n_tiles);
  CS_CUDA(cudaMemcpyAsync(h.data(), ftile, 4 * n_tiles, cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaStreamSynchronize(s));
  for (int64_t t = 0; t < n_tiles; ++t) h64[t] = h[t];
  CS_CUDA(cudaMemcpy(fragments, h64.data(), 8 * n_tiles, cudaMemcpyHostToDevice));
  return CS_OK;
}

int cs_build_covariances(cs_ctx* c, int64_t n, const double* scales, const double* quats,
                         double* out, void* stream) {
  if (!c || n < 0) return fail(CS_EINVAL, "bad argument");
  CS_CUDA(cudaSetDevice(c->device));
  launch_build_covariances(n, scales, quats, out, (cudaStream_t)stream);
  CS_CHECK_LAUNCH();
  return CS_OK;
}

int cs_sh_to_colors(cs_ctx* c, int64_t n, const double* sh, int32_t coeffs, const double* dirs,
                    int32_t degree, double* out, void* stream) {
  if (!c || n < 0) return fail(CS_EINVAL, "bad argument");
  if (degree < 0 || degree > 3) return fail(CS_EINVAL, "degree must be 0..3");
  if ((degree + 1) * (degree + 1) > coeffs) return fail(CS_EINVAL, "sh narrower than degree");
  CS_CUDA(cudaSetDevice(c->device));
  launch_sh_to_colors(n, sh, coeffs, dirs, degree, out, (cudaStream_t)stream);
  CS_CHECK_LAUNCH();
  return CS_OK;
}

int cs_block_of_points(cs_ctx* c, int64_t n, const void* positions, int32_t f32,
                       const double* p_min, const double* p_max, int32_t nx, int32_t ny,
                       int32_t nz, int32_t* out, void* stream) {
  if (!c || n < 0 || nx < 1 || ny < 1 || nz < 1) return fail(CS_EINVAL, "bad argument");
  CS_CUDA(cudaSetDevice(c->device));
  launch_block_of_points(n, positions, f32, p_min, p_max, nx, ny, nz, out, (cudaStream_t)stream);
  CS_CHECK_LAUNCH();
  return CS_OK;
}

int cs_fuse_filter(cs_ctx* c, int64_t n, const void* positions, int32_t f32, const double* p_min,
                   const double* p_max, int32_t nx, int32_t ny, int32_t nz, int32_t block,
                   int64_t* kept_idx, int64_t* kept_count, void* stream) {
  if (!c || n < 0 || nx < 1 || ny < 1 || nz < 1) return fail(CS_EINVAL, "bad argument");
  std::lock_guard<std::mutex> lock(c->mu);
  CS_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t chunks = (n + 255) / 256 + 1;
  if (c->st_fuse.ensure(8 * chunks)) return fail(CS_ENOMEM, "fuse status");
  CS_CUDA(cudaMemsetAsync(c->st_fuse.p, 0, 8 * chunks, s));
  CS_CUDA(cudaMemsetAsync(c->fuse_ticket.p, 0, 4, s));
  launch_fuse_filter(n, positions, f32, p_min, p_max, nx, ny, nz, block, c->st_fuse.as<uint64_t>(),
                     c->fuse_ticket.as<uint32_t>(), kept_idx, kept_count, s);
  CS_CHECK_LAUNCH();
  return CS_OK;
}

// ---- LoD generation (lod.py:54-248) ------------------------------------------

static int check_cloud(const cs_cloud* cl) {
  if (!cl || cl->count < 0) return fail(CS_EINVAL, "bad cloud descriptor");
  if (cl->count > 0 && (!cl->pos_op || !cl->scale || !cl->quat))
    return fail(CS_EINVAL, "bad cloud descriptor");
  if (cl->count >= (1ll << 32)) return fail(CS_EINVAL, "more than 2^32 Gaussians");
  return CS_OK;
}

int cs_significance(cs_ctx* c, const cs_cloud* cloud, const cs_camera* cams, int32_t n_cams,
                    const cs_settings* st, double* scores, int32_t* hits, void* stream) {
  if (!c || !st || !scores || n_cams < 0 || (n_cams > 0 && !cams)) return fail(CS_EINVAL, "bad argument");
  int rc = check_cloud(cloud);
  if (rc) return rc;
  CS_CUDA(cudaSetDevice(c->device));
  CS_CUDA(significance_run(*cloud, cams, n_cams, *st, scores, hits, (cudaStream_t)stream));
  return CS_OK;
}

int cs_priority(cs_ctx* c, int64_t n, const double* scores, int32_t* order, void* stream) {
  if (!c || n < 0 || (n > 0 && (!scores || !order))) return fail(CS_EINVAL, "bad argument");
  if (n >= (1ll << 32)) return fail(CS_EINVAL, "more than 2^32 scores");
  CS_CUDA(cudaSetDevice(c->device));
  CS_CUDA(priority_run(n, scores, order, (cudaStream_t)stream));
  return CS_OK;
}

int cs_lod_rows(cs_ctx* c, int64_t n, const int32_t* order, const int32_t* membership,
                int32_t n_blocks, const double* rates, int32_t n_levels, int32_t* rows,
                int64_t* counts, void* stream) {
  if (!c || n < 0 || n_blocks < 1 || n_blocks > 4096 || n_levels < 1 || !rates || !counts)
    return fail(CS_EINVAL, "bad argument");
  if (n > 0 && (!order || !membership || !rows)) return fail(CS_EINVAL, "bad argument");
  if (n >= (1ll << 32)) return fail(CS_EINVAL, "more than 2^32 Gaussians");
  std::vector<int64_t> keep(n_levels);
  for (int L = 0; L < n_levels; ++L) {  // _keep_count, lod.py:104-111
    const double r = rates[L];
    if (!(r > 0.0 && r <= 1.0)) return fail(CS_EINVAL, "compression rate must be in (0, 1]");
    const double k = (double)n;
    keep[L] = n == 0 ? 0 : std::min<int64_t>(n, std::max<int64_t>(1, (int64_t)std::ceil(r * k - 1e-9 * k)));
  }
  CS_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  int64_t* dcounts = nullptr;
  CS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dcounts), sizeof(int64_t) * n_levels * n_blocks, s));
  CS_CUDA(cudaMemsetAsync(dcounts, 0, sizeof(int64_t) * n_levels * n_blocks, s));
  CS_CUDA(lod_rows_run(n, order, membership, n_blocks, keep.data(), n_levels, rows, dcounts, s));
  CS_CUDA(cudaMemcpyAsync(counts, dcounts, sizeof(int64_t) * n_levels * n_blocks,
                          cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaFreeAsync(dcounts, s));
  CS_CUDA(cudaStreamSynchronize(s));
  return CS_OK;
}

int cs_mad_bounds(cs_ctx* c, const cs_cloud* cloud, const int32_t* membership, int32_t n_blocks,
                  double n_mad, double* bmin, double* bmax, void* stream) {
  if (!c || n_blocks < 1 || n_blocks > 4096 || !bmin || !bmax) return fail(CS_EINVAL, "bad argument");
  if (!(n_mad > 0)) return fail(CS_EINVAL, "n_mad must be positive");
  int rc = check_cloud(cloud);
  if (rc) return rc;
  if (cloud->count > 0 && !membership) return fail(CS_EINVAL, "bad argument");
  CS_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  double *db = nullptr;
  CS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&db), sizeof(double) * 6 * n_blocks, s));
  CS_CUDA(cudaMemsetAsync(db, 0, sizeof(double) * 6 * n_blocks, s));
  std::vector<int64_t> cnt(n_blocks, 0);
  if (cloud->count > 0)
    CS_CUDA(mad_bounds_run(*cloud, membership, n_blocks, n_mad, db, db + 3 * n_blocks, cnt.data(), s));
  CS_CUDA(cudaMemcpyAsync(bmin, db, sizeof(double) * 3 * n_blocks, cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaMemcpyAsync(bmax, db + 3 * n_blocks, sizeof(double) * 3 * n_blocks, cudaMemcpyDeviceToHost, s));
  CS_CUDA(cudaFreeAsync(db, s));
  CS_CUDA(cudaStreamSynchronize(s));
  return CS_OK;
}

int cs_gather_cloud(cs_ctx* c, const cs_cloud* src, const int32_t* rows, int64_t n,
                    const cs_cloud* dst, void* stream) {
  if (!c || !dst || n < 0 || (n > 0 && !rows)) return fail(CS_EINVAL, "bad argument");
  int rc = check_cloud(src);
  if (rc) return rc;
  if (dst->fp64 != src->fp64) return fail(CS_EINVAL, "source and destination precision differ");
  if (n > 0 && (!dst->pos_op || !dst->scale || !dst->quat || !dst->sh || !src->sh))
    return fail(CS_EINVAL, "bad destination descriptor");
  if (dst->sh_coeffs < 1 || dst->sh_stride < 3 * dst->sh_coeffs) return fail(CS_EINVAL, "bad sh layout");
  CS_CUDA(cudaSetDevice(c->device));
  launch_gather_cloud(*src, rows, n, *dst, (cudaStream_t)stream);
  CS_CHECK_LAUNCH();
  return CS_OK;
}

// ---- training-data assignment (partition.py:172-439) -------------------------

int cs_bounds_contain(cs_ctx* c, int64_t n, const void* positions, int32_t f32, int32_t stride,
                      const double* p_min, const double* p_max, const double* lo, const double* hi,
                      uint8_t* mask, int64_t* count, void* stream) {
  if (!c || n < 0 || !lo || !hi || (stride != 3 && stride != 4) || (n > 0 && !positions) ||
      (!p_min) != (!p_max))
    return fail(CS_EINVAL, "bad argument");
  CS_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  std::lock_guard<std::mutex> lock(c->mu);
  if (c->scratch4.ensure(sizeof(unsigned long long))) return fail(CS_ENOMEM, "count");
  launch_bounds_contain(n, positions, f32, stride, p_min, p_max, lo, hi, mask,
                        c->scratch4.as<unsigned long long>(), s);
  CS_CHECK_LAUNCH();
  if (count) {
    unsigned long long h = 0;
    CS_CUDA(cudaMemcpyAsync(&h, c->scratch4.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    CS_CUDA(cudaStreamSynchronize(s));
    *count = (int64_t)h;
  }
  return CS_OK;
}

int cs_ssim(cs_ctx* c, const float* img_a, const float* img_b, int32_t height, int32_t width,
            const double* window, double* acc4, void* stream) {
  if (!c || !img_a || !img_b || !window || !acc4) return fail(CS_EINVAL, "NULL argument");
  if (height < 11 || width < 11) return fail(CS_EINVAL, "images must be at least 11x11 for ssim");
  CS_CUDA(cudaSetDevice(c->device));
  CS_CUDA(ssim_run(img_a, img_b, height, width, window, acc4, (cudaStream_t)stream));
  return CS_OK;
}

int cs_measure_fp64_peak(cs_ctx* c, double* tflops, void* stream) {
  if (!c || !tflops) return fail(CS_EINVAL, "NULL argument");
  CS_CUDA(cudaSetDevice(c->device));
  CS_CUDA(fp64_peak_run(tflops, (cudaStream_t)stream));
  return CS_OK;
}

}  // extern "C"

// capi.cu — the C-ABI (include/isg.h): context, device buffers, frame orchestration.
//
// A context owns one stream and every device buffer; a frame is launched entirely
// asynchronously (K1 -> depth sort -> scan/emit -> tile sort -> ranges -> blend), the key
// count never travels to the host inside a frame: kernels read it from device memory and the
// blend kernels skip the frame if the preallocated key capacity overflowed.  Host-synchronous
// entry points (isg_render, isg_loss_backward, isg_read_loss, isg_synchronize) check the
// overflow and validation flags, grow the capacity and re-run the frame when needed.
//
// Errors mirror the reference: invalid splats/cameras -> ISG_E_DOMAIN with the message the
// reference's std::domain_error carries (src/splat3d.cpp:10-37); bad arguments ->
// ISG_E_ARG (std::invalid_argument, include/isosplat/particles.hpp:73-83).
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "isg_internal.cuh"
#include "pdl.cuh"

// Stage timing (isg_profile_*): CUDA events around each kernel of a frame, on the launching
// stream, so bench.py can report the dominant kernel's live launch duration.
enum Stage {
  ST_RESET, ST_PREPROCESS, ST_DEPTH_SORT, ST_SCAN_EMIT, ST_TILE_SCAN, ST_FILL, ST_TILE_SORT,
  ST_BLEND_FWD, ST_BLEND_BWD, ST_LOSS_REDUCE, ST_PROJECT_BWD, ST_PROJECT_ADAM, ST_ADAM,
  ST_ALLREDUCE, ST_IMAGE_LOSS, ST_COUNT
};
static const char* kStageNames[ST_COUNT] = {
    "frame_reset", "preprocess", "depth_sort", "scan_emit", "tile_scan", "fill", "tile_sort",
    "blend_fwd", "blend_bwd", "loss_reduce", "project_bwd", "project_adam", "adam",
    "allreduce", "image_loss"};


struct isg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t copy_stream = nullptr;  // host<->device uploads overlapped with compute
  cudaEvent_t ev_main = nullptr, ev_copy = nullptr;
  // target ring for host-buffer training (isg_upload_target_async / isg_loss_backward_slot):
  // per slot the device image, the event of its last upload and of the last frame that read it
  float* tring[ISG_TARGET_SLOTS] = {};
  size_t tring_floats[ISG_TARGET_SLOTS] = {};
  cudaEvent_t ev_tup[ISG_TARGET_SLOTS] = {}, ev_tread[ISG_TARGET_SLOTS] = {};
  bool tring_read[ISG_TARGET_SLOTS] = {};
  // image ring for host-buffer rendering (isg_render_host_async / isg_image_wait)
  float* iring[ISG_IMAGE_SLOTS] = {};
  size_t iring_floats[ISG_IMAGE_SLOTS] = {};
  cudaEvent_t ev_irend[ISG_IMAGE_SLOTS] = {}, ev_icopy[ISG_IMAGE_SLOTS] = {};
  bool iring_copied[ISG_IMAGE_SLOTS] = {};
  std::string err;

  // scene (SoA float4) and Adam moments (n x 2 float4 each)
  int64_t n = 0, n_alloc = 0;
  float4* ms = nullptr;
  float4* co = nullptr;
  float4* m = nullptr;
  float4* v = nullptr;
  float2* raw = nullptr;  // optimizer space: (log sigma, logit opacity) per splat
  int64_t adam_t = 0;

  // per-splat work buffers
  isg::RenderRec* rec = nullptr;  // 32-B render record per splat
  uint32_t* ntiles = nullptr;     // tiles touched per splat
  uint32_t* slot_off = nullptr;   // start of splat g's gradient-slot list
  float4* gradx = nullptr;        // [kMaxRanks exchange slots | grad3d]: one all-reduce buffer
  float4* grad3d = nullptr;       // n x 2, indexed by splat (= gradx + kMaxRanks)
  float* grad2d = nullptr;        // n x 8 direct-mode 2D gradient sums (zero between views)
  bool deterministic = false;     // slot mode (bitwise deterministic) instead of direct mode
  bool pending_direct = false;    // the pending view's K7 ran in direct mode
  uint2* tilebox = nullptr;                 // compact tile bbox + hit mask per splat
  uint32_t* depth[2] = {nullptr, nullptr};  // depth keys (+ radix ping-pong) / depth order
  uint32_t* order[2] = {nullptr, nullptr};
  int order_buf = 0;

  // (tile, splat) pairs, key_cap slots
  int binning = isg::kBinRadix;
  int64_t key_cap = 0;
  uint2* sorted = nullptr;                  // per list entry: (splat, gradient slot)
  uint16_t* submask = nullptr;              // per list entry: sub-quarters reached (16 bits)
  float4* partial = nullptr;                // gradient slot: 2D grads of one pair (2 x float4)
  unsigned long long* bucket = nullptr;     // tile-bucket mode: (depth << 32 | splat), unsorted
  uint32_t* slot_of = nullptr;              // tile-bucket mode: slot lists per splat
  uint32_t* tkey[2] = {nullptr, nullptr};   // radix mode: tile keys
  uint32_t* tval[2] = {nullptr, nullptr};   // radix mode: emission indices
  uint32_t* emit_gid = nullptr;             // radix mode: splat of emission index e
  bool radix_alloc = false;
  uint64_t buf_gen = 0;                     // bumped whenever a device buffer is reallocated
  isg::AdaptScratch* adapt = nullptr;       // adaptive control's persistent scratch

  // sort / scan scratch
  isg::SortScratch sort{};  // adaptive control (zeroed per call)
  int64_t sort_tiles_alloc = 0;
  // per-frame scratch, ONE allocation zeroed by ONE memset per frame: [scan look-back words |
  // depth-sort hist+counters | tile-sort hist+counters | depth-sort look-back | tile-sort
  // look-back]
  unsigned char* arena = nullptr;
  size_t arena_bytes = 0;
  int64_t arena_n = -1, arena_cap = -1;
  size_t arena_depth_end = 0;  // bytes to zero when only the depth sort runs (tile-bucket)
  unsigned long long* scan_scratch = nullptr;  // = arena
  isg::SortScratch sort_depth{}, sort_tile{};

  // pixels / tiles
  int64_t pix_alloc = 0, tiles_alloc = 0;
  float* img = nullptr;
  float* target = nullptr;
  float* t_last = nullptr;
  uint32_t* n_proc = nullptr;
  uint2* ranges = nullptr;
  uint32_t* tile_cnt = nullptr;
  uint32_t* cursor = nullptr;
  double* tile_loss = nullptr;

  // image loss: ISG_LOSS_L2 (fused into K7) or ISG_LOSS_L1_DSSIM (k_ssim.cu -> dL/dC -> K7)
  int loss_kind = ISG_LOSS_L2;
  float lambda = 0.2f;
  int64_t ssim_pix_alloc = 0, ssim_part_alloc = 0;
  float* coef = nullptr;       // 9 W H gradient-coefficient planes
  float* dldc = nullptr;       // dL/dC, HWC3
  double2* ssim_part = nullptr;

  // device scalars: [0] n_keys [1] first_bad [2] n_visible [3] scan tile counter [4] n
  uint32_t* sc = nullptr;
  unsigned long long* total = nullptr;     // isg::TotalWord: keys, skipped, overflow record
  double* loss = nullptr;                  // [0] accumulated, [1] last view, [2] last step
  isg::AdamState* adam_state = nullptr;    // [0] live, [1] snapshot (step counter on device)
  // pinned readback
  uint32_t* h_sc = nullptr;
  unsigned long long* h_total = nullptr;
  double* h_loss = nullptr;

  // frame state
  bool have_frame = false;
  bool last_tracked = false;  // the last frame recorded t_last / n_proc
  isg::FrameParams last_fp{};
  bool pending = false;  // `partial` holds an un-projected view
  isg::FrameParams pending_fp{};
  bool grad3d_valid = false;
  bool frame_unchecked = false;  // frames launched since the last overflow check

  // stats
  int64_t n_keys = 0, n_visible = 0, regrow = 0, launches = 0, overflowed_frames = 0;

  // snapshot of (scene, Adam moments, step) for reject-and-retry optimisation
  float4* snap = nullptr;  // ms | co | m (2n) | v (2n)
  int64_t snap_n = 0, snap_t = 0;
  bool snap_valid = false;

  // NCCL (multi-GPU exchange, see isg_adam_step)
  void* nccl_comm = nullptr;
  bool own_comm = false;  // false: attached with isg_nccl_attach, the caller destroys it
  int nranks = 1, rank = 0;
  int exchange_chunks = 4;                 // pipelined chunks of the gradient exchange
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_grad[isg::kMaxExchangeChunks] = {}, ev_red[isg::kMaxExchangeChunks] = {};

  // CUDA-graph capture of the context stream (isg_graph_*)
  bool capturing = false;
  int64_t capture_launches0 = 0;
  uint64_t capture_gen0 = 0;

  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_used;
  double prof_ms[ST_COUNT] = {};
  int64_t prof_calls[ST_COUNT] = {};
};

namespace {
cudaEvent_t prof_event(isg_ctx* c) {
  if (c->ev_pool.empty()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = c->ev_pool.back();
  c->ev_pool.pop_back();
  return e;
}
struct StageScope {
  isg_ctx* c;
  int stage;
  cudaEvent_t a = nullptr;
  StageScope(isg_ctx* c_, int s) : c(c_), stage(s) {
    if (c->prof && !c->capturing) {
      a = prof_event(c);
      cudaEventRecord(a, c->stream);
    }
  }
  ~StageScope() {
    if (a) {
      cudaEvent_t b = prof_event(c);
      cudaEventRecord(b, c->stream);
      c->ev_used.push_back({stage, {a, b}});
    }
  }
};
}  // namespace
#define ISG_STAGE(st) StageScope stage_scope_##st(ctx, st)

namespace {

using isg::FrameParams;

isg_status fail(isg_ctx* c, isg_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}

// Host-synchronising entry points cannot run inside a stream capture.
#define ISG_NO_CAPTURE(name)                                                               \
  do {                                                                                     \
    if (ctx->capturing)                                                                    \
      return fail(ctx, ISG_E_STATE, name ": synchronising call inside isg_graph_begin/end"); \
  } while (0)

isg_status cuda_fail(isg_ctx* c, cudaError_t e, const char* where) {
  return fail(c, e == cudaErrorMemoryAllocation ? ISG_E_OOM : ISG_E_CUDA,
              std::string(where) + ": " + cudaGetErrorString(e));
}

#define ISG_CUDA(call)                                   \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
  } while (0)

#define ISG_CHECK_LAUNCH()                                         \
  do {                                                             \
    cudaError_t e_ = cudaGetLastError();                           \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, "kernel launch"); \
  } while (0)

template <class T>
cudaError_t realloc_dev(isg_ctx* ctx, T** p, size_t count, bool graph_visible = true) {
  // captured graphs hold the old pointers (isg_graph_launch checks the generation); buffers
  // no graph-captured kernel touches (the snapshot) pass graph_visible = false
  if (graph_visible) ctx->buf_gen++;
  if (*p) cudaFree(*p);
  *p = nullptr;
  if (count == 0) count = 1;
  return cudaMalloc((void**)p, sizeof(T) * count);
}

// initial key capacity for a scene of n splats (grown on overflow up to kMaxItems)
int64_t default_key_cap(int64_t n) {
  return std::min<int64_t>(std::max<int64_t>(6 * n, 1 << 20), isg::kMaxItems);
}

int bits_for(int64_t v) {  // bits needed to represent values in [0, v)
  int b = 1;
  while (b < 32 && (int64_t(1) << b) < v) ++b;
  return b;
}

isg_status ensure_scene(isg_ctx* ctx, int64_t n) {
  if (n <= ctx->n_alloc) return ISG_OK;
  const int64_t a = std::max<int64_t>(n, 1);
  ISG_CUDA(realloc_dev(ctx, &ctx->ms, a));
  ISG_CUDA(realloc_dev(ctx, &ctx->co, a));
  ISG_CUDA(realloc_dev(ctx, &ctx->m, 2 * a));
  ISG_CUDA(realloc_dev(ctx, &ctx->v, 2 * a));
  ISG_CUDA(realloc_dev(ctx, &ctx->raw, a));
  ISG_CUDA(realloc_dev(ctx, &ctx->grad2d, 8 * a));
  ISG_CUDA(cudaMemset(ctx->grad2d, 0, sizeof(float) * 8 * a));
  ISG_CUDA(realloc_dev(ctx, &ctx->rec, a));
  ISG_CUDA(realloc_dev(ctx, &ctx->ntiles, a));
  ISG_CUDA(realloc_dev(ctx, &ctx->slot_off, a));
  ISG_CUDA(realloc_dev(ctx, &ctx->gradx, 2 * a + isg::kMaxRanks));
  ctx->grad3d = ctx->gradx + isg::kMaxRanks;
  ISG_CUDA(realloc_dev(ctx, &ctx->tilebox, a));
  for (int i = 0; i < 2; ++i) {
    ISG_CUDA(realloc_dev(ctx, &ctx->depth[i], a));
    ISG_CUDA(realloc_dev(ctx, &ctx->order[i], a));
  }
  ctx->n_alloc = a;
  return ISG_OK;
}

// The per-frame scratch arena for a scene of n_alloc splats and key_cap pairs.
isg_status ensure_arena(isg_ctx* ctx) {
  if (ctx->arena && ctx->arena_n == ctx->n_alloc && ctx->arena_cap == ctx->key_cap) return ISG_OK;
  const int64_t a = std::max<int64_t>(ctx->n_alloc, 1), cap = std::max<int64_t>(ctx->key_cap, 1);
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t scan = align(sizeof(unsigned long long) *
                            (std::max(isg::scan_emit_scratch_words(a), isg::fill_scratch_words(a)) + 1));
  const size_t hist = align(sizeof(uint32_t) * (isg::kMaxPasses * 256 + isg::kMaxPasses + 1));
  const size_t lb_depth = align(isg::sort_lookback_bytes(a, isg::kMaxPasses));
  const size_t lb_tile = align(isg::sort_lookback_bytes(cap, isg::kMaxPasses));
  const size_t bytes = scan + 2 * hist + lb_depth + lb_tile;
  if (ctx->arena) cudaFree(ctx->arena);
  ctx->arena = nullptr;
  ctx->buf_gen++;
  ISG_CUDA(cudaMalloc(&ctx->arena, bytes));
  ISG_CUDA(cudaMemset(ctx->arena, 0, bytes));
  ctx->arena_bytes = bytes;
  ctx->arena_n = ctx->n_alloc;
  ctx->arena_cap = ctx->key_cap;
  unsigned char* p = ctx->arena;
  ctx->scan_scratch = reinterpret_cast<unsigned long long*>(p);
  auto carve = [&](isg::SortScratch& ss, size_t hist_off, size_t lb_off, int64_t items) {
    ss.hist = reinterpret_cast<uint32_t*>(p + hist_off);
    ss.counters = ss.hist + isg::kMaxPasses * 256;
    ss.lookback = reinterpret_cast<uint32_t*>(p + lb_off);
    ss.max_tiles = std::max<int64_t>(isg::sort_tiles_for(items), 1);
  };
  carve(ctx->sort_depth, scan, scan + 2 * hist, a);
  carve(ctx->sort_tile, scan + hist, scan + 2 * hist + lb_depth, cap);
  ctx->arena_depth_end = scan + 2 * hist + lb_depth;
  return ISG_OK;
}

isg_status ensure_sort_scratch(isg_ctx* ctx, int64_t cap) {
  const int64_t tiles = isg::sort_tiles_for(cap);
  if (tiles <= ctx->sort_tiles_alloc && ctx->sort.hist) return ISG_OK;
  const int64_t t = std::max<int64_t>(tiles, 1);
  ISG_CUDA(realloc_dev(ctx, &ctx->sort.hist, isg::kMaxPasses * 256));
  ISG_CUDA(realloc_dev(ctx, &ctx->sort.counters, isg::kMaxPasses + 1));
  ISG_CUDA(realloc_dev(ctx, &ctx->sort.lookback, (size_t)isg::kMaxPasses * isg::sort_lookback_words(t)));
  ctx->sort.max_tiles = t;
  ctx->sort_tiles_alloc = t;
  return ISG_OK;
}

isg_status ensure_keys(isg_ctx* ctx, int64_t cap) {
  if (cap <= ctx->key_cap) return ISG_OK;
  ISG_CUDA(realloc_dev(ctx, &ctx->sorted, cap));
  ISG_CUDA(realloc_dev(ctx, &ctx->submask, cap));
  ISG_CUDA(realloc_dev(ctx, &ctx->partial, 2 * cap));
  ISG_CUDA(realloc_dev(ctx, &ctx->bucket, cap));
  ISG_CUDA(realloc_dev(ctx, &ctx->slot_of, cap));
  if (ctx->radix_alloc) {
    for (int i = 0; i < 2; ++i) {
      ISG_CUDA(realloc_dev(ctx, &ctx->tkey[i], cap));
      ISG_CUDA(realloc_dev(ctx, &ctx->tval[i], cap));
    }
    ISG_CUDA(realloc_dev(ctx, &ctx->emit_gid, cap));
  }
  ctx->key_cap = cap;
  return ISG_OK;
}

// Radix binning needs its own buffers (allocated on first use).
isg_status ensure_radix(isg_ctx* ctx) {
  if (ctx->radix_alloc) return ISG_OK;
  ctx->radix_alloc = true;
  const int64_t cap = ctx->key_cap;
  if (cap > 0) {
    for (int i = 0; i < 2; ++i) {
      ISG_CUDA(realloc_dev(ctx, &ctx->tkey[i], cap));
      ISG_CUDA(realloc_dev(ctx, &ctx->tval[i], cap));
    }
    ISG_CUDA(realloc_dev(ctx, &ctx->emit_gid, cap));
  }
  return ISG_OK;
}

isg_status ensure_pixels(isg_ctx* ctx, int W, int H) {
  const int64_t pix = (int64_t)W * H;
  const int64_t tiles =
      (int64_t)((W + isg::kTile - 1) / isg::kTile) * ((H + isg::kTile - 1) / isg::kTile);
  if (pix > ctx->pix_alloc) {
    ISG_CUDA(realloc_dev(ctx, &ctx->img, 3 * pix));
    ISG_CUDA(realloc_dev(ctx, &ctx->target, 3 * pix));
    ISG_CUDA(realloc_dev(ctx, &ctx->t_last, pix));
    ISG_CUDA(realloc_dev(ctx, &ctx->n_proc, pix));
    ctx->pix_alloc = pix;
  }
  if (tiles > ctx->tiles_alloc) {
    ISG_CUDA(realloc_dev(ctx, &ctx->ranges, tiles));
    ISG_CUDA(realloc_dev(ctx, &ctx->tile_cnt, tiles));
    ISG_CUDA(realloc_dev(ctx, &ctx->cursor, tiles));
    ISG_CUDA(realloc_dev(ctx, &ctx->tile_loss, tiles));
    ctx->tiles_alloc = tiles;
  }
  return ISG_OK;
}

// Camera::validate (splat3d.cpp:27-37) on the FP32 camera.  Orthonormality is checked to
// 1e-5 here (FP32 cannot hold 1e-9); the C++ drop-in validates the FP64 camera to 1e-9 first.
isg_status validate_camera(isg_ctx* ctx, const isg_camera* c) {
  if (!c) return fail(ctx, ISG_E_ARG, "camera: null pointer");
  for (int i = 0; i < 9; ++i)
    if (!std::isfinite(c->R[i])) return fail(ctx, ISG_E_DOMAIN, "Camera: non-finite transform");
  for (int i = 0; i < 3; ++i)
    if (!std::isfinite(c->t[i])) return fail(ctx, ISG_E_DOMAIN, "Camera: non-finite transform");
  double worst = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double d = 0.0;
      for (int k = 0; k < 3; ++k) d += (double)c->R[3 * i + k] * (double)c->R[3 * j + k];
      worst = std::max(worst, std::fabs(d - (i == j ? 1.0 : 0.0)));
    }
  if (worst > 1e-5) return fail(ctx, ISG_E_DOMAIN, "Camera.rotation: not orthonormal within 1e-9");
  if (!(c->focal > 0.0f) || !std::isfinite(c->focal))
    return fail(ctx, ISG_E_DOMAIN, "Camera.focal: must be > 0");
  if (!std::isfinite(c->cx) || !std::isfinite(c->cy))
    return fail(ctx, ISG_E_DOMAIN, "Camera: non-finite transform");
  if (c->width <= 0 || c->height <= 0) return fail(ctx, ISG_E_DOMAIN, "Camera: bad image size");
  if ((int64_t)c->width * c->height > (int64_t)1 << 30)
    return fail(ctx, ISG_E_ARG, "Camera: image too large");
  return ISG_OK;
}

FrameParams make_fp(const isg_camera* cam, const float bg[3], float t_min) {
  FrameParams fp;
  fp.cam = *cam;
  fp.tiles_x = (cam->width + isg::kTile - 1) / isg::kTile;
  fp.tiles_y = (cam->height + isg::kTile - 1) / isg::kTile;
  fp.n_tiles = fp.tiles_x * fp.tiles_y;
  for (int i = 0; i < 3; ++i) fp.bg[i] = bg ? bg[i] : 0.0f;
  fp.t_min = t_min;
  return fp;
}

// Splat slot lists: explicit in tile-bucket mode, contiguous (null) in radix mode.
const uint32_t* slot_list(const isg_ctx* ctx) {
  return ctx->binning == isg::kBinRadix ? nullptr : ctx->slot_of;
}

// The pending view's direct-mode 2D gradient sums (nullptr: slot mode).
float* pending_grad2d(const isg_ctx* ctx) { return ctx->pending_direct ? ctx->grad2d : nullptr; }

// Drop a pending view's 2D gradients unprojected (its direct-mode sums are zeroed for the
// next view; slot-mode slots are simply overwritten by the next backward).
isg_status drop_pending(isg_ctx* ctx) {
  if (ctx->pending && ctx->pending_direct && ctx->n_alloc > 0)
    ISG_CUDA(cudaMemsetAsync(ctx->grad2d, 0, sizeof(float) * 8 * ctx->n_alloc, ctx->stream));
  ctx->pending = false;
  return ISG_OK;
}

// Project a pending view's 2D gradients into the 3D accumulator (K8a).
isg_status flush_pending(isg_ctx* ctx) {
  if (!ctx->pending) return ISG_OK;
  ISG_STAGE(ST_PROJECT_BWD);
  isg::launch_project_backward(ctx->ms, ctx->co, ctx->n, ctx->pending_fp, ctx->slot_off,
                               slot_list(ctx), ctx->ntiles, ctx->partial, pending_grad2d(ctx),
                               ctx->total, ctx->key_cap, ctx->grad3d, !ctx->grad3d_valid,
                               ctx->stream);
  ISG_CHECK_LAUNCH();
  ctx->launches++;
  ctx->grad3d_valid = true;
  ctx->pending = false;
  return ISG_OK;
}

// Launch one frame: K1, depth sort, scan/emit, tile sort, ranges, K6 into `out` (nullptr =
// the context's own image buffer, resolved after it is sized for this camera).
// track: the forward also records the per-pixel state the backward starts from.
isg_status launch_frame(isg_ctx* ctx, const FrameParams& fp, float* out, bool track) {
  isg_status s = flush_pending(ctx);
  if (s != ISG_OK) return s;
  if ((s = ensure_pixels(ctx, fp.cam.width, fp.cam.height)) != ISG_OK) return s;
  if (!out) out = ctx->img;
  if (ctx->key_cap == 0) {
    if ((s = ensure_keys(ctx, default_key_cap(ctx->n))) != ISG_OK) return s;
  }
  if ((s = ensure_arena(ctx)) != ISG_OK) return s;
  const bool radix = ctx->binning == isg::kBinRadix;
  if (radix && (s = ensure_radix(ctx)) != ISG_OK) return s;
  cudaStream_t st = ctx->stream;
  const int64_t n = ctx->n;
  // the tile sort uses ceil(tile bits / 8) passes: 2 up to 65536 tiles, 3 beyond
  const int tile_passes = (bits_for(fp.n_tiles) + 7) / 8;
  {
  ISG_STAGE(ST_RESET);
  // scan look-back + both sorts' histograms, counters and look-back statuses, and the scalars
  // sc[0..7] + the frame's key total (contiguous): one zeroing kernel
  const size_t zero = radix ? (size_t)((unsigned char*)ctx->sort_tile.lookback - ctx->arena) +
                                  isg::sort_lookback_bytes(ctx->key_cap, tile_passes)
                            : ctx->arena_depth_end;
  isg::launch_zero2(ctx->arena, zero, ctx->sc, sizeof(uint32_t) * 8 + sizeof(unsigned long long),
                    st);
  ISG_CHECK_LAUNCH();
  ctx->launches++;
  if (!radix) ISG_CUDA(cudaMemsetAsync(ctx->tile_cnt, 0, sizeof(uint32_t) * fp.n_tiles, st));
  }
  {
  ISG_STAGE(ST_PREPROCESS);
  // radix mode: K1 also builds the depth sort's digit histograms
  isg::launch_preprocess(ctx->ms, ctx->co, n, fp, ctx->rec, ctx->depth[0], ctx->ntiles,
                         ctx->tilebox, radix ? nullptr : ctx->tile_cnt, ctx->sc,
                         radix ? ctx->sort_depth.hist : nullptr,
                         radix ? ctx->sort_depth.counters + isg::kMaxPasses : nullptr, st);
  ISG_CHECK_LAUNCH();
  ctx->launches++;
  }
  if (radix && n > 0) {
    {
    ISG_STAGE(ST_DEPTH_SORT);
    isg::SortOptions dopt;
    dopt.scratch_zeroed = dopt.hist_ready = true;
    ctx->order_buf = isg::radix_sort_pairs(ctx->depth, ctx->order, true, ctx->sc + 4, n, 32,
                                           ctx->sort_depth, st, &ctx->launches, dopt);
    ISG_CHECK_LAUNCH();
    }
    {
    ISG_STAGE(ST_SCAN_EMIT);
    // slot lists (slot_off) only for the deterministic backward; direct mode needs none
    isg::launch_scan_emit(ctx->order[ctx->order_buf], ctx->ntiles, ctx->tilebox, ctx->ms, n, fp,
                          ctx->deterministic ? ctx->slot_off : nullptr, ctx->tkey[0], ctx->emit_gid, ctx->key_cap,
                          ctx->scan_scratch, ctx->sc + 3, ctx->sc + 0, ctx->total, ctx->ranges,
                          fp.n_tiles, tile_passes, ctx->sort_tile.hist,
                          ctx->sort_tile.counters + isg::kMaxPasses, st);
    ISG_CHECK_LAUNCH();
    ctx->launches++;
    }
    {
    ISG_STAGE(ST_TILE_SORT);
    isg::SortOptions topt;
    topt.scratch_zeroed = topt.hist_ready = true;  // k_scan_emit built the histograms
    topt.epi.emit_gid = ctx->emit_gid;
    topt.epi.sorted = ctx->sorted;
    topt.epi.ranges = ctx->ranges;
    if (ctx->deterministic) {
      // values: emission indices (a pair's gradient slot), splat ids gathered at the end
      isg::radix_sort_pairs(ctx->tkey, ctx->tval, true, ctx->sc + 0, ctx->key_cap,
                            bits_for(fp.n_tiles), ctx->sort_tile, st, &ctx->launches, topt);
    } else {
      // direct mode needs no slot: the values are the splat ids themselves (read in emission
      // order by the first pass), no random gather of emit_gid in the last one
      topt.epi.vals_are_gids = true;
      uint32_t* vals[2] = {ctx->emit_gid, ctx->tval[1]};
      isg::radix_sort_pairs(ctx->tkey, vals, false, ctx->sc + 0, ctx->key_cap,
                            bits_for(fp.n_tiles), ctx->sort_tile, st, &ctx->launches, topt);
    }
    ISG_CHECK_LAUNCH();
    }
    // empty tiles keep (0xFFFFFFFF, 0): the blend kernels read them as empty, and only the
    // parity hook (isg_debug_bins) needs their oracle form (s, s)
  } else if (!radix) {
    {
    ISG_STAGE(ST_TILE_SCAN);
    isg::launch_tile_scan(ctx->tile_cnt, fp.n_tiles, ctx->key_cap, ctx->ranges, ctx->cursor,
                          ctx->sc + 0, ctx->total, st);
    ISG_CHECK_LAUNCH();
    ctx->launches++;
    }
    if (n > 0) {
      ISG_STAGE(ST_FILL);
      isg::launch_fill(ctx->ms, ctx->ntiles, ctx->tilebox, ctx->depth[0], n, fp, ctx->cursor,
                       ctx->bucket, ctx->slot_of, ctx->slot_off, ctx->key_cap, ctx->scan_scratch,
                       ctx->sc + 3, st);
      ISG_CHECK_LAUNCH();
      ctx->launches++;
    }
    {
    ISG_STAGE(ST_TILE_SORT);
    isg::launch_tile_sort(fp, ctx->ranges, ctx->bucket, ctx->total, ctx->key_cap, ctx->sorted,
                          ctx->partial, st);
    ISG_CHECK_LAUNCH();
    ctx->launches++;
    }
  } else {  // radix, empty scene: every tile empty at 0
    ISG_CUDA(cudaMemsetAsync(ctx->ranges, 0, sizeof(uint2) * fp.n_tiles, st));
  }
  ISG_STAGE(ST_BLEND_FWD);
  isg::launch_blend_fwd(fp, ctx->ranges, ctx->sorted, ctx->submask, ctx->rec, ctx->total,
                        ctx->key_cap, out, ctx->t_last, ctx->n_proc, track, st);
  ISG_CHECK_LAUNCH();
  ctx->launches++;
  ctx->last_tracked = track;
  ctx->have_frame = true;
  ctx->last_fp = fp;
  ctx->frame_unchecked = true;
  return ISG_OK;
}

const char* splat_message(const float* a, const float* c) {
  if (!std::isfinite(a[0]) || !std::isfinite(a[1]) || !std::isfinite(a[2]))
    return "IsoSplat3D.mu: non-finite coordinates";
  if (!(a[3] > 0.0f) || !std::isfinite(a[3])) return "IsoSplat3D.sigma: must be positive and finite";
  if (!std::isfinite(c[0]) || !std::isfinite(c[1]) || !std::isfinite(c[2]))
    return "IsoSplat3D.color: non-finite";
  return "IsoSplat3D.opacity: must be in [0,1]";
}

// Read back the frame scalars (syncs).  Returns ISG_E_DOMAIN for an invalid splat, and sets
// *overflow when the key capacity was exceeded (capacity is grown for the re-run).
// with_loss: also read the loss scalars back in the same synchronisation.
isg_status check_frame(isg_ctx* ctx, bool* overflow, bool with_loss = false) {
  *overflow = false;
  ISG_CUDA(cudaMemcpyAsync(ctx->h_sc, ctx->sc, sizeof(uint32_t) * 8, cudaMemcpyDeviceToHost,
                           ctx->stream));
  ISG_CUDA(cudaMemcpyAsync(ctx->h_total, ctx->total, sizeof(unsigned long long) * isg::kTotalWords,
                           cudaMemcpyDeviceToHost, ctx->stream));
  if (with_loss)
    ISG_CUDA(cudaMemcpyAsync(ctx->h_loss, ctx->loss, sizeof(double) * 4, cudaMemcpyDeviceToHost,
                             ctx->stream));
  ISG_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->frame_unchecked = false;
  ctx->n_visible = ctx->h_sc[2];
  ctx->n_keys = (int64_t)ctx->h_total[0];
  if (ctx->h_sc[1] != 0u) {
    const uint32_t bad = 0xFFFFFFFFu - ctx->h_sc[1];
    float a[4], c[4];
    ISG_CUDA(cudaMemcpy(a, ctx->ms + bad, sizeof a, cudaMemcpyDeviceToHost));
    ISG_CUDA(cudaMemcpy(c, ctx->co + bad, sizeof c, cudaMemcpyDeviceToHost));
    return fail(ctx, ISG_E_DOMAIN, splat_message(a, c));
  }
  // the sticky record covers every frame since the last check, not only the last one
  const unsigned long long need =
      std::max<unsigned long long>(ctx->h_total[isg::kTotalOverflowMax], ctx->h_total[isg::kTotalKeys]);
  if (ctx->h_total[isg::kTotalOverflowFrames] != 0 || need > (unsigned long long)ctx->key_cap) {
    *overflow = true;
    ctx->overflowed_frames += (int64_t)ctx->h_total[isg::kTotalOverflowFrames];
    ISG_CUDA(cudaMemsetAsync(ctx->total + isg::kTotalOverflowMax, 0, sizeof(unsigned long long) * 2,
                             ctx->stream));
    const int64_t want = (int64_t)need + (int64_t)need / 4 + 1024;
    if (want > isg::kMaxItems)
      return fail(ctx, ISG_E_OVERFLOW, "binning: more than 2^30 (tile, splat) pairs");
    if (want > ctx->key_cap) {
      isg_status s = ensure_keys(ctx, want);
      if (s != ISG_OK) return s;
      ctx->regrow++;  // the frame arena follows the new capacity at the next launch
    }
  }
  return ISG_OK;
}

// A host-synchronous entry point first settles the asynchronous frames issued since the last
// check (isg_*_device calls, graph replays): if one of them overflowed the key capacity it was
// skipped, along with any Adam step that followed it, and the caller must re-run them.
isg_status check_async(isg_ctx* ctx) {
  if (!ctx->frame_unchecked) return ISG_OK;
  bool ov = false;
  isg_status s = check_frame(ctx, &ov);
  if (s != ISG_OK) return s;
  if (ov) {
    if ((s = drop_pending(ctx)) != ISG_OK) return s;  // the step is re-run as a whole
    return fail(ctx, ISG_E_OVERFLOW,
                "tile-key capacity was exceeded by an asynchronous frame; it was skipped (with "
                "the Adam step after it) and capacity has been grown -- re-run the frames issued "
                "since the last synchronisation");
  }
  return ISG_OK;
}

// Buffers of the L1 + D-SSIM loss for a W x H image.
isg_status ensure_image_loss(isg_ctx* ctx, int W, int H) {
  const int64_t pix = (int64_t)W * H;
  if (pix > ctx->ssim_pix_alloc) {
    ISG_CUDA(realloc_dev(ctx, &ctx->coef, 9 * pix));
    ISG_CUDA(realloc_dev(ctx, &ctx->dldc, 3 * pix));
    ctx->ssim_pix_alloc = pix;
  }
  const int64_t parts = isg::ssim_part_count(W, H);
  if (parts > ctx->ssim_part_alloc) {
    ISG_CUDA(realloc_dev(ctx, &ctx->ssim_part, parts));
    ctx->ssim_part_alloc = parts;
  }
  return ISG_OK;
}

// ssim (loss.cpp:104-108) needs the 11x11 window to fit.
isg_status check_loss_size(isg_ctx* ctx, int W, int H) {
  if (ctx->loss_kind == ISG_LOSS_L1_DSSIM && ctx->lambda != 0.0f &&
      (W < 2 * isg::kSsimHalf + 1 || H < 2 * isg::kSsimHalf + 1))
    return fail(ctx, ISG_E_DOMAIN, "ssim: image smaller than the 11x11 window");
  return ISG_OK;
}

isg_status run_backward(isg_ctx* ctx, const FrameParams& fp, const float* target_dev,
                        float weight) {
  const int W = fp.cam.width, H = fp.cam.height;
  if (ctx->loss_kind == ISG_LOSS_L1_DSSIM) {
    isg_status s = ensure_image_loss(ctx, W, H);
    if (s != ISG_OK) return s;
    {
    ISG_STAGE(ST_IMAGE_LOSS);
    ctx->launches += isg::launch_image_loss(W, H, ctx->img, target_dev, ctx->lambda,
                                            (double)weight, true, ctx->coef, ctx->ssim_part,
                                            ctx->dldc, ctx->total, ctx->key_cap, ctx->loss,
                                            ctx->loss + 1, ctx->stream);
    ISG_CHECK_LAUNCH();
    }
    ISG_STAGE(ST_BLEND_BWD);
    isg::launch_blend_bwd(fp, ctx->ranges, ctx->sorted, ctx->submask, ctx->rec, ctx->total, ctx->key_cap,
                          ctx->img, ctx->dldc, ctx->t_last, ctx->n_proc, 1.0f, ctx->partial,
                          ctx->tile_loss, true, ctx->deterministic ? nullptr : ctx->grad2d,
                          ctx->stream);
    ISG_CHECK_LAUNCH();
    ctx->launches += 1;
  } else {
    const float scale = weight / (3.0f * (float)W * (float)H);
    {
    ISG_STAGE(ST_BLEND_BWD);
    isg::launch_blend_bwd(fp, ctx->ranges, ctx->sorted, ctx->submask, ctx->rec, ctx->total, ctx->key_cap,
                          ctx->img, target_dev, ctx->t_last, ctx->n_proc, scale, ctx->partial,
                          ctx->tile_loss, false, ctx->deterministic ? nullptr : ctx->grad2d,
                          ctx->stream);
    ISG_CHECK_LAUNCH();
    }
    ISG_STAGE(ST_LOSS_REDUCE);
    isg::launch_loss_reduce(ctx->tile_loss, fp.n_tiles, (double)weight / (3.0 * W * (double)H),
                            ctx->loss, ctx->loss + 1, ctx->stream);
    ISG_CHECK_LAUNCH();
    ctx->launches += 2;
  }
  ctx->pending = true;
  ctx->pending_fp = fp;
  ctx->pending_direct = !ctx->deterministic;
  return ISG_OK;
}

// Multi-GPU step (defined after the NCCL loader at the end of the file).
isg_status exchange_and_adam(isg_ctx* ctx, const float lr[4], float b1, float b2, float eps);

}  // namespace

// ============================================================================================
extern "C" {

int isg_abi_version(void) { return ISG_ABI_VERSION; }

const char* isg_status_string(isg_status s) {
  switch (s) {
    case ISG_OK: return "ok";
    case ISG_E_DOMAIN: return "domain error";
    case ISG_E_ARG: return "invalid argument";
    case ISG_E_CUDA: return "cuda error";
    case ISG_E_OOM: return "out of device memory";
    case ISG_E_OVERFLOW: return "capacity overflow";
    case ISG_E_NCCL: return "nccl error";
    case ISG_E_STATE: return "invalid call order";
  }
  return "unknown";
}

const char* isg_last_error(const isg_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

isg_status isg_create(int device, int64_t max_gaussians, int32_t max_width, int32_t max_height,
                      isg_ctx** out) {
  if (!out) return ISG_E_ARG;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return ISG_E_CUDA;
  }
  if (device < 0 || device >= count) return ISG_E_ARG;
  isg_ctx* ctx = new isg_ctx();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete ctx;
    return ISG_E_CUDA;
  }
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return ISG_E_CUDA;
  }
  ctx->own_stream = true;
  isg_status s = ISG_OK;
  auto chk = [&](cudaError_t e) {
    if (e != cudaSuccess && s == ISG_OK) s = e == cudaErrorMemoryAllocation ? ISG_E_OOM : ISG_E_CUDA;
  };
  chk(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  chk(cudaEventCreateWithFlags(&ctx->ev_main, cudaEventDisableTiming));
  chk(cudaEventCreateWithFlags(&ctx->ev_copy, cudaEventDisableTiming));
  // sc[0..7] followed by total[0..1] (one allocation: the per-frame part is zeroed at once)
  chk(cudaMalloc(&ctx->sc, sizeof(uint32_t) * 8 + sizeof(unsigned long long) * isg::kTotalWords));
  if (s == ISG_OK) ctx->total = reinterpret_cast<unsigned long long*>(ctx->sc + 8);
  chk(cudaMalloc(&ctx->loss, sizeof(double) * 4));
  chk(cudaMalloc(&ctx->adam_state, sizeof(isg::AdamState) * 2));
  chk(cudaMallocHost(&ctx->h_sc, sizeof(uint32_t) * 8));
  chk(cudaMallocHost(&ctx->h_total, sizeof(unsigned long long) * isg::kTotalWords));
  chk(cudaMallocHost(&ctx->h_loss, sizeof(double) * 4));
  if (s == ISG_OK) {
    chk(cudaMemset(ctx->total, 0, sizeof(unsigned long long) * isg::kTotalWords));
    std::memset(ctx->h_total, 0, sizeof(unsigned long long) * isg::kTotalWords);
    chk(cudaMemset(ctx->loss, 0, sizeof(double) * 4));
    chk(cudaMemset(ctx->adam_state, 0, sizeof(isg::AdamState) * 2));
  }
  if (s == ISG_OK && max_gaussians > 0) s = ensure_scene(ctx, max_gaussians);
  if (s == ISG_OK && max_width > 0 && max_height > 0) s = ensure_pixels(ctx, max_width, max_height);
  if (s != ISG_OK) {
    isg_destroy(ctx);
    return s;
  }
  *out = ctx;
  return ISG_OK;
}

isg_status isg_nccl_detach(isg_ctx* ctx);

void isg_destroy(isg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->nccl_comm) isg_nccl_detach(ctx);
  void* dev[] = {ctx->ms, ctx->co, ctx->m, ctx->v, ctx->raw, ctx->grad2d, ctx->rec, ctx->ntiles, ctx->slot_off, ctx->tilebox,
                 ctx->gradx, ctx->depth[0], ctx->depth[1], ctx->order[0], ctx->order[1],
                 ctx->sorted, ctx->submask, ctx->partial, ctx->bucket, ctx->slot_of, ctx->tkey[0], ctx->tkey[1],
                 ctx->tval[0], ctx->tval[1], ctx->emit_gid, ctx->sort.hist, ctx->sort.lookback,
                 ctx->sort.counters, ctx->arena, ctx->img, ctx->target, ctx->t_last,
                 ctx->n_proc, ctx->ranges, ctx->tile_cnt, ctx->cursor, ctx->tile_loss, ctx->sc,
                 ctx->loss, ctx->snap, ctx->coef, ctx->dldc, ctx->ssim_part,
                 ctx->adam_state};
  for (void* p : dev)
    if (p) cudaFree(p);
  isg::adapt_scratch_free(ctx->adapt);
  if (ctx->h_sc) cudaFreeHost(ctx->h_sc);
  if (ctx->h_total) cudaFreeHost(ctx->h_total);
  if (ctx->h_loss) cudaFreeHost(ctx->h_loss);
  for (auto& u : ctx->ev_used) {
    cudaEventDestroy(u.second.first);
    cudaEventDestroy(u.second.second);
  }
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->ev_main) cudaEventDestroy(ctx->ev_main);
  for (int i = 0; i < isg::kMaxExchangeChunks; ++i) {
    if (ctx->ev_grad[i]) cudaEventDestroy(ctx->ev_grad[i]);
    if (ctx->ev_red[i]) cudaEventDestroy(ctx->ev_red[i]);
  }
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  if (ctx->ev_copy) cudaEventDestroy(ctx->ev_copy);
  for (int k = 0; k < ISG_IMAGE_SLOTS; ++k) {
    if (ctx->ev_irend[k]) cudaEventDestroy(ctx->ev_irend[k]);
    if (ctx->ev_icopy[k]) cudaEventDestroy(ctx->ev_icopy[k]);
    if (ctx->iring[k]) cudaFree(ctx->iring[k]);
  }
  for (int k = 0; k < ISG_TARGET_SLOTS; ++k) {
    if (ctx->ev_tup[k]) cudaEventDestroy(ctx->ev_tup[k]);
    if (ctx->ev_tread[k]) cudaEventDestroy(ctx->ev_tread[k]);
    if (ctx->tring[k]) cudaFree(ctx->tring[k]);
  }
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
  }
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

isg_status isg_set_stream(isg_ctx* ctx, void* stream) {
  if (!ctx) return ISG_E_ARG;
  ISG_NO_CAPTURE("isg_set_stream");
  cudaSetDevice(ctx->device);
  ISG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  if (stream) {
    ctx->stream = (cudaStream_t)stream;
    ctx->own_stream = false;
  } else {
    ISG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = true;
  }
  return ISG_OK;
}

isg_status isg_synchronize(isg_ctx* ctx) {
  if (!ctx) return ISG_E_ARG;
  ISG_NO_CAPTURE("isg_synchronize");
  cudaSetDevice(ctx->device);
  if (ctx->frame_unchecked) return check_async(ctx);
  ISG_CUDA(cudaStreamSynchronize(ctx->stream));
  return ISG_OK;
}

isg_status isg_get_stats(const isg_ctx* ctx, isg_stats* out) {
  if (!ctx || !out) return ISG_E_ARG;
  out->n_gaussians = ctx->n;
  out->n_visible = ctx->n_visible;
  out->n_keys = ctx->n_keys;
  out->key_capacity = ctx->key_cap;
  out->n_tiles = ctx->have_frame ? ctx->last_fp.n_tiles : 0;
  out->adam_steps = ctx->adam_t;
  out->skipped_updates = ctx->h_total ? (int64_t)ctx->h_total[1] : 0;
  out->regrow_events = ctx->regrow;
  out->kernel_launches = ctx->launches;
  out->overflowed_frames = ctx->overflowed_frames;
  return ISG_OK;
}

static isg_status set_scene_impl(isg_ctx* ctx, int64_t n, const float* ms, const float* co,
                                 cudaMemcpyKind kind) {
  if (!ctx) return ISG_E_ARG;
  if (kind == cudaMemcpyHostToDevice) ISG_NO_CAPTURE("isg_set_scene");
  if (n < 0 || n > isg::kMaxItems) return fail(ctx, ISG_E_ARG, "set_scene: bad splat count (> 2^30)");
  if (n > 0 && (!ms || !co)) return fail(ctx, ISG_E_ARG, "set_scene: null pointer");
  cudaSetDevice(ctx->device);
  isg_status s = ensure_scene(ctx, n);
  if (s != ISG_OK) return s;
  if (n > 0) {
    ISG_CUDA(cudaMemcpyAsync(ctx->ms, ms, sizeof(float4) * n, kind, ctx->stream));
    ISG_CUDA(cudaMemcpyAsync(ctx->co, co, sizeof(float4) * n, kind, ctx->stream));
    ISG_CUDA(cudaMemsetAsync(ctx->m, 0, sizeof(float4) * 2 * n, ctx->stream));
    ISG_CUDA(cudaMemsetAsync(ctx->v, 0, sizeof(float4) * 2 * n, ctx->stream));
    isg::launch_raw_init(ctx->ms, ctx->co, n, ctx->raw, ctx->stream);
    ISG_CHECK_LAUNCH();
    ctx->launches++;
  }
  // frames of the previous scene are void: their overflow record with them
  ISG_CUDA(cudaMemsetAsync(ctx->total + isg::kTotalOverflowMax, 0, sizeof(unsigned long long) * 2,
                           ctx->stream));
  ctx->frame_unchecked = false;
  if (ctx->n != n || ctx->key_cap < 4 * n) {
    // size the key buffers for the new scene on the next frame
    if (ctx->key_cap < default_key_cap(n)) {
      s = ensure_keys(ctx, default_key_cap(n));
      if (s != ISG_OK) return s;
    }
  }
  ctx->n = n;
  ctx->adam_t = 0;
  ISG_CUDA(cudaMemsetAsync(ctx->adam_state, 0, sizeof(isg::AdamState), ctx->stream));
  ctx->snap_valid = false;
  if ((s = drop_pending(ctx)) != ISG_OK) return s;
  ctx->grad3d_valid = false;
  ctx->have_frame = false;
  ISG_CUDA(cudaMemsetAsync(ctx->loss, 0, sizeof(double) * 2, ctx->stream));
  if (kind == cudaMemcpyHostToDevice) ISG_CUDA(cudaStreamSynchronize(ctx->stream));
  return ISG_OK;
}

isg_status isg_set_scene(isg_ctx* ctx, int64_t n, const float* ms, const float* co) {
  return set_scene_impl(ctx, n, ms, co, cudaMemcpyHostToDevice);
}

isg_status isg_set_scene_device(isg_ctx* ctx, int64_t n, const float* ms, const float* co) {
  return set_scene_impl(ctx, n, ms, co, cudaMemcpyDeviceToDevice);
}

isg_status isg_get_scene(isg_ctx* ctx, float* ms, float* co) {
  if (!ctx) return ISG_E_ARG;
  ISG_NO_CAPTURE("isg_get_scene");
  cudaSetDevice(ctx->device);
  if (ctx->n > 0) {
    if (ms) ISG_CUDA(cudaMemcpyAsync(ms, ctx->ms, sizeof(float4) * ctx->n, cudaMemcpyDeviceToHost, ctx->stream));
    if (co) ISG_CUDA(cudaMemcpyAsync(co, ctx->co, sizeof(float4) * ctx->n, cudaMemcpyDeviceToHost, ctx->stream));
  }
  ISG_CUDA(cudaStreamSynchronize(ctx->stream));
  return ISG_OK;
}

isg_status isg_render_device(isg_ctx* ctx, const isg_camera* cam, const float bg[3], float t_min,
                             float* out_dev) {
  if (!ctx) return ISG_E_ARG;
  if (!out_dev) return fail(ctx, ISG_E_ARG, "render: null output");
  if (!(t_min >= 0.0f) || !(t_min < 1.0f)) return fail(ctx, ISG_E_ARG, "render: t_min must be in [0,1)");
  cudaSetDevice(ctx->device);
  isg_status s = validate_camera(ctx, cam);
  if (s != ISG_OK) return s;
  return launch_frame(ctx, make_fp(cam, bg, t_min), out_dev, false);
}

isg_status isg_render_host_async(isg_ctx* ctx, const isg_camera* cam, const float bg[3],
                                 float t_min, int32_t slot, float* host_dst) {
  if (!ctx) return ISG_E_ARG;
  ISG_NO_CAPTURE("isg_render_host_async");
  if (slot < 0 || slot >= ISG_IMAGE_SLOTS) return fail(ctx, ISG_E_ARG, "render_host_async: bad slot");
  if (!host_dst) return fail(ctx, ISG_E_ARG, "render: null output");
  if (!(t_min >= 0.0f) || !(t_min < 1.0f)) return fail(ctx, ISG_E_ARG, "render: t_min must be in [0,1)");
  cudaSetDevice(ctx->device);
  isg_status s = validate_camera(ctx, cam);
  if (s != ISG_OK) return s;
  const size_t floats = 3 * (size_t)cam->width * (size_t)cam->height;
  if (floats > ctx->iring_floats[slot]) {
    if (ctx->iring[slot]) {  // nothing may still write or read the old image
      ISG_CUDA(cudaStreamSynchronize(ctx->copy_stream));
      ISG_CUDA(cudaStreamSynchronize(ctx->stream));
      cudaFree(ctx->iring[slot]);
      ctx->iring[slot] = nullptr;
    }
    ctx->iring_floats[slot] = 0;
    ctx->iring_copied[slot] = false;
    ISG_CUDA(cudaMalloc(&ctx->iring[slot], sizeof(float) * floats));
    if (!ctx->ev_irend[slot]) ISG_CUDA(cudaEventCreateWithFlags(&ctx->ev_irend[slot], cudaEventDisableTiming));
    if (!ctx->ev_icopy[slot]) ISG_CUDA(cudaEventCreateWithFlags(&ctx->ev_icopy[slot], cudaEventDisableTiming));
    ctx->iring_floats[slot] = floats;
  }
  // the slot's previous image may still be on its way to the host
  if (ctx->iring_copied[slot]) ISG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_icopy[slot], 0));
  if ((s = launch_frame(ctx, make_fp(cam, bg, t_min), ctx->iring[slot], false)) != ISG_OK) return s;
  ISG_CUDA(cudaEventRecord(ctx->ev_irend[slot], ctx->stream));
  ISG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_irend[slot], 0));
  ISG_CUDA(cudaMemcpyAsync(host_dst, ctx->iring[slot], sizeof(float) * floats,
                           cudaMemcpyDeviceToHost, ctx->copy_stream));
  ISG_CUDA(cudaEventRecord(ctx->ev_icopy[slot], ctx->copy_stream));
  ctx->iring_copied[slot] = true;
  return ISG_OK;
}

isg_status isg_image_wait(isg_ctx* ctx, int32_t slot) {
  if (!ctx) return ISG_E_ARG;
  ISG_NO_CAPTURE("isg_image_wait");
  if (slot < 0 || slot >= ISG_IMAGE_SLOTS) return fail(ctx, ISG_E_ARG, "image_wait: bad slot");
  if (!ctx->iring_copied[slot]) return ISG_OK;
  cudaSetDevice(ctx->device);
  ISG_CUDA(cudaEventSynchronize(ctx->ev_icopy[slot]));
  return ISG_OK;
}

isg_status isg_render(isg_ctx* ctx, const isg_camera* cam, const float bg[3], float t_min,
                      float* out_hwc3) {
  if (!ctx) return ISG_E_ARG;
  ISG_NO_CAPTURE("isg_render");
  if (!out_hwc3) return fail(ctx, ISG_E_ARG, "render: null output");
  if (!(t_min >= 0.0f) || !(t_min < 1.0f)) return fail(ctx, ISG_E_ARG, "render: t_min must be in [0,1)");
  cudaSetDevice(ctx->device);
  isg_status s = validate_camera(ctx, cam);
  if (s != ISG_OK) return s;
  if ((s = check_async(ctx)) != ISG_OK) return s;
  const FrameParams fp = make_fp(cam, bg, t_min);
  for (int attempt = 0; attempt < 3; ++attempt) {
    if ((s = launch_frame(ctx, fp, nullptr, false)) != ISG_OK) return s;
    // image read-back queued behind the frame; one synchronisation covers both
    ISG_CUDA(cudaMemcpyAsync(out_hwc3, ctx->img, sizeof(float) * 3 * (size_t)cam->width * cam->height,
                             cudaMemcpyDeviceToHost, ctx->stream));
    bool ov = false;
    if ((s = check_frame(ctx, &ov)) != ISG_OK) return s;
    if (ov) continue;  // the copied image is stale: re-run with grown buffers
    return ISG_OK;
  }
  return fail(ctx, ISG_E_OVERFLOW, "render: key capacity kept overflowing");
}

isg_status isg_loss_backward_device(isg_ctx* ctx, const isg_camera* cam, const float bg[3],
                                    float t_min, const float* target_dev, float weight) {
  if (!ctx) return ISG_E_ARG;
  if (!target_dev) return fail(ctx, ISG_E_ARG, "loss_backward: null target");
  if (!(t_min >= 0.0f) || !(t_min < 1.0f)) return fail(ctx, ISG_E_ARG, "loss_backward: t_min must be in [0,1)");
  if (!std::isfinite(weight)) return fail(ctx, ISG_E_ARG, "loss_backward: non-finite weight");
  cudaSetDevice(ctx->device);
  isg_status s = validate_camera(ctx, cam);
  if (s != ISG_OK) return s;
  if ((s = check_loss_size(ctx, cam->width, cam->height)) != ISG_OK) return s;
  const FrameParams fp = make_fp(cam, bg, t_min);
  if ((s = launch_frame(ctx, fp, nullptr, true)) != ISG_OK) return s;
  return run_backward(ctx, fp, target_dev, weight);
}

isg_status isg_upload_target_async(isg_ctx* ctx, int32_t slot, const float* host_hwc3,
                                   int32_t width, int32_t height) {
  if (!ctx) return ISG_E_ARG;
  ISG_NO_CAPTURE("isg_upload_target_async");
  if (slot < 0 || slot >= ISG_TARGET_SLOTS) return fail(ctx, ISG_E_ARG, "upload_target: bad slot");
  if (!host_hwc3 || width <= 0 || height <= 0)
    return fail(ctx, ISG_E_ARG, "upload_target: null target or empty image");
  cudaSetDevice(ctx->device);
  const size_t floats = 3 * (size_t)width * (size_t)height;
  if (floats > ctx->tring_floats[slot]) {
    // (re)allocating the slot: nothing may still read or fill it
    if (ctx->tring[slot]) {
      ISG_CUDA(cudaStreamSynchronize(ctx->copy_stream));
      ISG_CUDA(cudaStreamSynchronize(ctx->stream));
      cudaFree(ctx->tring[slot]);
      ctx->tring[slot] = nullptr;
    }
    ctx->tring_floats[slot] = 0;
    ctx->tring_read[slot] = false;
    ISG_CUDA(cudaMalloc(&ctx->tring[slot], sizeof(float) * floats));
    if (!ctx->ev_tup[slot]) ISG_CUDA(cudaEventCreateWithFlags(&ctx->ev_tup[slot], cudaEventDisableTiming));
    if (!ctx->ev_tread[slot]) ISG_CUDA(cudaEventCreateWithFlags(&ctx->ev_tread[slot], cudaEventDisableTiming));
    ctx->tring_floats[slot] = floats;
  }
  // the slot's previous image may still be read by a frame enqueued earlier
  if (ctx->tring_read[slot]) ISG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_tread[slot], 0));
  ISG_CUDA(cudaMemcpyAsync(ctx->tring[slot], host_hwc3, sizeof(float) * floats,
                           cudaMemcpyHostToDevice, ctx->copy_stream));
  ISG_CUDA(cudaEventRecord(ctx->ev_tup[slot], ctx->copy_stream));
  return ISG_OK;
}

isg_status isg_loss_backward_slot(isg_ctx* ctx, const isg_camera* cam, const float bg[3],
                                  float t_min, int32_t slot, float weight) {
  if (!ctx) return ISG_E_ARG;
  if (slot < 0 || slot >= ISG_TARGET_SLOTS || !ctx->tring[slot])
    return fail(ctx, ISG_E_ARG, "loss_backward_slot: slot has no uploaded target");
  if (!(t_min >= 0.0f) || !(t_min < 1.0f)) return fail(ctx, ISG_E_ARG, "loss_backward: t_min must be in [0,1)");
  if (!std::isfinite(weight)) return fail(ctx, ISG_E_ARG, "loss_backward: non-finite weight");
  if (!cam || 3 * (size_t)cam->width * (size_t)cam->height > ctx->tring_floats[slot])
    return fail(ctx, ISG_E_ARG, "loss_backward_slot: camera larger than the uploaded target");
  cudaSetDevice(ctx->device);
  isg_status s = validate_camera(ctx, cam);
  if (s != ISG_OK) return s;
  if ((s = check_loss_size(ctx, cam->width, cam->height)) != ISG_OK) return s;
  const FrameParams fp = make_fp(cam, bg, t_min);
  // binning and the forward do not need the target: only the backward waits for the upload
  if ((s = launch_frame(ctx, fp, nullptr, true)) != ISG_OK) return s;
  // Inside a graph capture the wait and the record become external event nodes: each replay
  // waits for the slot's most recent upload enqueued before the launch, and marks the slot
  // read for the next upload into it (so a step can be captured once per slot and replayed
  // while the uploads run outside the graph).
  ISG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_tup[slot],
                               ctx->capturing ? cudaEventWaitExternal : 0));
  if ((s = run_backward(ctx, fp, ctx->tring[slot], weight)) != ISG_OK) return s;
  ISG_CUDA(cudaEventRecordWithFlags(ctx->ev_tread[slot], ctx->stream,
                                    ctx->capturing ? cudaEventRecordExternal : 0));
  ctx->tring_read[slot] = true;
  return ISG_OK;
}

isg_status isg_loss_backward(isg_ctx* ctx, const isg_camera* cam, const float bg[3], float t_min,
                             const float* target, float weight, double* loss_out) {
  if (!ctx) return ISG_E_ARG;
  ISG_NO_CAPTURE("isg_loss_backward");
  if (!target) return fail(ctx, ISG_E_ARG, "loss_backward: null target");
  if (!(t_min >= 0.0f) || !(t_min < 1.0f)) return fail(ctx, ISG_E_ARG, "loss_backward: t_min must be in [0,1)");
  if (!std::isfinite(weight)) return fail(ctx, ISG_E_ARG, "loss_backward: non-finite weight");
  cudaSetDevice(ctx->device);
  isg_status s = validate_camera(ctx, cam);
  if (s != ISG_OK) return s;
  if ((s = check_loss_size(ctx, cam->width, cam->height)) != ISG_OK) return s;
  if ((s = check_async(ctx)) != ISG_OK) return s;
  if ((s = ensure_pixels(ctx, cam->width, cam->height)) != ISG_OK) return s;
  const FrameParams fp = make_fp(cam, bg, t_min);
  // The target upload runs on the copy stream, overlapped with binning and the forward blend;
  // only K7 consumes it.  It first waits for earlier work on the main stream (a previous K7
  // may still read the buffer).
  ISG_CUDA(cudaEventRecord(ctx->ev_main, ctx->stream));
  ISG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_main, 0));
  ISG_CUDA(cudaMemcpyAsync(ctx->target, target, sizeof(float) * 3 * (size_t)cam->width * cam->height,
                           cudaMemcpyHostToDevice, ctx->copy_stream));
  ISG_CUDA(cudaEventRecord(ctx->ev_copy, ctx->copy_stream));
  for (int attempt = 0; attempt < 3; ++attempt) {
    if ((s = launch_frame(ctx, fp, nullptr, true)) != ISG_OK) return s;
    ISG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_copy, 0));
    if ((s = run_backward(ctx, fp, ctx->target, weight)) != ISG_OK) return s;
    bool ov = false;
    if ((s = check_frame(ctx, &ov, true)) != ISG_OK) return s;
    if (ov) {  // K6/K7 skipped the overflowed frame: nothing was accumulated
      ctx->pending = false;
      continue;
    }
    if (loss_out) *loss_out = ctx->h_loss[1];
    return ISG_OK;
  }
  return fail(ctx, ISG_E_OVERFLOW, "loss_backward: key capacity kept overflowing");
}

isg_status isg_read_loss(isg_ctx* ctx, double* loss_out) {
  if (!ctx || !loss_out) return ISG_E_ARG;
  isg_status s = isg_synchronize(ctx);
  if (s != ISG_OK) return s;
  ISG_CUDA(cudaMemcpyAsync(ctx->h_loss, ctx->loss, sizeof(double) * 2, cudaMemcpyDeviceToHost,
                           ctx->stream));
  ISG_CUDA(cudaStreamSynchronize(ctx->stream));
  *loss_out = ctx->h_loss[0];
  return ISG_OK;
}

isg_status isg_zero_grads(isg_ctx* ctx) {
  if (!ctx) return ISG_E_ARG;
  cudaSetDevice(ctx->device);
  isg_status s = drop_pending(ctx);  // the pending view's gradients are simply dropped
  if (s != ISG_OK) return s;
  ctx->grad3d_valid = false;
  ISG_CUDA(cudaMemsetAsync(ctx->loss, 0, sizeof(double) * 2, ctx->stream));
  return ISG_OK;
}

isg_status isg_grads_device(isg_ctx* ctx, float** grads_dev) {
  if (!ctx || !grads_dev) return ISG_E_ARG;
  cudaSetDevice(ctx->device);
  isg_status s = flush_pending(ctx);
  if (s != ISG_OK) return s;
  if (!ctx->grad3d_valid && ctx->n > 0) {
    ISG_CUDA(cudaMemsetAsync(ctx->grad3d, 0, sizeof(float4) * 2 * ctx->n, ctx->stream));
    ctx->grad3d_valid = true;
  }
  *grads_dev = reinterpret_cast<float*>(ctx->grad3d);
  return ISG_OK;
}

isg_status isg_get_grads(isg_ctx* ctx, float* grads) {
  if (!ctx || !grads) return ISG_E_ARG;
  float* d = nullptr;
  isg_status s = isg_grads_device(ctx, &d);
  if (s != ISG_OK) return s;
  if (ctx->n > 0)
    ISG_CUDA(cudaMemcpyAsync(grads, d, sizeof(float) * 8 * ctx->n, cudaMemcpyDeviceToHost, ctx->stream));
  ISG_CUDA(cudaStreamSynchronize(ctx->stream));
  return ISG_OK;
}

isg_status isg_set_grads(isg_ctx* ctx, const float* grads) {
  if (!ctx || !grads) return ISG_E_ARG;
  ISG_NO_CAPTURE("isg_set_grads");
  float* d = nullptr;
  isg_status s = isg_grads_device(ctx, &d);  // projects a pending view first
  if (s != ISG_OK) return s;
  if (ctx->n > 0)
    ISG_CUDA(cudaMemcpyAsync(d, grads, sizeof(float) * 8 * ctx->n, cudaMemcpyHostToDevice, ctx->stream));
  ISG_CUDA(cudaStreamSynchronize(ctx->stream));
  return ISG_OK;
}

isg_status isg_adam_step(isg_ctx* ctx, const float lr[4], float b1, float b2, float eps) {
  if (!ctx || !lr) return ISG_E_ARG;
  for (int i = 0; i < 4; ++i)
    if (!(lr[i] >= 0.0f) || !std::isfinite(lr[i])) return fail(ctx, ISG_E_ARG, "adam: learning rates must be >= 0");
  if (!(b1 >= 0.0f && b1 < 1.0f) || !(b2 >= 0.0f && b2 < 1.0f))
    return fail(ctx, ISG_E_ARG, "adam: betas must be in [0,1)");
  if (!(eps >= 0.0f)) return fail(ctx, ISG_E_ARG, "adam: eps must be >= 0");
  if (!ctx->pending && !ctx->grad3d_valid)
    return fail(ctx, ISG_E_STATE, "adam: no gradients accumulated since the last step");
  cudaSetDevice(ctx->device);
  ctx->adam_t++;  // host mirror (stats); the device counter drives the bias corrections
  if (ctx->pending && !ctx->grad3d_valid && !ctx->nccl_comm) {
    // single view since the last step: projection backward fused with Adam (K8)
    ISG_STAGE(ST_PROJECT_ADAM);
    isg::launch_adam_tick(lr, b1, b2, eps, ctx->adam_state, ctx->loss, ctx->total, ctx->stream);
    isg::launch_project_adam(ctx->ms, ctx->co, ctx->n, ctx->pending_fp, ctx->slot_off,
                             slot_list(ctx), ctx->ntiles, ctx->partial, pending_grad2d(ctx),
                             ctx->total, ctx->raw,
                             ctx->m, ctx->v, ctx->adam_state, ctx->stream);
    ISG_CHECK_LAUNCH();
    ctx->launches += 2;
    ctx->pending = false;
  } else if (ctx->nccl_comm) {
    isg_status s = exchange_and_adam(ctx, lr, b1, b2, eps);
    if (s != ISG_OK) return s;
  } else {
    isg_status s = flush_pending(ctx);
    if (s != ISG_OK) return s;
    ISG_STAGE(ST_ADAM);
    isg::launch_adam_tick(lr, b1, b2, eps, ctx->adam_state, ctx->loss, ctx->total, ctx->stream);
    isg::launch_adam(ctx->ms, ctx->co, ctx->n, ctx->grad3d, ctx->raw, ctx->m, ctx->v,
                     ctx->adam_state, ctx->total, ctx->stream);
    ISG_CHECK_LAUNCH();
    ctx->launches += 2;
  }
  ctx->grad3d_valid = false;
  return ISG_OK;
}

isg_status isg_last_step_loss(isg_ctx* ctx, double* loss_out) {
  if (!ctx || !loss_out) return ISG_E_ARG;
  isg_status s = isg_synchronize(ctx);
  if (s != ISG_OK) return s;
  ISG_CUDA(cudaMemcpyAsync(ctx->h_loss, ctx->loss, sizeof(double) * 3, cudaMemcpyDeviceToHost,
                           ctx->stream));
  ISG_CUDA(cudaStreamSynchronize(ctx->stream));
  *loss_out = ctx->h_loss[2];
  return ISG_OK;
}

namespace {
// The step loss straight into mapped pinned host memory: one thread's store over PCIe, chained
// to the Adam kernel by programmatic dependent launch (a D2H memcpy node would go through a copy
// engine and cost the next graph launch ~10 us of latency).
__global__ void k_store_loss(const double* __restrict__ src, double* __restrict__ dst) {
  isg::pdl_enter();
  *dst = *src;
}
}  // namespace

isg_status isg_step_loss_async(isg_ctx* ctx, double* host_dst) {
  if (!ctx || !host_dst) return ISG_E_ARG;
  cudaSetDevice(ctx->device);
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, host_dst) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
      pa.devicePointer != nullptr) {
    ISG_CUDA(isg::launch_pdl(k_store_loss, dim3(1), dim3(1), 0, ctx->stream,
                             (const double*)(ctx->loss + 2), (double*)pa.devicePointer));
    ctx->launches++;
    return ISG_OK;
  }
  cudaGetLastError();  // (pageable memory: cudaPointerGetAttributes reports it unregistered)
  ISG_CUDA(cudaMemcpyAsync(host_dst, ctx->loss + 2, sizeof(double), cudaMemcpyDefault,
                           ctx->stream));
  return ISG_OK;
}

isg_status isg_eval_loss(isg_ctx* ctx, const isg_camera* cam, const float bg[3], float t_min,
                         const float* target_dev, float weight, double* loss_out) {
  if (!ctx || !loss_out) return ISG_E_ARG;
  ISG_NO_CAPTURE("isg_eval_loss");
  if (!target_dev) return fail(ctx, ISG_E_ARG, "eval_loss: null target");
  if (!(t_min >= 0.0f) || !(t_min < 1.0f)) return fail(ctx, ISG_E_ARG, "eval_loss: t_min must be in [0,1)");
  cudaSetDevice(ctx->device);
  isg_status s = validate_camera(ctx, cam);
  if (s != ISG_OK) return s;
  if ((s = check_loss_size(ctx, cam->width, cam->height)) != ISG_OK) return s;
  if ((s = check_async(ctx)) != ISG_OK) return s;
  const FrameParams fp = make_fp(cam, bg, t_min);
  const int W = cam->width, H = cam->height;
  if (ctx->loss_kind == ISG_LOSS_L1_DSSIM && (s = ensure_image_loss(ctx, W, H)) != ISG_OK) return s;
  for (int attempt = 0; attempt < 3; ++attempt) {
    if ((s = launch_frame(ctx, fp, nullptr, false)) != ISG_OK) return s;
    if (ctx->loss_kind == ISG_LOSS_L1_DSSIM) {
      ISG_STAGE(ST_IMAGE_LOSS);
      ctx->launches += isg::launch_image_loss(W, H, ctx->img, target_dev, ctx->lambda,
                                              (double)weight, false, ctx->coef, ctx->ssim_part,
                                              nullptr, ctx->total, ctx->key_cap, nullptr,
                                              ctx->loss + 3, ctx->stream);
    } else {
      isg::launch_l2_tiles(fp, ctx->img, target_dev, ctx->tile_loss, ctx->stream);
      isg::launch_loss_reduce(ctx->tile_loss, fp.n_tiles, (double)weight / (3.0 * W * (double)H),
                              nullptr, ctx->loss + 3, ctx->stream);
      ctx->launches += 2;
    }
    ISG_CHECK_LAUNCH();
    bool ov = false;
    if ((s = check_frame(ctx, &ov, true)) != ISG_OK) return s;
    if (ov) continue;
    *loss_out = ctx->h_loss[3];
    return ISG_OK;
  }
  return fail(ctx, ISG_E_OVERFLOW, "eval_loss: key capacity kept overflowing");
}

isg_status isg_snapshot(isg_ctx* ctx) {
  if (!ctx) return ISG_E_ARG;
  cudaSetDevice(ctx->device);
  if (ctx->snap_n < ctx->n) {
    // ms | co | m (2n) | v (2n) | raw (n float2 = n/2 float4)
    ISG_CUDA(realloc_dev(ctx, &ctx->snap, 7 * std::max<int64_t>(ctx->n, 1), false));
    ctx->snap_n = ctx->n;
  }
  const size_t n = (size_t)ctx->n;
  if (n) {
    ISG_CUDA(cudaMemcpyAsync(ctx->snap, ctx->ms, sizeof(float4) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    ISG_CUDA(cudaMemcpyAsync(ctx->snap + n, ctx->co, sizeof(float4) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    ISG_CUDA(cudaMemcpyAsync(ctx->snap + 2 * n, ctx->m, sizeof(float4) * 2 * n, cudaMemcpyDeviceToDevice, ctx->stream));
    ISG_CUDA(cudaMemcpyAsync(ctx->snap + 4 * n, ctx->v, sizeof(float4) * 2 * n, cudaMemcpyDeviceToDevice, ctx->stream));
    ISG_CUDA(cudaMemcpyAsync(ctx->snap + 6 * n, ctx->raw, sizeof(float2) * n, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  ISG_CUDA(cudaMemcpyAsync(ctx->adam_state + 1, ctx->adam_state, sizeof(isg::AdamState),
                           cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->snap_t = ctx->adam_t;
  ctx->snap_valid = true;
  return ISG_OK;
}

isg_status isg_restore(isg_ctx* ctx) {
  if (!ctx) return ISG_E_ARG;
  if (!ctx->snap_valid || ctx->snap_n < ctx->n)
    return fail(ctx, ISG_E_STATE, "restore: no snapshot of the current scene");
  cudaSetDevice(ctx->device);
  const size_t n = (size_t)ctx->n;
  if (n) {
    ISG_CUDA(cudaMemcpyAsync(ctx->ms, ctx->snap, sizeof(float4) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    ISG_CUDA(cudaMemcpyAsync(ctx->co, ctx->snap + n, sizeof(float4) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    ISG_CUDA(cudaMemcpyAsync(ctx->m, ctx->snap + 2 * n, sizeof(float4) * 2 * n, cudaMemcpyDeviceToDevice, ctx->stream));
    ISG_CUDA(cudaMemcpyAsync(ctx->v, ctx->snap + 4 * n, sizeof(float4) * 2 * n, cudaMemcpyDeviceToDevice, ctx->stream));
    ISG_CUDA(cudaMemcpyAsync(ctx->raw, ctx->snap + 6 * n, sizeof(float2) * n, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  ISG_CUDA(cudaMemcpyAsync(ctx->adam_state, ctx->adam_state + 1, sizeof(isg::AdamState),
                           cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->adam_t = ctx->snap_t;
  ctx->have_frame = false;
  return ISG_OK;
}

isg_status isg_adaptive_control(isg_ctx* ctx, const isg_adapt_params* prm, uint64_t seed,
                                uint64_t round, isg_adapt_result* out) {
  if (!ctx || !prm) return ISG_E_ARG;
  ISG_NO_CAPTURE("isg_adaptive_control");
  // AdaptiveControlParams::validate (include/isosplat/optimize.hpp:21-27)
  if (!(prm->prune_threshold >= 0.0)) return fail(ctx, ISG_E_ARG, "prune_threshold: must be >= 0");
  if (!(prm->merge_distance_factor > 0.0))
    return fail(ctx, ISG_E_ARG, "merge_distance_factor: must be > 0");
  if (!(prm->merge_color_tol >= 0.0)) return fail(ctx, ISG_E_ARG, "merge_color_tol: must be >= 0");
  if (!(prm->split_sigma_max > 0.0)) return fail(ctx, ISG_E_ARG, "split_sigma_max: must be > 0");
  cudaSetDevice(ctx->device);
  isg_status s = isg_synchronize(ctx);
  if (s != ISG_OK) return s;
  const int64_t n = ctx->n;
  const int64_t cap = prm->max_particles > 0 ? prm->max_particles : 2 * n;
  if (cap > isg::kMaxItems) return fail(ctx, ISG_E_ARG, "max_particles: too large (> 2^30)");
  // grow the scene buffers (preserving the splats) so the appended split children fit
  if (cap > ctx->n_alloc) {
    float4 *ms_keep = nullptr, *co_keep = nullptr;
    ISG_CUDA(cudaMalloc(&ms_keep, sizeof(float4) * std::max<int64_t>(n, 1)));
    ISG_CUDA(cudaMalloc(&co_keep, sizeof(float4) * std::max<int64_t>(n, 1)));
    if (n) {
      ISG_CUDA(cudaMemcpyAsync(ms_keep, ctx->ms, sizeof(float4) * n, cudaMemcpyDeviceToDevice, ctx->stream));
      ISG_CUDA(cudaMemcpyAsync(co_keep, ctx->co, sizeof(float4) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    ISG_CUDA(cudaStreamSynchronize(ctx->stream));
    s = ensure_scene(ctx, cap);
    if (s == ISG_OK && n) {
      cudaMemcpyAsync(ctx->ms, ms_keep, sizeof(float4) * n, cudaMemcpyDeviceToDevice, ctx->stream);
      cudaMemcpyAsync(ctx->co, co_keep, sizeof(float4) * n, cudaMemcpyDeviceToDevice, ctx->stream);
      cudaStreamSynchronize(ctx->stream);
    }
    cudaFree(ms_keep);
    cudaFree(co_keep);
    if (s != ISG_OK) return s;
  }
  if ((s = ensure_sort_scratch(ctx, std::max(ctx->key_cap, ctx->n_alloc))) != ISG_OK) return s;
  isg::AdaptParamsDev p{prm->prune_threshold, prm->merge_distance_factor, prm->merge_color_tol,
                        prm->split_sigma_max, cap};
  isg::AdaptCounts c{};
  // (ctx->ms / ctx->co may come back swapped with the persistent scratch's temporaries)
  const cudaError_t e = isg::adaptive_control(ctx->ms, ctx->co, n, ctx->n_alloc, p, seed, round,
                                              ctx->sort, ctx->depth, ctx->order, ctx->adapt, &c,
                                              ctx->stream, &ctx->launches);
  ctx->buf_gen++;  // the scene may now live in the former scratch buffers
  if (e != cudaSuccess) return cuda_fail(ctx, e, "adaptive_control");
  // the optimizer restarts on the new set (the reference clears its momentum, optimize.cpp:344)
  ctx->n = c.n_after;
  if (ctx->n > 0) {
    ISG_CUDA(cudaMemsetAsync(ctx->m, 0, sizeof(float4) * 2 * ctx->n, ctx->stream));
    ISG_CUDA(cudaMemsetAsync(ctx->v, 0, sizeof(float4) * 2 * ctx->n, ctx->stream));
    isg::launch_raw_init(ctx->ms, ctx->co, ctx->n, ctx->raw, ctx->stream);
    ctx->launches++;
  }
  ctx->adam_t = 0;
  ISG_CUDA(cudaMemsetAsync(ctx->adam_state, 0, sizeof(isg::AdamState), ctx->stream));
  ctx->snap_valid = false;
  if ((s = drop_pending(ctx)) != ISG_OK) return s;
  ctx->grad3d_valid = false;
  ctx->have_frame = false;
  ISG_CUDA(cudaMemsetAsync(ctx->loss, 0, sizeof(double) * 2, ctx->stream));
  ISG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->key_cap < default_key_cap(ctx->n)) {
    if ((s = ensure_keys(ctx, default_key_cap(ctx->n))) != ISG_OK) return s;
  }
  if (out) {
    out->n_before = c.n_before;
    out->n_pruned = c.n_pruned;
    out->n_merged = c.n_merged;
    out->n_split = c.n_split;
    out->n_after = c.n_after;
  }
  return ISG_OK;
}

struct isg_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0;
  uint64_t buf_gen = 0;  // the context's buffer generation the graph's pointers belong to
};

isg_status isg_graph_begin(isg_ctx* ctx) {
  if (!ctx) return ISG_E_ARG;
  if (ctx->capturing) return fail(ctx, ISG_E_STATE, "graph_begin: already capturing");
  cudaSetDevice(ctx->device);
  isg_status s = isg_synchronize(ctx);  // pending overflow checks happen before the capture
  if (s != ISG_OK) return s;
  ISG_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  ctx->capturing = true;
  ctx->capture_launches0 = ctx->launches;
  ctx->capture_gen0 = ctx->buf_gen;
  return ISG_OK;
}

isg_status isg_graph_end(isg_ctx* ctx, isg_graph** out) {
  if (!ctx || !out) return ISG_E_ARG;
  if (!ctx->capturing) return fail(ctx, ISG_E_STATE, "graph_end: not capturing");
  cudaSetDevice(ctx->device);
  ctx->capturing = false;
  isg_graph* g = new isg_graph();
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &g->graph);
  if (e == cudaSuccess) e = cudaGraphInstantiate(&g->exec, g->graph, 0);
  if (e != cudaSuccess) {
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
    cudaGetLastError();
    return cuda_fail(ctx, e, "graph capture");
  }
  g->launches = ctx->launches - ctx->capture_launches0;
  g->buf_gen = ctx->buf_gen;
  if (ctx->buf_gen != ctx->capture_gen0) {  // a buffer grew inside the capture
    cudaGraphExecDestroy(g->exec);
    cudaGraphDestroy(g->graph);
    delete g;
    return fail(ctx, ISG_E_STATE,
                "graph_end: device buffers were reallocated during the capture; run the step "
                "once outside a capture (it sizes the buffers), then capture it");
  }
  *out = g;
  return ISG_OK;
}

isg_status isg_graph_launch(isg_ctx* ctx, isg_graph* g) {
  if (!ctx || !g) return ISG_E_ARG;
  if (ctx->capturing) return fail(ctx, ISG_E_STATE, "graph_launch: inside a capture");
  if (g->buf_gen != ctx->buf_gen)
    return fail(ctx, ISG_E_STATE,
                "graph_launch: device buffers were reallocated since the capture (scene size, "
                "key capacity, image size or adaptive control); capture the step again");
  cudaSetDevice(ctx->device);
  ISG_CUDA(cudaGraphLaunch(g->exec, ctx->stream));
  ctx->launches += g->launches;
  ctx->frame_unchecked = true;  // replayed frames are checked at the next synchronisation
  return ISG_OK;
}

void isg_graph_destroy(isg_graph* g) {
  if (!g) return;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
}

isg_status isg_set_loss(isg_ctx* ctx, int kind, float lambda) {
  if (!ctx) return ISG_E_ARG;
  if (kind != ISG_LOSS_L2 && kind != ISG_LOSS_L1_DSSIM)
    return fail(ctx, ISG_E_ARG, "set_loss: unknown loss kind");
  if (kind == ISG_LOSS_L1_DSSIM && !(lambda >= 0.0f && lambda <= 1.0f))
    return fail(ctx, ISG_E_DOMAIN, "loss: lambda must be in [0,1]");  // loss.cpp:186
  ctx->loss_kind = kind;
  if (kind == ISG_LOSS_L1_DSSIM) ctx->lambda = lambda;
  return ISG_OK;
}

isg_status isg_image_loss_device(isg_ctx* ctx, int32_t width, int32_t height,
                                 const float* fhat_dev, const float* target_dev, float weight,
                                 double* loss_out, float* dldc_dev) {
  if (!ctx || !loss_out || !fhat_dev || !target_dev) return ISG_E_ARG;
  ISG_NO_CAPTURE("isg_image_loss_device");
  if (width <= 0 || height <= 0) return fail(ctx, ISG_E_ARG, "image_loss: bad image size");
  if (!std::isfinite(weight)) return fail(ctx, ISG_E_ARG, "image_loss: non-finite weight");
  cudaSetDevice(ctx->device);
  isg_status s = check_loss_size(ctx, width, height);
  if (s != ISG_OK) return s;
  if ((s = isg_synchronize(ctx)) != ISG_OK) return s;
  if (ctx->loss_kind == ISG_LOSS_L1_DSSIM) {
    if ((s = ensure_image_loss(ctx, width, height)) != ISG_OK) return s;
    ISG_STAGE(ST_IMAGE_LOSS);
    ctx->launches += isg::launch_image_loss(width, height, fhat_dev, target_dev, ctx->lambda,
                                            (double)weight, dldc_dev != nullptr, ctx->coef,
                                            ctx->ssim_part, dldc_dev, nullptr, 0, nullptr,
                                            ctx->loss + 3, ctx->stream);
    ISG_CHECK_LAUNCH();
  } else {
    // mse (image.cpp:50-58) on the 16x16 tiling of the frame kernels
    if ((s = ensure_pixels(ctx, width, height)) != ISG_OK) return s;
    isg_camera cam{};
    cam.width = width;
    cam.height = height;
    const FrameParams fp = make_fp(&cam, nullptr, 0.0f);
    isg::launch_l2_tiles(fp, fhat_dev, target_dev, ctx->tile_loss, ctx->stream);
    isg::launch_loss_reduce(ctx->tile_loss, fp.n_tiles,
                            (double)weight / (3.0 * width * (double)height), nullptr,
                            ctx->loss + 3, ctx->stream);
    ISG_CHECK_LAUNCH();
    ctx->launches += 2;
    if (dldc_dev) {
      isg::launch_l2_grad(width, height, fhat_dev, target_dev,
                          2.0f * weight / (3.0f * (float)width * (float)height), dldc_dev,
                          ctx->stream);
      ISG_CHECK_LAUNCH();
      ctx->launches += 1;
    }
  }
  ISG_CUDA(cudaMemcpyAsync(ctx->h_loss + 3, ctx->loss + 3, sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
  ISG_CUDA(cudaStreamSynchronize(ctx->stream));
  *loss_out = ctx->h_loss[3];
  return ISG_OK;
}

isg_status isg_debug_bins(isg_ctx* ctx, uint64_t* keys, uint32_t* vals, int64_t* n_keys,
                          uint32_t* ranges) {
  if (!ctx || !n_keys) return ISG_E_ARG;
  if (!ctx->have_frame) return fail(ctx, ISG_E_STATE, "debug_bins: no frame rendered yet");
  cudaSetDevice(ctx->device);
  bool ov = false;
  isg_status s = check_frame(ctx, &ov);
  if (s != ISG_OK) return s;
  if (ov) return fail(ctx, ISG_E_OVERFLOW, "debug_bins: last frame overflowed");
  const int64_t nk = ctx->n_keys;
  *n_keys = nk;
  const FrameParams& fp = ctx->last_fp;
  if (ctx->binning == isg::kBinRadix)
    isg::launch_ranges_fix(ctx->sc + 0, ctx->key_cap, fp.n_tiles, ctx->ranges, ctx->stream);
  if ((keys || vals) && nk > 0) {
    uint64_t* dk = nullptr;
    uint32_t* dv = nullptr;
    ISG_CUDA(cudaMalloc(&dk, sizeof(uint64_t) * nk));
    ISG_CUDA(cudaMalloc(&dv, sizeof(uint32_t) * nk));
    isg::launch_debug_keys(ctx->ranges, ctx->sorted, ctx->ms, fp, dk, dv, ctx->stream);
    if (keys) cudaMemcpyAsync(keys, dk, sizeof(uint64_t) * nk, cudaMemcpyDeviceToHost, ctx->stream);
    if (vals) cudaMemcpyAsync(vals, dv, sizeof(uint32_t) * nk, cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    cudaFree(dk);
    cudaFree(dv);
  }
  if (ranges)
    ISG_CUDA(cudaMemcpyAsync(ranges, ctx->ranges, sizeof(uint2) * fp.n_tiles, cudaMemcpyDeviceToHost,
                             ctx->stream));
  ISG_CUDA(cudaStreamSynchronize(ctx->stream));
  ISG_CUDA(cudaGetLastError());
  return ISG_OK;
}

isg_status isg_set_deterministic(isg_ctx* ctx, int on) {
  if (!ctx) return ISG_E_ARG;
  ISG_NO_CAPTURE("isg_set_deterministic");
  cudaSetDevice(ctx->device);
  isg_status s = flush_pending(ctx);  // the pending view keeps the mode it was computed in
  if (s != ISG_OK) return s;
  ctx->deterministic = on != 0;
  return ISG_OK;
}

isg_status isg_set_binning(isg_ctx* ctx, int mode) {
  if (!ctx) return ISG_E_ARG;
  if (mode != ISG_BINNING_TILE_BUCKET && mode != ISG_BINNING_RADIX)
    return fail(ctx, ISG_E_ARG, "set_binning: unknown mode");
  cudaSetDevice(ctx->device);
  isg_status s = flush_pending(ctx);  // slot lists of a pending view are mode-specific
  if (s != ISG_OK) return s;
  ctx->binning = mode;
  ctx->have_frame = false;
  return ISG_OK;
}

isg_status isg_profile_enable(isg_ctx* ctx, int on) {
  if (!ctx) return ISG_E_ARG;
  ctx->prof = on != 0;
  isg::g_pdl_enabled = !ctx->prof;
  return ISG_OK;
}

int isg_profile_num_stages(void) { return ST_COUNT; }

const char* isg_profile_stage_name(int i) { return (i >= 0 && i < ST_COUNT) ? kStageNames[i] : ""; }

isg_status isg_profile_read(isg_ctx* ctx, double* ms, int64_t* calls) {
  if (!ctx) return ISG_E_ARG;
  cudaSetDevice(ctx->device);
  ISG_CUDA(cudaStreamSynchronize(ctx->stream));
  for (auto& u : ctx->ev_used) {
    float t = 0.f;
    cudaEventElapsedTime(&t, u.second.first, u.second.second);
    ctx->prof_ms[u.first] += t;
    ctx->prof_calls[u.first] += 1;
    ctx->ev_pool.push_back(u.second.first);
    ctx->ev_pool.push_back(u.second.second);
  }
  ctx->ev_used.clear();
  for (int i = 0; i < ST_COUNT; ++i) {
    if (ms) ms[i] = ctx->prof_ms[i];
    if (calls) calls[i] = ctx->prof_calls[i];
    ctx->prof_ms[i] = 0.0;
    ctx->prof_calls[i] = 0;
  }
  return ISG_OK;
}

isg_status isg_count_pairs(isg_ctx* ctx, int64_t* evaluated, int64_t* inside) {
  if (!ctx || !evaluated || !inside) return ISG_E_ARG;
  if (!ctx->have_frame) return fail(ctx, ISG_E_STATE, "count_pairs: no frame rendered yet");
  cudaSetDevice(ctx->device);
  bool ov = false;
  isg_status s = check_frame(ctx, &ov);
  if (s != ISG_OK) return s;
  if (ov) return fail(ctx, ISG_E_OVERFLOW, "count_pairs: last frame overflowed");
  const FrameParams& fp = ctx->last_fp;
  if (ctx->binning == isg::kBinRadix)
    isg::launch_ranges_fix(ctx->sc + 0, ctx->key_cap, fp.n_tiles, ctx->ranges, ctx->stream);
  unsigned long long* d = nullptr;
  ISG_CUDA(cudaMalloc(&d, 2 * sizeof(unsigned long long)));
  ISG_CUDA(cudaMemsetAsync(d, 0, 2 * sizeof(unsigned long long), ctx->stream));
  isg::launch_count_pairs(fp, ctx->ranges, ctx->sorted, ctx->rec, d, ctx->stream);
  unsigned long long h[2] = {0, 0};
  cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream);
  const cudaError_t e = cudaStreamSynchronize(ctx->stream);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "count_pairs");
  *evaluated = (int64_t)h[0];
  *inside = (int64_t)h[1];
  return ISG_OK;
}

isg_status isg_debug_pixel_state(isg_ctx* ctx, float* t_last, uint32_t* n_proc) {
  if (!ctx) return ISG_E_ARG;
  if (!ctx->have_frame) return fail(ctx, ISG_E_STATE, "debug_pixel_state: no frame rendered yet");
  cudaSetDevice(ctx->device);
  if (!ctx->last_tracked) {
    // render-only frames skip the per-pixel bookkeeping: re-run the last frame with it (into
    // the context's own image)
    isg_status s = flush_pending(ctx);
    if (s != ISG_OK) return s;
    if ((s = launch_frame(ctx, ctx->last_fp, nullptr, true)) != ISG_OK) return s;
  }
  const size_t pix = (size_t)ctx->last_fp.cam.width * ctx->last_fp.cam.height;
  if (t_last) ISG_CUDA(cudaMemcpyAsync(t_last, ctx->t_last, sizeof(float) * pix, cudaMemcpyDeviceToHost, ctx->stream));
  if (n_proc) ISG_CUDA(cudaMemcpyAsync(n_proc, ctx->n_proc, sizeof(uint32_t) * pix, cudaMemcpyDeviceToHost, ctx->stream));
  ISG_CUDA(cudaStreamSynchronize(ctx->stream));
  return ISG_OK;
}

}  // extern "C"

// ============================================================================================
// Multi-GPU: one process per GPU; NCCL resolved at run time so the library has no link-time
// NCCL dependency (and reuses the libnccl.so.2 torch already loaded, if any).
#include <nccl.h>  // types only

namespace {
struct NcclApi {
  bool ok = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*comm_user_rank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  // 1. an NCCL already in the process (e.g. the one torch loaded) — sharing it avoids two
  //    NCCL versions under one SONAME; 2. $ISG_NCCL_LIB; 3. the loader's search path.
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  const char* env = std::getenv("ISG_NCCL_LIB");
  if (!h && env && *env) h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
  if (!h) return api;
  api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
  api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
  api.all_reduce = (decltype(api.all_reduce))dlsym(h, "ncclAllReduce");
  api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
  api.comm_count = (decltype(api.comm_count))dlsym(h, "ncclCommCount");
  api.comm_user_rank = (decltype(api.comm_user_rank))dlsym(h, "ncclCommUserRank");
  api.get_version = (decltype(api.get_version))dlsym(h, "ncclGetVersion");
  api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
  api.ok = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.comm_destroy &&
           api.comm_count && api.comm_user_rank && api.error_string;
  return api;
}

// Stream and events of the pipelined exchange (created once per context).
isg_status exchange_resources(isg_ctx* ctx) {
  if (ctx->comm_stream) return ISG_OK;
  ISG_CUDA(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
  for (int i = 0; i < isg::kMaxExchangeChunks; ++i) {
    ISG_CUDA(cudaEventCreateWithFlags(&ctx->ev_grad[i], cudaEventDisableTiming));
    ISG_CUDA(cudaEventCreateWithFlags(&ctx->ev_red[i], cudaEventDisableTiming));
  }
  return ISG_OK;
}

isg_status attach_comm(isg_ctx* ctx, ncclComm_t comm, bool own) {
  NcclApi& api = nccl();
  int count = 0, rank = 0;
  ncclResult_t r = api.comm_count(comm, &count);
  if (r == ncclSuccess) r = api.comm_user_rank(comm, &rank);
  if (r != ncclSuccess) return fail(ctx, ISG_E_NCCL, std::string("nccl: ") + api.error_string(r));
  if (count > isg::kMaxRanks)
    return fail(ctx, ISG_E_ARG, "nccl: more ranks than the exchange supports (64)");
  isg_status s = exchange_resources(ctx);
  if (s != ISG_OK) return s;
  ctx->nccl_comm = comm;
  ctx->own_comm = own;
  ctx->nranks = count;
  ctx->rank = rank;
  return ISG_OK;
}

}  // namespace

namespace {
// The multi-GPU step (isg_adam_step with a communicator attached).  Every rank has projected,
// or is about to project, its own views' 2D gradients into grad3d (n x 8); the exchange sums
// them over ranks and every replica applies the identical Adam step (bitwise-identical scenes).
// Pipelined over `exchange_chunks` splat ranges on two streams:
//
//   compute: pack | K8a c0 | K8a c1 | ... | K8a cK | unpack, tick, Adam c0 | Adam c1 | ...
//   comm:            AR(slots + c0) | AR(c1) | ...   (Adam c waits for AR c)
//
// The all-reduce of chunk c overlaps the projection backward of chunk c + 1 and the Adam update
// of chunk c - 1.  The step's loss (a double as three exact floats) and every rank's overflow
// flag ride in front of chunk 0 (`nranks` slots just ahead of grad3d): one collective per chunk
// and no separate scalar exchange.  A rank whose view overflowed makes every rank skip the step.
isg_status exchange_and_adam(isg_ctx* ctx, const float lr[4], float b1, float b2, float eps) {
  NcclApi& api = nccl();
  cudaStream_t st = ctx->stream, cs = ctx->comm_stream;
  const int64_t n = ctx->n;
  const bool project = ctx->pending;  // the last view's 2D gradients are still to be projected
  const bool first = !ctx->grad3d_valid;
  if (!project && first && n > 0)
    ISG_CUDA(cudaMemsetAsync(ctx->grad3d, 0, sizeof(float4) * 2 * n, st));
  // chunks of >= 128K splats, boundaries on multiples of 256 splats
  const int chunks = (int)std::max<int64_t>(1, std::min<int64_t>(ctx->exchange_chunks, n >> 17));
  auto bound = [&](int c) -> int64_t {
    if (c >= chunks) return n;
    return std::min<int64_t>(n, ((n * c / chunks) + 255) & ~int64_t(255));
  };
  float4* slots = ctx->grad3d - ctx->nranks;  // contiguous with chunk 0
  {
    ISG_STAGE(ST_ALLREDUCE);
    isg::launch_loss_pack(ctx->loss, ctx->total, slots, ctx->rank, ctx->nranks, st);
    ctx->launches++;
    for (int c = 0; c < chunks; ++c) {
      const int64_t b = bound(c), e = bound(c + 1);
      if (project && e > b) {
        isg::launch_project_backward(ctx->ms, ctx->co, n, ctx->pending_fp, ctx->slot_off,
                                     slot_list(ctx), ctx->ntiles, ctx->partial,
                                     pending_grad2d(ctx), ctx->total, ctx->key_cap, ctx->grad3d,
                                     first, st, b, e);
        ctx->launches++;
      }
      ISG_CHECK_LAUNCH();
      ISG_CUDA(cudaEventRecord(ctx->ev_grad[c], st));
      ISG_CUDA(cudaStreamWaitEvent(cs, ctx->ev_grad[c], 0));
      const float4* base = c == 0 ? slots : ctx->grad3d + 2 * b;
      const size_t count = (size_t)(ctx->grad3d + 2 * e - base) * 4;
      const ncclResult_t r = api.all_reduce(base, (void*)base, count, ncclFloat32, ncclSum,
                                            (ncclComm_t)ctx->nccl_comm, cs);
      if (r != ncclSuccess)
        return fail(ctx, ISG_E_NCCL, std::string("ncclAllReduce: ") + api.error_string(r));
      ISG_CUDA(cudaEventRecord(ctx->ev_red[c], cs));
    }
  }
  ctx->pending = false;
  ctx->grad3d_valid = true;
  ISG_STAGE(ST_ADAM);
  ISG_CUDA(cudaStreamWaitEvent(st, ctx->ev_red[0], 0));
  isg::launch_loss_unpack(ctx->loss, ctx->total, slots, ctx->nranks, st);
  isg::launch_adam_tick(lr, b1, b2, eps, ctx->adam_state, ctx->loss, ctx->total, st);
  ctx->launches += 2;
  for (int c = 0; c < chunks; ++c) {
    const int64_t b = bound(c), e = bound(c + 1);
    if (c > 0) ISG_CUDA(cudaStreamWaitEvent(st, ctx->ev_red[c], 0));
    if (e > b) {
      isg::launch_adam(ctx->ms + b, ctx->co + b, e - b, ctx->grad3d + 2 * b, ctx->raw + b,
                       ctx->m + 2 * b, ctx->v + 2 * b, ctx->adam_state, ctx->total, st);
      ctx->launches++;
    }
  }
  ISG_CHECK_LAUNCH();
  return ISG_OK;
}
}  // namespace

extern "C" {

isg_status isg_nccl_get_unique_id(void* out) {
  if (!out) return ISG_E_ARG;
  NcclApi& api = nccl();
  if (!api.ok) return ISG_E_NCCL;
  ncclUniqueId id;
  if (api.get_unique_id(&id) != ncclSuccess) return ISG_E_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, &id, sizeof id);
  return ISG_OK;
}

isg_status isg_nccl_init(isg_ctx* ctx, int nranks, int rank, const void* uid) {
  if (!ctx || !uid || nranks < 1 || rank < 0 || rank >= nranks) return ISG_E_ARG;
  if (nranks > isg::kMaxRanks) return fail(ctx, ISG_E_ARG, "nccl: more than 64 ranks");
  NcclApi& api = nccl();
  if (!api.ok) return fail(ctx, ISG_E_NCCL, "nccl: libnccl.so.2 not loadable");
  cudaSetDevice(ctx->device);
  if (ctx->nccl_comm) isg_nccl_detach(ctx);
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof id);
  ncclComm_t comm = nullptr;
  const ncclResult_t r = api.comm_init_rank(&comm, nranks, id, rank);
  if (r != ncclSuccess) return fail(ctx, ISG_E_NCCL, std::string("ncclCommInitRank: ") + api.error_string(r));
  const isg_status s = attach_comm(ctx, comm, true);
  if (s != ISG_OK) api.comm_destroy(comm);
  return s;
}

isg_status isg_nccl_attach(isg_ctx* ctx, void* comm) {
  if (!ctx || !comm) return ISG_E_ARG;
  NcclApi& api = nccl();
  if (!api.ok) return fail(ctx, ISG_E_NCCL, "nccl: libnccl.so.2 not loadable");
  cudaSetDevice(ctx->device);
  if (ctx->nccl_comm) isg_nccl_detach(ctx);
  return attach_comm(ctx, (ncclComm_t)comm, false);
}

isg_status isg_nccl_info(isg_ctx* ctx, int* nranks, int* rank, int* nccl_version) {
  if (!ctx) return ISG_E_ARG;
  NcclApi& api = nccl();
  if (nccl_version) {
    *nccl_version = 0;
    if (api.ok && api.get_version) api.get_version(nccl_version);
  }
  if (!ctx->nccl_comm) {
    if (nranks) *nranks = 1;
    if (rank) *rank = 0;
    return ISG_OK;
  }
  int c = 0, u = 0;  // asked of the communicator itself, not the context's copy
  ncclResult_t r = api.comm_count((ncclComm_t)ctx->nccl_comm, &c);
  if (r == ncclSuccess) r = api.comm_user_rank((ncclComm_t)ctx->nccl_comm, &u);
  if (r != ncclSuccess) return fail(ctx, ISG_E_NCCL, std::string("nccl: ") + api.error_string(r));
  if (nranks) *nranks = c;
  if (rank) *rank = u;
  return ISG_OK;
}

isg_status isg_set_exchange_chunks(isg_ctx* ctx, int chunks) {
  if (!ctx) return ISG_E_ARG;
  if (chunks < 1 || chunks > isg::kMaxExchangeChunks)
    return fail(ctx, ISG_E_ARG, "exchange chunks: must be in [1, 8]");
  ctx->exchange_chunks = chunks;
  return ISG_OK;
}

isg_status isg_nccl_detach(isg_ctx* ctx) {
  if (!ctx) return ISG_E_ARG;
  if (ctx->nccl_comm) {
    cudaStreamSynchronize(ctx->stream);
    if (ctx->comm_stream) cudaStreamSynchronize(ctx->comm_stream);
    if (ctx->own_comm) nccl().comm_destroy((ncclComm_t)ctx->nccl_comm);
  }
  ctx->nccl_comm = nullptr;
  ctx->own_comm = false;
  ctx->nranks = 1;
  ctx->rank = 0;
  return ISG_OK;
}

}  // extern "C"

// isg_internal.cuh — shared definitions of the sm_100a kernels and the C-ABI layer.
//
// Pipeline of one view (all on one stream, no host sync inside a frame):
//   K1  k_preprocess      per splat: validate, project, 3-sigma radius, tile count, 32-B record
//   binning (two interchangeable modes, identical output):
//     radix (default)        onesweep depth sort (histograms from K1) -> k_scan_emit (tile
//                            histograms) -> onesweep tile sort whose last pass writes the
//                            pairs and the ranges                            (k_sort.cu)
//     tile-bucket            K2 k_tile_scan -> K3 k_fill -> K4 k_tile_sort   (k_bin.cu)
//     output: per-tile ranges and, per list entry, (splat, gradient slot) in (depth, index)
//     order; per splat, the list of its gradient slots.
//   K6  k_blend_fwd       16x16-tile front-to-back blend with early termination
//   K7  k_blend_bwd       reverse walk + fused L2 gradient (or a given dL/dC, k_ssim.cu) ->
//                         per-(tile, splat) gradient slots
//   K8  k_project_adam    per-splat slot sum, projection backward (+ Adam when fused)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "../../include/isg.h"

namespace isg {

constexpr int kTile = ISG_TILE;
constexpr int kTilePixels = kTile * kTile;
constexpr float kNearPlane = 1e-3f;  // splat3d.hpp:55
// Opacity floor of the render record's log2(opacity) (k_preprocess.cu): alpha / o stays defined
// in the backward, and an alpha of at most 2^-60 is an exact no-op on 1 - alpha
constexpr float kOpacityFloor = 0x1p-60f;

enum BinningMode { kBinTileBucket = 0, kBinRadix = 1 };

// Device counters `total[kTotalWords]` (u64).  The frame reset zeroes only kTotalKeys; the
// overflow record is sticky until the host's next check (capi.cu check_frame), so a skipped
// frame is never lost behind later frames, and every Adam kernel refuses to step while it is
// set (no update from a partial view batch).
enum TotalWord {
  kTotalKeys = 0,            // (tile, splat) pairs of the current frame
  kTotalSkipped = 1,         // Adam updates skipped for non-finite gradients (cumulative)
  kTotalOverflowMax = 2,     // max pairs needed by an overflowed frame since the last check
  kTotalOverflowFrames = 3,  // frames skipped for overflow since the last check
  kTotalWords = 4
};
// Largest key capacity / scene size: the onesweep look-back status words hold 30-bit counts.
constexpr int64_t kMaxItems = int64_t(1) << 30;

// ---- per-frame constant parameters --------------------------------------------------------
struct FrameParams {
  isg_camera cam;
  int tiles_x, tiles_y, n_tiles;
  float bg[3];
  float t_min;
};

// Render record of one splat, indexed by splat (32 B, two float4):
//   geo = (u, v, r2max = (9*sigma2d)*sigma2d, -log2(e)/sigma2d^2),  col = (r, g, b, log2 opacity)
struct __align__(16) RenderRec {
  float4 geo;
  float4 col;
};

// ---- radix sort (onesweep, 8-bit digits, u32 keys + u32 values) ---------------------------
constexpr int kSortThreads = 256;
#ifndef ISG_SORT_ITEMS
#define ISG_SORT_ITEMS 8
#endif
constexpr int kSortItems = ISG_SORT_ITEMS;  // items per thread
constexpr int kSortTileItems = kSortThreads * kSortItems;
constexpr int kMaxPasses = 4;

struct SortScratch {
  uint32_t* hist;       // kMaxPasses x 256 global digit histograms -> exclusive digit offsets
  uint32_t* lookback;   // kMaxPasses x max_tiles x 256 status words
  uint32_t* counters;   // kMaxPasses dynamic tile counters + 1 histogram completion counter
  int64_t max_tiles;    // per pass
};

inline int64_t sort_tiles_for(int64_t cap) { return (cap + kSortTileItems - 1) / kSortTileItems; }

// Stable LSD sort of n (device count *n_dev, <= cap) pairs on bits [0, key_bits).  keys/vals
// are ping-pong buffers; returns the index (0/1) of the buffer holding the result.  With
// iota_vals the first pass uses the item index as the value (vals[0] is not read).
// scratch_zeroed: the caller zeroed s (hist, counters, the passes' look-back) on the stream.
// Optional epilogue of a sort's last pass (the tile sort): instead of (keys, vals) it writes
// sorted[o] = (emit_gid[val], val) and the per-tile [start, end) of the key runs into `ranges`
// (pre-set to (0xFFFFFFFF, 0) per tile; launch_ranges_fix then fills the empty tiles).
struct SortEpilogue {
  const uint32_t* emit_gid = nullptr;
  uint2* sorted = nullptr;
  uint2* ranges = nullptr;
  // the sorted values are splat ids already (the direct-mode backward needs no gradient slot):
  // sorted[o] = (val, o), no emit_gid gather
  bool vals_are_gids = false;
};
struct SortOptions {
  bool scratch_zeroed = false;  // hist / counters / look-back already zero (one frame memset)
  bool hist_ready = false;      // hist already holds the exclusive digit offsets (the keys'
                                // producer built them: radix_hist.cuh); no k_hist launch
  SortEpilogue epi;
};
int radix_sort_pairs(uint32_t* keys[2], uint32_t* vals[2], bool iota_vals, const uint32_t* n_dev,
                     int64_t cap, int key_bits, SortScratch& s, cudaStream_t st,
                     int64_t* launches, const SortOptions& opt = SortOptions());

// Byte size of a sort's look-back region for `passes` passes over up to `cap` items.
// Per pass: one status row (256 words) per tile (level 1) and one per group of tiles (level 2,
// k_sort.cu's two-level look-back; rows for groups of 8 tiles or more).
#ifndef ISG_LOOKBACK_GROUP
#define ISG_LOOKBACK_GROUP 8
#endif
inline size_t sort_lookback_words(int64_t tiles) {
  const int64_t t = std::max<int64_t>(tiles, 1);
  return (size_t)256 * (t + (t + ISG_LOOKBACK_GROUP - 1) / ISG_LOOKBACK_GROUP);
}
inline size_t sort_lookback_bytes(int64_t cap, int passes) {
  return sizeof(uint32_t) * sort_lookback_words(sort_tiles_for(cap)) * passes;
}

// ---- K1 ------------------------------------------------------------------------------------
// sc: [1] 0xFFFFFFFF - first invalid splat (atomicMax; 0 = none), [2] visible splats, [4] n.  tilebox: compact tile
// bbox + hit mask per splat (see for_each_tile).  tile_cnt (tile-bucket mode) may be null.
void launch_preprocess(const float4* ms, const float4* co, int64_t n, const FrameParams& fp,
                       RenderRec* rec, uint32_t* depth_key, uint32_t* ntiles, uint2* tilebox,
                       uint32_t* tile_cnt, uint32_t* sc, uint32_t* hist, uint32_t* hist_done,
                       cudaStream_t st);

// zero [a, a + a_bytes) and [b, b + b_bytes) (the frame's scratch reset)
void launch_zero2(void* a, size_t a_bytes, void* b, size_t b_bytes, cudaStream_t st);

// ---- tile-bucket binning (k_bin.cu) -------------------------------------------------------
int64_t fill_scratch_words(int64_t n);  // + 1 zeroed u64 words of look-back scratch
void launch_tile_scan(const uint32_t* cnt, int n_tiles, int64_t cap, uint2* ranges,
                      uint32_t* cursor, uint32_t* n_keys, unsigned long long* total,
                      cudaStream_t st);
void launch_fill(const float4* ms, const uint32_t* ntiles, const uint2* tilebox,
                 const uint32_t* depth_key, int64_t n, const FrameParams& fp, uint32_t* cursor,
                 unsigned long long* bucket, uint32_t* slot_of, uint32_t* slot_off, int64_t cap,
                 unsigned long long* lookback, uint32_t* counter, cudaStream_t st);
// scratch: the gradient-slot buffer (2 float4 per key), used only for tiles > 2048 entries.
void launch_tile_sort(const FrameParams& fp, const uint2* ranges, const unsigned long long* bucket,
                      const unsigned long long* total, int64_t cap, uint2* sorted, float4* scratch,
                      cudaStream_t st);

// ---- radix binning (k_sort.cu) ------------------------------------------------------------
int64_t scan_emit_scratch_words(int64_t n);  // + 1 zeroed u64 words
void launch_scan_emit(const uint32_t* order, const uint32_t* ntiles, const uint2* tilebox,
                      const float4* ms, int64_t n, const FrameParams& fp, uint32_t* slot_off,
                      uint32_t* tile_keys, uint32_t* emit_gid, int64_t key_cap,
                      unsigned long long* scratch, uint32_t* counter, uint32_t* n_keys,
                      unsigned long long* n_keys_total, uint2* ranges, int n_tiles,
                      int tile_passes, uint32_t* tile_hist, uint32_t* tile_hist_done,
                      cudaStream_t st);
// Empty tiles of the ranges the tile sort's epilogue wrote get (s, s), s = the start of the
// next non-empty tile (n if none) — the position the tile would occupy, like the oracle.
void launch_ranges_fix(const uint32_t* n_keys, int64_t key_cap, int n_tiles, uint2* ranges,
                       cudaStream_t st);

// ---- blending (k_blend.cu) ----------------------------------------------------------------
// sorted: per list entry (splat, gradient slot), tile-major, (depth, index) order per tile;
// submask: per list entry, the 4x4 sub-quarters of the tile the splat's 3-sigma circle reaches
// (bit 8 w + k: group k of warp w; the closest-point tests K6 makes anyway), written by a
// tracked forward for the backward of the same frame.
void launch_blend_fwd(const FrameParams& fp, const uint2* ranges, const uint2* sorted,
                      uint16_t* submask,
                      const RenderRec* rec, unsigned long long* total, int64_t key_cap,
                      float* out, float* t_last, uint32_t* n_proc, bool track, cudaStream_t st);
// (track: also write t_last / n_proc and submask, the backward's per-pixel and per-entry
// state; render-only frames skip that bookkeeping)
// Writes every pair's 2D gradient to partial[2 slot], partial[2 slot + 1].
// given_dldc: `target` is dL/dC (G = loss_scale * target) and tile_loss is not meaningful;
// otherwise G = 2 loss_scale (img - target) and tile_loss[t] = sum over the tile of |d|^2.
void launch_blend_bwd(const FrameParams& fp, const uint2* ranges, const uint2* sorted,
                      const uint16_t* submask, const RenderRec* rec, const unsigned long long* total, int64_t key_cap,
                      const float* img, const float* target, const float* t_last,
                      const uint32_t* n_proc, float loss_scale, float4* partial,
                      double* tile_loss, bool given_dldc, float* grad2d, cudaStream_t st);
// grad2d != nullptr: "direct" accumulation -- each sub-quarter's pre-reduced gradients are
// added (red.global.add.v2.f32) into grad2d[splat] (n x 8: sum go dx, sum go dy, sum go r2,
// sum go, drgb, 0; unscaled), which K8 reads densely, scales and re-zeroes.  Not bitwise
// deterministic (L2 reduction order); the slot mode (grad2d == nullptr) is.

// ---- L1 + D-SSIM image loss (k_ssim.cu) ---------------------------------------------------
constexpr int kSsimHalf = 5;  // 11-tap window
int64_t ssim_part_count(int W, int H);  // double2 partials per frame
// loss = weight ((1-lambda) L1 + lambda (1 - SSIM)) of fhat against target: *accum += loss
// (if not null), *set = loss.  grad: also dL/dfhat (weight included) into dldc (HWC3), using
// coef (9 W H floats) as scratch.  lambda == 0 skips SSIM (needs W, H >= 11 otherwise).
// total/key_cap (may be null): a frame whose key capacity overflowed contributes nothing.
// Returns the number of kernels launched.
int launch_image_loss(int W, int H, const float* fhat, const float* target, float lambda,
                       double weight, bool grad, float* coef, double2* part, float* dldc,
                       const unsigned long long* total, int64_t key_cap, double* accum,
                       double* set, cudaStream_t st);
// dldc = scale (fhat - target) elementwise (the mse pixel gradient, scale = 2 w / (3 W H))
void launch_l2_grad(int W, int H, const float* fhat, const float* target, float scale,
                    float* dldc, cudaStream_t st);
// s = scale * sum(tile_loss) (fixed order); *accum += s (if accum), *set = s
void launch_loss_reduce(const double* tile_loss, int n_tiles, double scale, double* accum,
                        double* set, cudaStream_t st);
// tile_loss[t] = sum over tile t of |img - target|^2 (evaluation without gradients)
void launch_l2_tiles(const FrameParams& fp, const float* img, const float* target,
                     double* tile_loss, cudaStream_t st);

// ---- optimizer (k_adam.cu) ----------------------------------------------------------------
// Adam scalars live in device memory (AdamState), written by k_adam_tick once per step from
// the step counter on the device, so a captured CUDA graph replays correct bias corrections.
struct AdamParams {
  float lr[4];
  float b1, b2, eps;
  float step_size[4];  // lr / (1 - b1^t)
  float bc2_sqrt;      // sqrt(1 - b2^t)
  float inv_bc2_sqrt;  // 1 / sqrt(1 - b2^t)
};
struct AdamState {
  AdamParams p;
  long long t;  // steps taken
};

// t += 1, bias corrections of step t into st->p; moves the step's accumulated loss
// (loss[0]) to loss[2] and restarts the accumulator.
// A no-op (no tick) while total[kTotalOverflowMax] is set.
void launch_adam_tick(const float lr[4], float b1, float b2, float eps, AdamState* st_dev,
                      double* loss, const unsigned long long* total, cudaStream_t st);
// Optimizer-space state raw[i] = (log sigma, logit clamp(opacity)) of the splats as set.
constexpr float kOpacityEps = 1e-6f;
void launch_raw_init(const float4* ms, const float4* co, int64_t n, float2* raw, cudaStream_t st);

// Splat g's slots: slot_of[slot_off[g] + k] (or slot_off[g] + k when slot_of is null).
// K8a: 2D grads of one view -> 3D grads (overwrite when `first`, else accumulate).
// grad2d != nullptr: direct mode (dense sums, read and re-zeroed; co supplies the opacity).
void launch_project_backward(const float4* ms, const float4* co, int64_t n,
                             const FrameParams& fp, const uint32_t* slot_off,
                             const uint32_t* slot_of, const uint32_t* ntiles,
                             const float4* partial, float* grad2d,
                             const unsigned long long* total, int64_t cap, float4* grad3d,
                             bool first, cudaStream_t st, int64_t begin = 0, int64_t end = -1);
// Multi-GPU exchange slots (kMaxRanks float4 ahead of the gradient buffer): pack this rank's
// step loss (exact double as three floats) and overflow flag; unpack after the all-reduce.
constexpr int kMaxRanks = 64;
constexpr int kMaxExchangeChunks = 8;  // pipelined all-reduce chunks (isg_set_exchange_chunks)
void launch_loss_pack(const double* loss, const unsigned long long* total, float4* slots,
                      int rank, int nranks, cudaStream_t st);
void launch_loss_unpack(double* loss, unsigned long long* total, const float4* slots, int nranks,
                        cudaStream_t st);
// K8 fused: 2D grads of one view -> 3D -> Adam.
void launch_project_adam(float4* ms, float4* co, int64_t n, const FrameParams& fp,
                         const uint32_t* slot_off, const uint32_t* slot_of,
                         const uint32_t* ntiles, const float4* partial, float* grad2d,
                         unsigned long long* total, float2* raw, float4* m, float4* v,
                         const AdamState* ap, cudaStream_t st);
// K8b: Adam from accumulated 3D grads.
void launch_adam(float4* ms, float4* co, int64_t n, const float4* grad3d, float2* raw, float4* m,
                 float4* v, const AdamState* ap, unsigned long long* total, cudaStream_t st);

// ---- adaptive control (k_adapt.cu) ----------------------------------------------------------
struct AdaptParamsDev {
  double prune_threshold, merge_distance_factor, merge_color_tol, split_sigma_max;
  int64_t max_particles;  // effective cap
};
struct AdaptCounts {
  int64_t n_before, n_pruned, n_merged, n_split, n_after;
};
// Persistent device / pinned scratch of adaptive_control (grown on demand, reused across calls:
// per-call allocations dominated a pass).  Owned by the context; free with adapt_scratch_free.
struct AdaptScratch;
void adapt_scratch_free(AdaptScratch* s);
// Prune -> merge -> split of the n splats in (ms, co), in place; ms/co may be swapped with the
// scratch's temporaries (all hold >= n_alloc >= max(n, max_particles) records).  keys/vals:
// two ping-pong pairs of >= n words; sort: radix scratch for >= n items.  Synchronises.
cudaError_t adaptive_control(float4*& ms, float4*& co, int64_t n, int64_t n_alloc,
                             const AdaptParamsDev& p, uint64_t seed, uint64_t round,
                             SortScratch& sort, uint32_t* keys[2], uint32_t* vals[2],
                             AdaptScratch*& scratch, AdaptCounts* counts, cudaStream_t st,
                             int64_t* launches);

// measurement hook: per-pixel walk of the last frame's lists until termination; out[0] +=
// entries evaluated, out[1] += entries inside their 3-sigma circle (out zeroed by the caller)
void launch_count_pairs(const FrameParams& fp, const uint2* ranges, const uint2* sorted,
                        const RenderRec* rec, unsigned long long* out, cudaStream_t st);

// ---- parity hook -------------------------------------------------------------------------
void launch_debug_keys(const uint2* ranges, const uint2* sorted, const float4* ms,
                       const FrameParams& fp, uint64_t* keys, uint32_t* gids, cudaStream_t st);

}  // namespace isg

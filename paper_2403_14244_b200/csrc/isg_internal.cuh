// isg_internal.cuh — shared definitions of the sm_100a kernels and the C-ABI layer.
//
// Pipeline of one view (all on one stream, no host sync inside a frame):
//   K1  k_preprocess      per splat: validate, project, 3-sigma radius, tile count, depth key
//   K4a radix sort        (depth key, splat) over all splats           -> depth order
//   K2/3 k_scan_emit      decoupled look-back scan of tile counts in depth order, gather of
//                         the depth-ordered render records, emission of (tile, rank) pairs
//   K4b radix sort        (tile, rank) pairs, stable                   -> per-tile depth order
//   K5  k_ranges          per-tile [start, end)
//   K6  k_blend_fwd       16x16-tile front-to-back blend with early termination
//   K7  k_blend_bwd       reverse walk + fused L2 gradient, per-splat 2D grads
//   K8  k_project_adam    projection backward (+ Adam when fused)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/isg.h"

namespace isg {

constexpr int kTile = ISG_TILE;
constexpr int kTilePixels = kTile * kTile;
constexpr float kNearPlane = 1e-3f;  // splat3d.hpp:55

// ---- per-frame constant parameters --------------------------------------------------------
struct FrameParams {
  isg_camera cam;
  int tiles_x, tiles_y, n_tiles;
  float bg[3];
  float t_min;
};

// Render record of one visible splat, gathered into depth order (32 B, two float4):
//   geo = (u, v, sigma2d, r2max = (9*sigma2d)*sigma2d),   col = (r, g, b, opacity)
struct __align__(16) RenderRec {
  float4 geo;
  float4 col;
};

// ---- radix sort (onesweep, 8-bit digits, u32 keys + u32 values) ---------------------------
constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;  // items per thread
constexpr int kSortTileItems = kSortThreads * kSortItems;
constexpr int kMaxPasses = 4;

struct SortScratch {
  uint32_t* hist;       // kMaxPasses x 256 global digit histograms
  uint32_t* lookback;   // kMaxPasses x max_tiles x 256 status words
  uint32_t* counters;   // kMaxPasses dynamic tile counters
  int64_t max_tiles;    // per pass
};

inline int64_t sort_tiles_for(int64_t cap) { return (cap + kSortTileItems - 1) / kSortTileItems; }

// Stable LSD sort of n (device count *n_dev, <= cap) pairs on bits [0, key_bits).  keys/vals
// are ping-pong buffers; returns the index (0/1) of the buffer holding the result.  With
// iota_vals the first pass uses the item index as the value (vals[0] is not read).
int radix_sort_pairs(uint32_t* keys[2], uint32_t* vals[2], bool iota_vals, const uint32_t* n_dev,
                     int64_t cap, int key_bits, SortScratch& s, cudaStream_t st,
                     int64_t* launches);

// ---- launchers ----------------------------------------------------------------------------
// K1.  Also writes *n_dev = n (device-side count for the depth sort).
void launch_preprocess(const float4* ms, const float4* co, int64_t n, const FrameParams& fp,
                       float4* rec_geo, uint32_t* depth_key, uint32_t* ntiles,
                       uint32_t* first_bad, uint32_t* n_dev, cudaStream_t st);

// K2/K3: scan of ntiles in depth order, record gather, emission of the (tile, splat) pairs.
// Pair e (the emission slot) gets tile_keys[e] = tile and emit_rank[e] = depth rank; splat g's
// pairs occupy slots [emit_off[g], emit_off[g] + ntiles[g]).
// scratch: scan_emit_scratch_words(n) + 1 zeroed u64 words; counter: zeroed u32.
int64_t scan_emit_scratch_words(int64_t n);
void launch_scan_emit(const uint32_t* order, const uint32_t* ntiles, const float4* rec_geo,
                      const float4* co, int64_t n, const FrameParams& fp, RenderRec* rec_sorted,
                      uint32_t* emit_off, uint32_t* tile_keys, uint32_t* emit_rank,
                      int64_t key_cap, unsigned long long* scratch, uint32_t* counter,
                      uint32_t* n_keys, unsigned long long* n_keys_total, uint32_t* n_visible,
                      cudaStream_t st);

void launch_ranges(const uint32_t* sorted_tiles, const uint32_t* n_keys, int64_t key_cap,
                   uint2* ranges, cudaStream_t st);

// K6.  vals: emission slots sorted by (tile, depth, index).
void launch_blend_fwd(const FrameParams& fp, const uint2* ranges, const uint32_t* vals,
                      const uint32_t* emit_rank, const RenderRec* rec,
                      const unsigned long long* total, int64_t key_cap, float* out, float* t_last,
                      uint32_t* n_proc, cudaStream_t st);

// K7.  Writes every pair's 2D gradient to partial[2e], partial[2e+1] (emission slot e).
void launch_blend_bwd(const FrameParams& fp, const uint2* ranges, const uint32_t* vals,
                      const uint32_t* emit_rank, const RenderRec* rec,
                      const unsigned long long* total, int64_t key_cap, const float* img,
                      const float* target, const float* t_last, const uint32_t* n_proc,
                      float loss_scale, float4* partial, double* tile_loss, cudaStream_t st);

// loss[0] += scale * sum(tile_loss), loss[1] = scale * sum(tile_loss)
void launch_loss_reduce(const double* tile_loss, int n_tiles, double scale, double* loss,
                        cudaStream_t st);

struct AdamParams {
  float lr[4];
  float b1, b2, eps;
  float step_size[4];  // lr / (1 - b1^t)
  float bc2_sqrt;      // sqrt(1 - b2^t)
};

// K8a: 2D grads of one view -> 3D grads (overwrite when `first`, else accumulate).
void launch_project_backward(const float4* ms, int64_t n, const FrameParams& fp,
                             const uint32_t* emit_off, const uint32_t* ntiles,
                             const float4* partial, const unsigned long long* total, int64_t cap,
                             float4* grad3d, bool first, cudaStream_t st);
// K8 fused: 2D grads of one view -> 3D -> Adam.
void launch_project_adam(float4* ms, float4* co, int64_t n, const FrameParams& fp,
                         const uint32_t* emit_off, const uint32_t* ntiles, const float4* partial,
                         const unsigned long long* total, int64_t cap, float4* m, float4* v,
                         const AdamParams& ap, unsigned long long* skipped, cudaStream_t st);
// K8b: Adam from accumulated 3D grads.
void launch_adam(float4* ms, float4* co, int64_t n, const float4* grad3d, float4* m, float4* v,
                 const AdamParams& ap, unsigned long long* skipped, cudaStream_t st);

void launch_debug_keys(const uint32_t* tiles, const uint32_t* slots, const uint32_t* emit_rank,
                       const uint32_t* order, const float4* ms, const FrameParams& fp,
                       int64_t nkeys, uint64_t* keys, uint32_t* gids, cudaStream_t st);

}  // namespace isg

// K2-K5 — binning: scan + emission, onesweep LSD radix sort, per-tile ranges.
//
// Replaces the reference's single global std::stable_sort on double depth
// (/root/reference/proj/src/splat3d.cpp:164-169, ties broken by input index) with the
// tile-binned order the blend kernels need: per 16x16 tile, splats in (depth, index) order.
//
//   1. radix sort (depth bits, splat) over all splats          -> rank r = depth order
//   2. k_scan_emit: decoupled look-back exclusive scan of the tile counts in rank order and
//      emission of (tile, splat) pairs in rank order (so equal tiles already appear in depth
//      order), staged per CTA in shared memory and written coalesced
//   3. radix sort (tile, emission index) — stable, only ceil(log2(tiles)) bits; its last
//      pass writes the (splat, slot) pairs in final order and the tile runs' bounds
//   4. k_ranges_fix: empty tiles get (s, s) at the position they would occupy
//
// The radix sort is a onesweep LSD sort (one kernel per 8-bit digit pass plus one upfront
// histogram kernel): every CTA takes a dynamic tile id, ranks its 2048 keys stably with a
// ballot-based warp multisplit, publishes per-digit counts to a decoupled look-back array,
// scatters through shared memory and writes coalesced runs per digit.
#include <algorithm>

#include "isg_math.cuh"
#include "lookback.cuh"
#include "radix_hist.cuh"

#ifndef ISG_HIST_MODE
#define ISG_HIST_MODE 2
#endif
#ifndef ISG_EPI_PREFETCH
#define ISG_EPI_PREFETCH 1
#endif
#ifndef ISG_LOOKBACK_WIN
#define ISG_LOOKBACK_WIN 4
#endif
// ISG_LOOKBACK_GROUP (tiles per level-2 group) is defined in isg_internal.cuh, which sizes the
// look-back rows by it

namespace isg {

namespace {

constexpr int kLbWin = ISG_LOOKBACK_WIN;      // level-2 rows read per round trip (4: +0.2% vs 8)
constexpr int kLbGroup = ISG_LOOKBACK_GROUP;  // tiles per level-2 group
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kCountMask = (1u << 30) - 1;

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  return *(const volatile uint32_t*)p;
}
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) {
  *(volatile uint32_t*)p = v;
}

// Lanes of the warp holding the same 9-bit value (digit, or 256 = no item): 9 ballots instead of
// one match.any (a slow MIO-pipe instruction on this part).
#ifndef ISG_MATCH_PTX
#define ISG_MATCH_PTX 1
#endif
__device__ __forceinline__ uint32_t warp_match9(uint32_t d) {
  uint32_t peers = 0xffffffffu;
#if ISG_MATCH_PTX
  // per bit: the bit as a predicate (ptxas sets several at once with R2P), its ballot, the
  // lane's all-ones / all-zeros mask from the same predicate, one LOP3 peers &= ~(ballot ^
  // mask) — about 3.3 instructions per bit where the C++ form compiles to six.  Depth sort
  // 0.0633 -> 0.0575 ms, tile sort 0.0751 -> 0.0674 ms (C3).
#pragma unroll
  for (int b = 0; b < 9; ++b) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 t, m, s;\n\t"
        "and.b32 t, %1, %2;\n\t"
        "setp.ne.u32 p, t, 0;\n\t"
        "vote.sync.ballot.b32 m, p, 0xffffffff;\n\t"
        "selp.b32 s, -1, 0, p;\n\t"
        "lop3.b32 %0, %0, m, s, 0x90;\n\t}"  // a & ~(b ^ c)
        : "+r"(peers)
        : "r"(d), "r"(1u << b));
  }
#else
#pragma unroll
  for (int b = 0; b < 9; ++b) {
    const bool bit = (d >> b) & 1u;
    const uint32_t m = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? m : ~m;
  }
#endif
  return peers;
}

// ---- upfront histogram of all passes -------------------------------------------------------
// (Not used by the frame's two sorts: their producers, k_preprocess and k_scan_emit, build the
// same histograms while writing the keys; see radix_hist.cuh.)
__global__ void __launch_bounds__(256) k_hist(const uint32_t* __restrict__ keys,
                                              const uint32_t* __restrict__ n_dev, int64_t cap,
                                              int passes, uint32_t* __restrict__ hist,
                                              uint32_t* __restrict__ done) {
  pdl_enter();
  __shared__ uint32_t sh[kMaxPasses][256];
  hist_zero(sh);
  __syncthreads();
  const int64_t n = min((int64_t)*n_dev, cap);
  // grid-stride over whole warps, kHistUnroll keys per thread in flight at once
  constexpr int kHistUnroll = 8;
  const int64_t stride = (int64_t)gridDim.x * 256 * kHistUnroll;
  for (int64_t i0 = ((int64_t)blockIdx.x * 256 + (threadIdx.x & ~31)) * kHistUnroll; i0 < n;
       i0 += stride) {
    uint32_t k[kHistUnroll];
    bool valid[kHistUnroll];
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      const int64_t i = i0 + 32 * u + (threadIdx.x & 31);
      valid[u] = i < n;
      k[u] = valid[u] ? keys[i] : 0u;
    }
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) hist_add_warp(sh, k[u], valid[u], passes);
  }
  hist_publish(sh, passes, hist, done);
}

// ---- one onesweep digit pass -----------------------------------------------------------------
struct OnesweepSmem {
  uint32_t keys[kSortTileItems];
  uint32_t vals[kSortTileItems];
  uint32_t wcnt[kSortThreads / 32][257];
  uint32_t local_start[256];
  uint32_t bin_base[256];
  uint32_t warp_tmp[8];
  uint32_t tile;
  uint32_t gids[kSortTileItems];  // epilogue pass only: splat of each item
};

template <bool kEpi>
// A 4-CTA minimum per SM (64 registers): the PTX ballot match lets ptxas batch the ballots of
// several items and take 77 registers (3 CTAs) otherwise — depth sort 0.0578 vs 0.0575 ms,
// tile sort 0.0739 vs 0.0674.  (5 / 6 CTAs: spills, equal or slower.)
#ifndef ISG_SORT_MINB
#define ISG_SORT_MINB 4
#endif
#if ISG_SORT_MINB > 0
#define ISG_SORT_BOUNDS __launch_bounds__(kSortThreads, ISG_SORT_MINB)
#else
#define ISG_SORT_BOUNDS __launch_bounds__(kSortThreads)
#endif
__global__ void ISG_SORT_BOUNDS k_onesweep(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
    const uint32_t* __restrict__ n_dev, int64_t cap, int shift,
    const uint32_t* __restrict__ hist, uint32_t* __restrict__ lookback,
    uint32_t* __restrict__ counter, SortEpilogue epi) {
  pdl_enter();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  OnesweepSmem& S = *reinterpret_cast<OnesweepSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t n = min((int64_t)*n_dev, cap);
  if (tid == 0) S.tile = atomicAdd(counter, 1u);
  for (int i = tid; i < (kSortThreads / 32) * 257; i += kSortThreads) (&S.wcnt[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = S.tile;
  const int64_t base = (int64_t)tile * kSortTileItems;
  if (base >= n) return;

  uint32_t key[kSortItems], val[kSortItems], rank[kSortItems], dig[kSortItems];
  const int64_t wbase = base + (int64_t)w * 32 * kSortItems + lane;
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t idx = wbase + j * 32;
    const bool valid = idx < n;
    key[j] = valid ? keys_in[idx] : 0u;
    val[j] = valid ? (vals_in ? vals_in[idx] : (uint32_t)idx) : 0u;
    dig[j] = valid ? ((key[j] >> shift) & 255u) : 256u;
  }
  // epilogue: the splat gathers are issued now and land during the ranking and look-back
  uint32_t gid[kEpi ? kSortItems : 1];
  if constexpr (kEpi) {
#pragma unroll
    for (int j = 0; j < kSortItems; ++j)
      gid[j] = ISG_EPI_PREFETCH && !epi.vals_are_gids && dig[j] < 256u ? epi.emit_gid[val[j]] : 0u;
  }
  // stable warp multisplit: rank = items of the same digit earlier in (iteration, lane) order
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const uint32_t d = dig[j];
    const uint32_t peers = warp_match9(d);
    // only each digit's leader lane touches the counter; the others get it by shuffle, so
    // one __syncwarp per round orders the rounds
    const int leader = __ffs(peers) - 1;
    uint32_t before = 0;
    if (lane == leader) before = S.wcnt[w][d];
    before = __shfl_sync(0xffffffffu, before, leader);
    rank[j] = before + __popc(peers & lt);
    if (lane == leader) S.wcnt[w][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive prefix across warps; tile count
  uint32_t cnt = 0;
#pragma unroll
  for (int ww = 0; ww < kSortThreads / 32; ++ww) {
    const uint32_t c = S.wcnt[ww][tid];
    S.wcnt[ww][tid] = cnt;
    cnt += c;
  }
  // publish this tile's aggregate (or inclusive prefix for tile 0) as early as possible
  // level 1: this tile's per-digit count, published as early as possible (never upgraded)
  st_volatile(lookback + (int64_t)tile * 256 + tid, kFlagAgg | cnt);
  uint32_t tot;
  const uint32_t local_start = block_excl_scan_256(cnt, S.warp_tmp, tot);
  S.local_start[tid] = local_start;
  __syncthreads();
  // scatter into shared memory in tile-sorted order (independent of the global offsets, so the
  // per-item registers are dead before the look-back)
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const uint32_t d = dig[j];
    if (d < 256u) {
      const uint32_t pos = S.local_start[d] + S.wcnt[w][d] + rank[j];
      S.keys[pos] = key[j];
      S.vals[pos] = val[j];
      if constexpr (kEpi) S.gids[pos] = gid[j];
    }
  }
  const uint32_t gpre = hist[tid];  // exclusive digit offset (k_hist's last block scanned)
  // Two-level decoupled look-back for digit `tid`.  Tiles form groups of kLbGroup; a tile sums
  // the counts of the earlier tiles of its own group (level 1, one round of loads), and the
  // prefix of all earlier groups from the level-2 words: each group's last tile publishes the
  // group's count (AGG) as soon as it has read its group, and the inclusive prefix through the
  // group (INC) once it knows the group's start.  A tile therefore reads at most kLbGroup - 1
  // level-1 rows and one row per earlier group back to the nearest inclusive one, instead of
  // every earlier tile's row when the whole pass is resident at once (one wave: small sorts).
  uint32_t excl = 0;
  {
    uint32_t* const l2 = lookback + 256 * ((cap + kSortTileItems - 1) / kSortTileItems);
    const int64_t g = (int64_t)tile / kLbGroup;
    const int r = (int)((int64_t)tile - g * kLbGroup);
    uint32_t sw[kLbGroup - 1];
#pragma unroll
    for (int q = 0; q < kLbGroup - 1; ++q)
      sw[q] = q < r ? ld_volatile(lookback + ((int64_t)tile - 1 - q) * 256 + tid) : kFlagAgg;
#pragma unroll
    for (int q = 0; q < kLbGroup - 1; ++q) {
      if (q < r) {
        while ((sw[q] & ~kCountMask) == 0)
          sw[q] = ld_volatile(lookback + ((int64_t)tile - 1 - q) * 256 + tid);
        excl += sw[q] & kCountMask;
      }
    }
    const bool last = r == kLbGroup - 1;
    if (last) st_volatile(l2 + g * 256 + tid, (g == 0 ? kFlagInc : kFlagAgg) | (excl + cnt));
    if (g > 0) {
      uint32_t gp = 0;
      int64_t p = g - 1;
      bool found = false;
      while (!found) {
        uint32_t w2[kLbWin];
#pragma unroll
        for (int q = 0; q < kLbWin; ++q)
          w2[q] = p - q >= 0 ? ld_volatile(l2 + (p - q) * 256 + tid) : kFlagInc;
#pragma unroll
        for (int q = 0; q < kLbWin; ++q) {
          if (found) break;
          while ((w2[q] & ~kCountMask) == 0) w2[q] = ld_volatile(l2 + (p - q) * 256 + tid);
          gp += w2[q] & kCountMask;
          found = (w2[q] & ~kCountMask) == kFlagInc;
        }
        p -= kLbWin;
      }
      if (last) st_volatile(l2 + g * 256 + tid, kFlagInc | (gp + excl + cnt));
      excl += gp;
    }
  }
  S.bin_base[tid] = gpre + excl - local_start;
  __syncthreads();
  const int nvalid = (int)min((int64_t)kSortTileItems, n - base);
  if constexpr (kEpi) {
    // last pass of the tile sort: (splat, slot) pairs in final order, and the tile runs'
    // bounds.  Items adjacent in shared memory with the same digit are adjacent in the output,
    // so a run's first / last item here bounds the tile's range; runs continuing in other
    // tiles of the sort are merged by the atomics.
    for (int i = tid; i < nvalid; i += kSortThreads) {
      const uint32_t k = S.keys[i];
      const uint32_t o = S.bin_base[(k >> shift) & 255u] + (uint32_t)i;
      const uint32_t v = S.vals[i];
      epi.sorted[o] = epi.vals_are_gids
                          ? make_uint2(v, o)
                          : make_uint2(ISG_EPI_PREFETCH ? S.gids[i] : epi.emit_gid[v], v);
      if (i == 0 || S.keys[i - 1] != k) atomicMin(&epi.ranges[k].x, o);
      if (i == nvalid - 1 || S.keys[i + 1] != k) atomicMax(&epi.ranges[k].y, o + 1u);
    }
  } else {
    for (int i = tid; i < nvalid; i += kSortThreads) {
      const uint32_t k = S.keys[i];
      const uint32_t o = S.bin_base[(k >> shift) & 255u] + (uint32_t)i;
      keys_out[o] = k;
      vals_out[o] = S.vals[i];
    }
  }
}

// ---- ranges fix-up ---------------------------------------------------------------------------
// The tile sort's epilogue left empty tiles at (0xFFFFFFFF, 0).  One CTA: each thread takes a
// contiguous segment of tiles, a block-wide suffix minimum over the segments' smallest starts
// gives every empty tile the start of the next non-empty tile (n when none follows).
constexpr int kFixThreads = 1024;
__global__ void __launch_bounds__(kFixThreads) k_ranges_fix(const uint32_t* __restrict__ n_dev,
                                                            int64_t cap, int n_tiles,
                                                            uint2* __restrict__ ranges) {
  __shared__ uint32_t s_min[kFixThreads];
  const int64_t n = min((int64_t)*n_dev, cap);
  const int tid = threadIdx.x;
  const int seg = (n_tiles + kFixThreads - 1) / kFixThreads;
  const int k0 = min(tid * seg, n_tiles), k1 = min(k0 + seg, n_tiles);
  if (n == 0) {
    for (int k = k0; k < k1; ++k) ranges[k] = make_uint2(0u, 0u);
    return;
  }
  uint32_t m = 0xFFFFFFFFu;
  for (int k = k0; k < k1; ++k) m = min(m, ranges[k].x);
  s_min[tid] = m;
  __syncthreads();
  // inclusive suffix minimum (Hillis-Steele)
  for (int o = 1; o < kFixThreads; o <<= 1) {
    const uint32_t other = tid + o < kFixThreads ? s_min[tid + o] : 0xFFFFFFFFu;
    __syncthreads();
    s_min[tid] = min(s_min[tid], other);
    __syncthreads();
  }
  uint32_t next = tid + 1 < kFixThreads ? s_min[tid + 1] : 0xFFFFFFFFu;
  if (next == 0xFFFFFFFFu) next = (uint32_t)n;
  for (int k = k1 - 1; k >= k0; --k) {
    const uint2 r = ranges[k];
    if (r.x == 0xFFFFFFFFu) {
      ranges[k] = make_uint2(next, next);
    } else {
      next = r.x;
    }
  }
}

// ---- scan of tile counts in depth order + record gather + emission --------------------------
constexpr int kScanThreads = 256;
#ifndef ISG_SCAN_ITEMS
#define ISG_SCAN_ITEMS 4
#endif
constexpr int kScanItems = ISG_SCAN_ITEMS;
constexpr int kScanTileItems = kScanThreads * kScanItems;
// Staged keys per window (16 KB of shared memory) with a 6-CTA minimum per SM (40 registers):
// C3 0.049 ms vs 0.052 for 4096-key windows at 4 CTAs / SM.
#ifndef ISG_EMIT_WINDOW
#define ISG_EMIT_WINDOW 2048
#endif
constexpr int kEmitWindow = ISG_EMIT_WINDOW;

#ifndef ISG_SCAN_MINB
#define ISG_SCAN_MINB 6
#endif
__global__ void __launch_bounds__(kScanThreads, ISG_SCAN_MINB) k_scan_emit(
    const uint32_t* __restrict__ order, const uint32_t* __restrict__ ntiles,
    const uint2* __restrict__ tilebox, const float4* __restrict__ ms, int64_t n, FrameParams fp,
    uint32_t* __restrict__ slot_off, uint32_t* __restrict__ tile_keys,
    uint32_t* __restrict__ emit_gid, int64_t key_cap,
    unsigned long long* __restrict__ lookback, uint32_t* __restrict__ counter,
    uint32_t* __restrict__ n_keys, unsigned long long* __restrict__ n_keys_total,
    uint2* __restrict__ ranges, int n_tiles, int tile_passes, uint32_t* __restrict__ tile_hist,
    uint32_t* __restrict__ tile_hist_done) {
  pdl_enter();
  __shared__ uint32_t sh[kMaxPasses][256];  // the tile sort's digit histograms
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp[8];
  __shared__ unsigned long long s_excl;
  __shared__ uint32_t s_emit_key[kEmitWindow];
  __shared__ uint32_t s_emit_gid[kEmitWindow];
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(counter, 1u);
  hist_zero(sh);
  // empty ranges for the tile sort's epilogue (its atomics run after this kernel)
  for (int k = blockIdx.x * kScanThreads + tid; k < n_tiles; k += gridDim.x * kScanThreads)
    ranges[k] = make_uint2(0xFFFFFFFFu, 0u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base = (int64_t)tile * kScanTileItems;
  if (base >= n) return;
  const int64_t r0 = base + (int64_t)tid * kScanItems;
  uint32_t g[kScanItems], c[kScanItems];
  uint2 box[kScanItems];
  uint32_t sum = 0;
  // all gathers of the thread's splats in flight before the scan (the emission needs them)
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) g[j] = r0 + j < n ? order[r0 + j] : 0u;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const bool ok = r0 + j < n;
    box[j] = ok ? tilebox[g[j]] : make_uint2(0u, 0u);
    c[j] = tilebox_count(box[j]);
    sum += c[j];
  }
  uint32_t tot;
  const uint32_t t_begin = block_excl_scan_256(sum, s_warp, tot);
  const uint32_t t_end = t_begin + sum;  // this thread's range, CTA-relative
  // warp 0 runs the decoupled look-back for the CTA's global offset while the other warps
  // already stage the first window (staging needs only CTA-relative positions)
  if (tid < 32) {
    const unsigned long long excl = lookback_warp(lookback, tile, tot);
    if (tid == 0) {
      s_excl = excl;
      if (base + kScanTileItems >= n) {
        const unsigned long long total = excl + tot;
        *n_keys_total = total;
        *n_keys = (uint32_t)min((unsigned long long)key_cap, total);
      }
    }
  }
  unsigned long long cta0 = 0;
#define ISG_WRITE_SLOT_OFFSETS()                                                   \
  do {                                                                             \
    cta0 = s_excl;                                                                 \
    uint32_t pos_ = t_begin;                                                       \
    _Pragma("unroll") for (int j = 0; j < kScanItems; ++j) {                       \
      if (slot_off && r0 + j < n) slot_off[g[j]] = (uint32_t)min(cta0 + pos_, 0xFFFFFFFFull); \
      pos_ += c[j];                                                                \
    }                                                                              \
  } while (0)
  // Emission.  The CTA's keys occupy one contiguous range [s_excl, s_excl + tot) of the
  // output, so they are staged in shared memory window by window and written back coalesced
  // (per-thread emission straight to global memory scatters every store across 32 lines).
  // An item straddling a window boundary is enumerated again in the next window.
  for (uint32_t w = 0; w < tot; w += kEmitWindow) {
    const uint32_t wend = w + kEmitWindow;
    if (t_begin < wend && t_end > w) {
      uint32_t pos = t_begin;
#pragma unroll
      for (int j = 0; j < kScanItems; ++j) {
        const uint32_t p0 = pos;
        pos += c[j];
        if (c[j] == 0 || pos <= w || p0 >= wend) continue;
        const float4 m = (box[j].x >> 24) ? make_float4(0.f, 0.f, 0.f, 0.f) : ms[g[j]];
        uint32_t q = p0;
        const uint32_t gg = g[j];
        for_each_tile(box[j], m, fp, [&](int t) {
          if (q >= w && q < wend) {
            s_emit_key[q - w] = (uint32_t)t;
            s_emit_gid[q - w] = gg;
          }
          ++q;
        });
      }
    }
    __syncthreads();  // window staged (and, the first time, s_excl published)
    if (w == 0) ISG_WRITE_SLOT_OFFSETS();
    const uint32_t cnt = min(tot - w, (uint32_t)kEmitWindow);
    const unsigned long long o0 = cta0 + w;
    for (uint32_t i0 = 0; i0 < cnt; i0 += kScanThreads) {  // warp-uniform trip count
      const uint32_t i = i0 + tid;
      const bool ok = i < cnt && o0 + i < (unsigned long long)key_cap;
      const uint32_t k = ok ? s_emit_key[i] : 0u;
      if (ok) {
        tile_keys[o0 + i] = k;
        emit_gid[o0 + i] = s_emit_gid[i];
      }
      hist_add_warp(sh, k, ok, tile_passes);  // only keys that are written are counted
    }
    __syncthreads();
  }
  if (tot == 0) {  // (CTA-uniform) no keys: the offsets still need s_excl
    __syncthreads();
    ISG_WRITE_SLOT_OFFSETS();
  }
#undef ISG_WRITE_SLOT_OFFSETS
  hist_publish(sh, tile_passes, tile_hist, tile_hist_done);
}

}  // namespace

int64_t scan_emit_scratch_words(int64_t n) { return (n + kScanTileItems - 1) / kScanTileItems; }

void launch_scan_emit(const uint32_t* order, const uint32_t* ntiles, const uint2* tilebox,
                      const float4* ms, int64_t n, const FrameParams& fp, uint32_t* slot_off,
                      uint32_t* tile_keys, uint32_t* emit_gid, int64_t key_cap,
                      unsigned long long* scratch, uint32_t* counter, uint32_t* n_keys,
                      unsigned long long* n_keys_total, uint2* ranges, int n_tiles,
                      int tile_passes, uint32_t* tile_hist, uint32_t* tile_hist_done,
                      cudaStream_t st) {
  const int64_t tiles = scan_emit_scratch_words(n);
  if (tiles == 0) return;  // caller zeroed the counts
  launch_pdl(k_scan_emit, dim3((unsigned)tiles), dim3(kScanThreads), 0, st, order, ntiles,
             tilebox, ms, n, fp, slot_off, tile_keys, emit_gid, key_cap, scratch, counter, n_keys,
             n_keys_total, ranges, n_tiles, tile_passes, tile_hist, tile_hist_done);
}

void launch_ranges_fix(const uint32_t* n_keys, int64_t key_cap, int n_tiles, uint2* ranges,
                       cudaStream_t st) {
  k_ranges_fix<<<1, kFixThreads, 0, st>>>(n_keys, key_cap, n_tiles, ranges);
}

int radix_sort_pairs(uint32_t* keys[2], uint32_t* vals[2], bool iota_vals, const uint32_t* n_dev,
                     int64_t cap, int key_bits, SortScratch& s, cudaStream_t st,
                     int64_t* launches, const SortOptions& opt) {
  const SortEpilogue& epi = opt.epi;
  const int passes = (key_bits + 7) / 8;
  const int64_t tiles = (cap + kSortTileItems - 1) / kSortTileItems;
  // caller guarantees tiles <= s.max_tiles and passes <= kMaxPasses
  if (!opt.scratch_zeroed) {
    cudaMemsetAsync(s.hist, 0, sizeof(uint32_t) * kMaxPasses * 256, st);
    cudaMemsetAsync(s.counters, 0, sizeof(uint32_t) * (kMaxPasses + 1), st);
    cudaMemsetAsync(s.lookback, 0, sizeof(uint32_t) * sort_lookback_words(tiles) * passes, st);
  }
  if (!opt.hist_ready) {
    const int hist_blocks = (int)std::min<int64_t>(std::max<int64_t>(tiles, 1), 148 * 4);
    launch_pdl(k_hist, dim3(hist_blocks), dim3(256), 0, st, (const uint32_t*)keys[0], n_dev,
               cap, passes, s.hist, s.counters + kMaxPasses);
  }
  int cur = 0;
  const size_t smem = sizeof(OnesweepSmem);
  static const bool attr_set = [&] {  // once, outside any graph capture
    cudaFuncSetAttribute(k_onesweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaFuncSetAttribute(k_onesweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    return true;
  }();
  (void)attr_set;
  for (int p = 0; p < passes; ++p) {
    const bool fin = p == passes - 1 && epi.sorted;
    launch_pdl(fin ? k_onesweep<true> : k_onesweep<false>,
               dim3((unsigned)std::max<int64_t>(tiles, 1)), dim3(kSortThreads), smem, st,
               (const uint32_t*)keys[cur], (const uint32_t*)((p == 0 && iota_vals) ? nullptr : vals[cur]),
               keys[cur ^ 1], vals[cur ^ 1], n_dev, cap, 8 * p, (const uint32_t*)(s.hist + 256 * p),
               s.lookback + sort_lookback_words(tiles) * p, s.counters + p,
               fin ? epi : SortEpilogue());
    cur ^= 1;
  }
  if (launches) *launches += (opt.hist_ready ? 0 : 1) + passes;
  return cur;
}

}  // namespace isg

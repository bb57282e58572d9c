// Binning, "tile-bucket" mode (default): counting sort by tile + per-tile sort by depth.
//
// Replaces the reference's global std::stable_sort on double depth
// (/root/reference/proj/src/splat3d.cpp:164-169, ties broken by splat index) with the per-tile
// order the blend kernels need, without any global radix pass:
//
//   K1  k_preprocess      counts each splat's tiles and atomically bumps per-tile counters
//   K2  k_tile_scan       one CTA: exclusive scan of the tile counters -> ranges, cursors
//   K3  k_fill            decoupled look-back scan of per-splat counts (slot lists) and
//                         emission of (depth bits << 32 | splat) into each tile's bucket via an
//                         atomic cursor (bucket order is arbitrary)
//   K4  k_tile_sort       one CTA per tile: bitonic sort of the bucket in shared memory by the
//                         64-bit key (depth, splat) -> exactly the (tile, depth, index) order of
//                         the oracle; emits (splat, slot) pairs for the blend kernels
//
// Every tile list of the BASELINE configs fits in shared memory (max 1568 entries at
// 3M/1080p); longer lists take a slower global-memory merge path inside the same kernel.
#include <algorithm>

#include "isg_math.cuh"
#include "lookback.cuh"

namespace isg {

namespace {

constexpr int kScanThreads = 1024;
constexpr int kFillThreads = 256;
constexpr int kFillItems = 4;
constexpr int kFillTile = kFillThreads * kFillItems;
// inclusive warp scan + block exclusive scan (blockDim.x threads, <= 32 warps)
__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v,
                                                              unsigned long long* s_warp,
                                                              unsigned long long& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    unsigned long long s = lane < nw ? s_warp[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) s_warp[lane] = s;  // inclusive prefix of warp totals
  }
  __syncthreads();
  total = s_warp[nw - 1];
  const unsigned long long wpre = w ? s_warp[w - 1] : 0ull;
  __syncthreads();
  return wpre + x - v;
}

}  // namespace

// ---- K2: tile offsets ------------------------------------------------------------------------
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(const uint32_t* __restrict__ cnt,
                                                            int n_tiles, int64_t cap,
                                                            uint2* __restrict__ ranges,
                                                            uint32_t* __restrict__ cursor,
                                                            uint32_t* __restrict__ n_keys,
                                                            unsigned long long* __restrict__ total) {
  __shared__ unsigned long long s_warp[32];
  const int per = (n_tiles + kScanThreads - 1) / kScanThreads;
  const int t0 = threadIdx.x * per;
  unsigned long long sum = 0;
  for (int i = 0; i < per; ++i)
    if (t0 + i < n_tiles) sum += cnt[t0 + i];
  unsigned long long tot;
  unsigned long long off = block_excl_scan(sum, s_warp, tot);
  for (int i = 0; i < per; ++i) {
    const int t = t0 + i;
    if (t >= n_tiles) break;
    const uint32_t c = cnt[t];
    const uint32_t s = (uint32_t)min(off, (unsigned long long)0xFFFFFFFFull);
    ranges[t] = make_uint2(s, (uint32_t)min(off + c, (unsigned long long)0xFFFFFFFFull));
    cursor[t] = s;
    off += c;
  }
  if (threadIdx.x == 0) {
    *total = tot;
    *n_keys = (uint32_t)min(tot, (unsigned long long)cap);
  }
}

// ---- K3: per-splat slot lists + bucket fill ---------------------------------------------------
__global__ void __launch_bounds__(kFillThreads) k_fill(
    const float4* __restrict__ ms, const uint32_t* __restrict__ ntiles,
    const uint2* __restrict__ tilebox, const uint32_t* __restrict__ depth_key, int64_t n,
    FrameParams fp, uint32_t* __restrict__ cursor, unsigned long long* __restrict__ bucket,
    uint32_t* __restrict__ slot_of, uint32_t* __restrict__ slot_off, int64_t cap,
    unsigned long long* __restrict__ lookback, uint32_t* __restrict__ counter) {
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_warp[32];
  __shared__ unsigned long long s_excl;
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base = (int64_t)tile * kFillTile;
  if (base >= n) return;
  const int64_t g0 = base + (int64_t)tid * kFillItems;
  uint32_t c[kFillItems];
  unsigned long long sum = 0;
#pragma unroll
  for (int j = 0; j < kFillItems; ++j) {
    c[j] = g0 + j < n ? ntiles[g0 + j] : 0u;
    sum += c[j];
  }
  unsigned long long tot;
  const unsigned long long texcl = block_excl_scan(sum, s_warp, tot);
  if (tid < 32) {
    const unsigned long long excl = lookback_warp(lookback, tile, tot);
    if (tid == 0) s_excl = excl;
  }
  __syncthreads();
  unsigned long long off = s_excl + texcl;
#pragma unroll
  for (int j = 0; j < kFillItems; ++j) {
    const int64_t g = g0 + j;
    if (g >= n) break;
    slot_off[g] = (uint32_t)min(off, (unsigned long long)0xFFFFFFFFull);
    if (c[j] == 0) continue;
    const unsigned long long key = ((unsigned long long)depth_key[g] << 32) | (uint32_t)g;
    const uint2 box = tilebox[g];
    const float4 m = (box.x >> 24) ? make_float4(0.f, 0.f, 0.f, 0.f) : ms[g];
    for_each_tile(box, m, fp, [&](int t) {
      const uint32_t slot = atomicAdd(&cursor[t], 1u);
      if (slot < (uint64_t)cap) bucket[slot] = key;
      if (off < (unsigned long long)cap) slot_of[off] = slot;
      ++off;
    });
  }
}

// ---- K4: per-tile sort ------------------------------------------------------------------------
constexpr int kSortCap = 2048;  // entries sorted in shared memory
constexpr int kTsThreads = 256;

__device__ __forceinline__ void bitonic_smem(unsigned long long* key, uint32_t* idx, int P) {
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < (P >> 1); i += blockDim.x) {
        const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
        const int hi = lo + j;
        const bool asc = (lo & k) == 0;
        const unsigned long long a = key[lo], b = key[hi];
        if ((a > b) == asc) {
          key[lo] = b;
          key[hi] = a;
          const uint32_t t = idx[lo];
          idx[lo] = idx[hi];
          idx[hi] = t;
        }
      }
      __syncthreads();
    }
  }
}

// Global-memory fallback for lists longer than kSortCap: sort runs of kSortCap in shared
// memory, then merge runs pairwise (merge path) between two scratch buffers carved out of the
// (not yet used) gradient-slot storage of this tile's range.
__device__ void long_list_sort(const unsigned long long* __restrict__ bucket, uint32_t start,
                               int L, unsigned long long* skey, uint32_t* sidx,
                               ulonglong2* bufA, ulonglong2* bufB, uint2* __restrict__ sorted) {
  for (int r0 = 0; r0 < L; r0 += kSortCap) {
    const int m = min(kSortCap, L - r0);
    int P = 1;
    while (P < m) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
      skey[i] = i < m ? bucket[start + r0 + i] : ~0ull;
      sidx[i] = (uint32_t)(r0 + i);
    }
    __syncthreads();
    bitonic_smem(skey, sidx, P);
    for (int i = threadIdx.x; i < m; i += blockDim.x)
      bufA[r0 + i] = make_ulonglong2(skey[i], (unsigned long long)sidx[i]);
    __syncthreads();
  }
  ulonglong2* src = bufA;
  ulonglong2* dst = bufB;
  for (int width = kSortCap; width < L; width <<= 1) {
    for (int r0 = 0; r0 < L; r0 += 2 * width) {
      const int a0 = r0, a1 = min(r0 + width, L), b1 = min(r0 + 2 * width, L);
      const int na = a1 - a0, nb = b1 - a1, tot = na + nb;
      const int per = (tot + blockDim.x - 1) / blockDim.x;
      const int d0 = min(tot, (int)threadIdx.x * per), d1 = min(tot, d0 + per);
      if (d0 < d1) {
        // merge path: find i in A, d0 - i in B
        int lo = max(0, d0 - nb), hi = min(d0, na);
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (src[a0 + mid].x <= src[a1 + d0 - 1 - mid].x) lo = mid + 1;
          else hi = mid;
        }
        int i = lo, j = d0 - lo;
        for (int d = d0; d < d1; ++d) {
          const bool takeA = j >= nb || (i < na && src[a0 + i].x <= src[a1 + j].x);
          dst[r0 + d] = takeA ? src[a0 + i++] : src[a1 + j++];
        }
      }
    }
    __syncthreads();
    ulonglong2* t = src;
    src = dst;
    dst = t;
  }
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    const ulonglong2 e = src[i];
    sorted[start + i] = make_uint2((uint32_t)e.x, start + (uint32_t)e.y);
  }
}

__global__ void __launch_bounds__(kTsThreads) k_tile_sort(
    const uint2* __restrict__ ranges, const unsigned long long* __restrict__ bucket,
    const unsigned long long* __restrict__ total, int64_t cap, uint2* __restrict__ sorted,
    float4* __restrict__ scratch) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* skey = reinterpret_cast<unsigned long long*>(smem_raw);
  uint32_t* sidx = reinterpret_cast<uint32_t*>(skey + kSortCap);
  if (*total > (unsigned long long)cap) return;
  const uint2 rg = ranges[blockIdx.x];
  const int L = (int)(rg.y - rg.x);
  if (L == 0) return;
  if (L > kSortCap) {
    ulonglong2* bufA = reinterpret_cast<ulonglong2*>(scratch + 2 * (size_t)rg.x);
    long_list_sort(bucket, rg.x, L, skey, sidx, bufA, bufA + L, sorted);
    return;
  }
  int P = 1;
  while (P < L) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    skey[i] = i < L ? bucket[rg.x + i] : ~0ull;
    sidx[i] = (uint32_t)i;
  }
  __syncthreads();
  bitonic_smem(skey, sidx, P);
  for (int i = threadIdx.x; i < L; i += blockDim.x)
    sorted[rg.x + i] = make_uint2((uint32_t)skey[i], rg.x + sidx[i]);
}

// ---- launchers --------------------------------------------------------------------------------
int64_t fill_scratch_words(int64_t n) { return (n + kFillTile - 1) / kFillTile; }

void launch_tile_scan(const uint32_t* cnt, int n_tiles, int64_t cap, uint2* ranges,
                      uint32_t* cursor, uint32_t* n_keys, unsigned long long* total,
                      cudaStream_t st) {
  k_tile_scan<<<1, kScanThreads, 0, st>>>(cnt, n_tiles, cap, ranges, cursor, n_keys, total);
}

void launch_fill(const float4* ms, const uint32_t* ntiles, const uint2* tilebox,
                 const uint32_t* depth_key, int64_t n, const FrameParams& fp, uint32_t* cursor,
                 unsigned long long* bucket, uint32_t* slot_of, uint32_t* slot_off, int64_t cap,
                 unsigned long long* lookback, uint32_t* counter, cudaStream_t st) {
  const int64_t tiles = fill_scratch_words(n);
  if (tiles == 0) return;
  k_fill<<<(unsigned)tiles, kFillThreads, 0, st>>>(ms, ntiles, tilebox, depth_key, n, fp, cursor,
                                                   bucket, slot_of, slot_off, cap, lookback,
                                                   counter);
}

void launch_tile_sort(const FrameParams& fp, const uint2* ranges, const unsigned long long* bucket,
                      const unsigned long long* total, int64_t cap, uint2* sorted, float4* scratch,
                      cudaStream_t st) {
  const size_t smem = kSortCap * (sizeof(unsigned long long) + sizeof(uint32_t));
  k_tile_sort<<<fp.n_tiles, kTsThreads, smem, st>>>(ranges, bucket, total, cap, sorted, scratch);
}

}  // namespace isg

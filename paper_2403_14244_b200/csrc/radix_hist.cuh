// radix_hist.cuh — digit histograms for the onesweep radix sort (k_sort.cu), built by the
// kernels that produce the keys (k_preprocess: depth keys, k_scan_emit: tile keys) so the sorts
// need no separate histogram pass.  Every 256-thread block accumulates `passes` 256-bin
// histograms in shared memory, adds its non-zero bins to the global ones, and the last block to
// finish turns them into exclusive digit offsets (what k_onesweep reads).
#pragma once
#include <stdint.h>

#include "isg_internal.cuh"

namespace isg {

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Exclusive scan of one u32 per thread over a 256-thread block.  s_warp: >= 8 words.
__device__ __forceinline__ uint32_t block_excl_scan_256(uint32_t v, uint32_t* s_warp,
                                                        uint32_t& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  uint32_t wpre = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t s = s_warp[i];
    wpre += (i < w) ? s : 0u;
    tot += s;
  }
  total = tot;
  __syncthreads();
  return wpre + x - v;
}

__device__ __forceinline__ void hist_zero(uint32_t (*sh)[256]) {
  for (int i = threadIdx.x; i < kMaxPasses * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
}

// Called by all 32 lanes.  A digit shared by the whole warp (the skewed high bytes: the
// exponent byte of positive depths, the top bits of tile ids) costs one shared atomic per warp
// instead of 32 serialised ones.  (Aggregating the two most common digits of a warp instead
// measured slower: the extra ballots cost more than the conflicts they save.)
__device__ __forceinline__ void hist_add_warp(uint32_t (*sh)[256], uint32_t key, bool valid,
                                              int passes) {
  const bool full = __all_sync(0xffffffffu, valid);
  for (int p = 0; p < passes; ++p) {
    const uint32_t d = (key >> (8 * p)) & 255u;
    const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
    if (full && __all_sync(0xffffffffu, d == d0)) {
      if ((threadIdx.x & 31) == 0) atomicAdd(&sh[p][d0], 32u);
    } else if (valid) {
      atomicAdd(&sh[p][d], 1u);
    }
  }
}

// 256-thread block, after its last hist_add_warp: publish and, in the last block to finish,
// scan (done: a zeroed counter; every block of the grid must call this).
__device__ __forceinline__ void hist_publish(uint32_t (*sh)[256], int passes,
                                             uint32_t* __restrict__ hist,
                                             uint32_t* __restrict__ done) {
  __syncthreads();
  for (int p = 0; p < passes; ++p) {
    const uint32_t c = sh[p][threadIdx.x];
    if (c) atomicAdd(&hist[p * 256 + threadIdx.x], c);
  }
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  __shared__ uint32_t s_warp[8];
  for (int p = 0; p < passes; ++p) {
    const uint32_t c = __ldcg(&hist[p * 256 + threadIdx.x]);
    uint32_t tot;
    const uint32_t ex = block_excl_scan_256(c, s_warp, tot);
    hist[p * 256 + threadIdx.x] = ex;
  }
}

}  // namespace isg

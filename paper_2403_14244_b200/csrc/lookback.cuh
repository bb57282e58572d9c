// lookback.cuh — decoupled look-back for single-pass scans (one 64-bit status word per CTA
// tile: 2 flag bits + 62-bit count).  Executed by ONE full warp: the lanes read a window of 32
// predecessors at once, so the exclusive prefix costs ~1 memory round trip per 32 tiles of
// "aggregate only" predecessors instead of one round trip per predecessor.
#pragma once
#include <stdint.h>

namespace isg {

constexpr unsigned long long kLbAgg = 1ull << 62;
constexpr unsigned long long kLbInc = 2ull << 62;
constexpr unsigned long long kLbMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long lb_load(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void lb_store(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Called by all 32 lanes of one warp.  Publishes `agg` for `tile`, walks back, publishes the
// inclusive prefix and returns the exclusive prefix (same value in every lane).
__device__ __forceinline__ unsigned long long lookback_warp(unsigned long long* status,
                                                            uint32_t tile,
                                                            unsigned long long agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) lb_store(status, kLbInc | agg);
    return 0ull;
  }
  if (lane == 0) lb_store(status + tile, kLbAgg | agg);
  unsigned long long excl = 0;
  int64_t hi = (int64_t)tile - 1;  // newest predecessor of the current window
  while (true) {
    const int64_t p = hi - lane;
    unsigned long long s = kLbInc;  // "before tile 0" counts as an inclusive zero
    if (p >= 0) {
      do {
        s = lb_load(status + p);
      } while ((s & ~kLbMask) == 0);
    }
    const unsigned inc = __ballot_sync(0xffffffffu, (s & ~kLbMask) == kLbInc);
    // lanes up to and including the first inclusive one (nearest predecessor) contribute
    const int stop = inc ? __ffs(inc) - 1 : 31;
    unsigned long long v = (lane <= stop) ? (s & kLbMask) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (inc) break;
    hi -= 32;
  }
  if (lane == 0) lb_store(status + tile, kLbInc | (excl + agg));
  return excl;
}

}  // namespace isg

// blend_common.cuh — pieces shared by the tile blend kernels (k_blend.cu, k_blend_bwd.cu).
#pragma once
#include <type_traits>

#include "isg_math.cuh"

namespace isg {
namespace blend {

constexpr float kLn2 = 0.6931471805599453f;
// smallest normal float: a final transmittance below it cannot be divided back up (k_blend.cu)
constexpr float kMinNormal = 1.17549435e-38f;
// start of an empty tile's range as the tile sort leaves it (isg_debug_bins fixes it up)
constexpr uint32_t kEmptyRange = 0xFFFFFFFFu;

__device__ __forceinline__ bool overflowed(const unsigned long long* total, int64_t cap) {
  return *total > (unsigned long long)cap;
}
// total[2] = max key count of any overflowed frame since the host's last check, total[3] =
// frames skipped; the per-frame reset leaves both alone (isg_internal.cuh, kTotal*)
__device__ __forceinline__ void note_overflow(unsigned long long* total) {
  atomicMax(total + kTotalOverflowMax, total[kTotalKeys]);
  atomicAdd(total + kTotalOverflowFrames, 1ull);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// L2 reduction of two consecutive floats (REDG.E.ADD.F32x2): fire-and-forget, no return value
__device__ __forceinline__ void red_add_v2(float* p, float a, float b) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}
// ... predicated in place (no branch around it: the walk loop stays one basic block).  The
// address is only formed, never dereferenced, when `on` is false.
__device__ __forceinline__ void red_add_v2_if(bool on, float* p, float a, float b) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n @q red.global.add.v2.f32 [%0], {%1, %2};\n}" ::"l"(p),
      "f"(a), "f"(b), "r"((unsigned)on)
      : "memory");
}

__device__ __forceinline__ float fast_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fast_sqrt(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// A batch of staged records of one tile list.
template <int B>
struct Stage {
  float4 geo[B];     // u, v, r2max, -log2e / sigma2d^2
  float4 col[B];     // r, g, b, opacity
  uint32_t slot[B];  // gradient slot of the (tile, splat) pair
  uint16_t mask[B];  // the pair's sub-quarter mask (sub_mask16)
};

// Stage list entries [beg, beg+cnt) of the sorted (splat, slot) array (thread t: entries t,
// t + NT, ...).  The 32-B record gathers are issued as cp.async; the caller waits + barriers
// before use.
// kSplat: st.slot holds the splat index instead of the pair's gradient slot.  kMask: also stage
// the entries' sub-quarter masks.
template <int NT, int B, bool kSplat = false, bool kMask = true>
__device__ __forceinline__ void stage_batch(Stage<B>& st, const uint2* __restrict__ sorted,
                                            const uint16_t* __restrict__ submask,
                                            const RenderRec* __restrict__ rec, uint32_t beg,
                                            int cnt) {
#pragma unroll
  for (int t = threadIdx.x; t < B; t += NT) {
    if (t < cnt) {
      const uint2 gs = sorted[beg + t];  // (splat, gradient slot)
      st.slot[t] = kSplat ? gs.x : gs.y;
      if (kMask) st.mask[t] = submask[beg + t];
      cp_async16(&st.geo[t], &rec[gs.x].geo);
      cp_async16(&st.col[t], &rec[gs.x].col);
    }
  }
  cp_async_commit();
}

}  // namespace blend
}  // namespace isg

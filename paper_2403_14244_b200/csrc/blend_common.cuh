// blend_common.cuh — pieces shared by the tile blend kernels (k_blend.cu, k_blend_bwd.cu).
#pragma once
#include "isg_math.cuh"

namespace isg {
namespace blend {

constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ bool overflowed(const unsigned long long* total, int64_t cap) {
  return *total > (unsigned long long)cap;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

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
};

// Stage list entries [beg, beg+cnt) of the sorted (splat, slot) array (thread t: entry t).
// The 32-B record gather is issued as cp.async; the caller waits + barriers before use.
template <int B>
__device__ __forceinline__ void stage_batch(Stage<B>& st, const uint2* __restrict__ sorted,
                                            const RenderRec* __restrict__ rec, uint32_t beg,
                                            int cnt) {
  const int t = threadIdx.x;
  if (t < cnt) {
    const uint2 gs = sorted[beg + t];  // (splat, gradient slot)
    st.slot[t] = gs.y;
    cp_async16(&st.geo[t], &rec[gs.x].geo);
    cp_async16(&st.col[t], &rec[gs.x].col);
  }
  cp_async_commit();
}

// Pixel-centre rectangle of an 8x8 region, clipped to the image.
struct Region {
  float x0, x1, y0, y1;
  bool valid;
};

__device__ __forceinline__ Region region_rect(const FrameParams& fp, int tile, int r) {
  Region g;
  const int tx = tile % fp.tiles_x, ty = tile / fp.tiles_x;
  const int W = fp.cam.width, H = fp.cam.height;
  const int x0 = tx * kTile + (r & 1) * 8, y0 = ty * kTile + (r >> 1) * 8;
  g.valid = x0 < W && y0 < H;
  g.x0 = (float)x0 + 0.5f;
  g.x1 = (float)(min(x0 + 8, W) - 1) + 0.5f;
  g.y0 = (float)y0 + 0.5f;
  g.y1 = (float)(min(y0 + 8, H) - 1) + 0.5f;
  return g;
}

// 3-sigma circle vs pixel-centre rectangle (conservative, exact rounding like tile_hit).
__device__ __forceinline__ bool rect_hit(const Region& g, float u, float v, float r2max) {
  const float cx = fminf(fmaxf(u, g.x0), g.x1);
  const float cy = fminf(fmaxf(v, g.y0), g.y1);
  return !(dist2_rn(__fsub_rn(cx, u), __fsub_rn(cy, v)) > r2max);
}

}  // namespace blend
}  // namespace isg

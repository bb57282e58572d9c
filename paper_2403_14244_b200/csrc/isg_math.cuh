// isg_math.cuh — device arithmetic shared by the kernels.  Every operation whose result
// decides WHICH (tile, splat) or (pixel, splat) pairs exist is written with explicit
// round-to-nearest intrinsics (no FMA contraction), in exactly the order of the FP32 oracle
// (oracle/isg_oracle.c: or32_project, or32_tile_hit, or32_tile_bbox, or32_blend_pixel), so
// tile keys, sort order, ranges and 3-sigma inclusion are bit-identical to it.
#pragma once
#include "isg_internal.cuh"
#include "pdl.cuh"

namespace isg {

struct Proj {
  float xc, yc, zc;
  float u, v, s, r2max;
  bool vis;
};

// project_iso (splat3d.cpp:59-64) in FP32.
__device__ __forceinline__ Proj project(const float4 ms, const isg_camera& c) {
  Proj p;
  float xc = __fmul_rn(c.R[0], ms.x);
  xc = __fadd_rn(xc, __fmul_rn(c.R[1], ms.y));
  xc = __fadd_rn(xc, __fmul_rn(c.R[2], ms.z));
  xc = __fadd_rn(xc, c.t[0]);
  float yc = __fmul_rn(c.R[3], ms.x);
  yc = __fadd_rn(yc, __fmul_rn(c.R[4], ms.y));
  yc = __fadd_rn(yc, __fmul_rn(c.R[5], ms.z));
  yc = __fadd_rn(yc, c.t[1]);
  float zc = __fmul_rn(c.R[6], ms.x);
  zc = __fadd_rn(zc, __fmul_rn(c.R[7], ms.y));
  zc = __fadd_rn(zc, __fmul_rn(c.R[8], ms.z));
  zc = __fadd_rn(zc, c.t[2]);
  p.xc = xc;
  p.yc = yc;
  p.zc = zc;
  p.vis = zc > kNearPlane;
  p.u = __fadd_rn(__fdiv_rn(__fmul_rn(c.focal, xc), zc), c.cx);
  p.v = __fadd_rn(__fdiv_rn(__fmul_rn(c.focal, yc), zc), c.cy);
  p.s = __fdiv_rn(__fmul_rn(ms.w, c.focal), zc);
  p.r2max = __fmul_rn(__fmul_rn(9.0f, p.s), p.s);
  return p;
}

// squared distance with the oracle's rounding: (dx*dx) + (dy*dy), each rounded.
__device__ __forceinline__ float dist2_rn(float dx, float dy) {
  return __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
}

// One axis of tile_hit: the rounded squared distance from c (u or v) to the pixel-centre span of
// tile t along an axis of lim pixels.  tile_hit == !(axis_d2(u, tx, W) + axis_d2(v, ty, H) >
// r2max) with the sum rounded once, bit for bit, so a row's term can be hoisted.
__device__ __forceinline__ float axis_d2(float c, int t, int lim) {
  const float lo = (float)(t * kTile) + 0.5f;
  const float hi = (float)(min(t * kTile + kTile, lim) - 1) + 0.5f;
  const float q = c < lo ? lo : (c > hi ? hi : c);
  const float d = __fsub_rn(q, c);
  return __fmul_rn(d, d);
}

// Exact tile test (or32_tile_hit).
__device__ __forceinline__ bool tile_hit(float u, float v, float r2max, int tx, int ty, int W,
                                         int H) {
  const int xe = min(tx * kTile + kTile, W) - 1;
  const int ye = min(ty * kTile + kTile, H) - 1;
  const float x0 = (float)(tx * kTile) + 0.5f, x1 = (float)xe + 0.5f;
  const float y0 = (float)(ty * kTile) + 0.5f, y1 = (float)ye + 0.5f;
  const float qx = u < x0 ? x0 : (u > x1 ? x1 : u);
  const float qy = v < y0 ? y0 : (v > y1 ? y1 : v);
  const float d2 = dist2_rn(__fsub_rn(qx, u), __fsub_rn(qy, v));
  return !(d2 > r2max);
}

// Conservative tile bounding box (or32_tile_bbox).
__device__ __forceinline__ bool tile_bbox(float u, float v, float s, int tiles_x, int tiles_y,
                                          int& x0, int& x1, int& y0, int& y1) {
  const float ext = __fadd_rn(__fmul_rn(__fmul_rn(3.0f, s), 1.0009765625f), 1.0f);
  const float inv = 1.0f / kTile;
  float fx0 = floorf(__fmul_rn(__fsub_rn(u, ext), inv));
  float fx1 = floorf(__fmul_rn(__fadd_rn(u, ext), inv));
  float fy0 = floorf(__fmul_rn(__fsub_rn(v, ext), inv));
  float fy1 = floorf(__fmul_rn(__fadd_rn(v, ext), inv));
  fx0 = fmaxf(fx0, 0.0f);
  fy0 = fmaxf(fy0, 0.0f);
  fx1 = fminf(fx1, (float)(tiles_x - 1));
  fy1 = fminf(fy1, (float)(tiles_y - 1));
  if (!(fx0 <= fx1) || !(fy0 <= fy1)) return false;
  x0 = (int)fx0;
  x1 = (int)fx1;
  y0 = (int)fy0;
  y1 = (int)fy1;
  return true;
}

// Tiles a splat touches, from K1's compact box record (small box: popc of the hit mask; bigger
// box, bw == 0: the count itself in .y).
__device__ __forceinline__ uint32_t tilebox_count(uint2 box) {
  return (box.x >> 24) ? (uint32_t)__popc(box.y) : box.y;
}

// Visit the tiles a splat touches, in row-major order (the order K1 counted them).  `box` is
// K1's compact record: x0 | y0 << 12 | bw << 24 and a hit mask over the (<= 32-tile) bbox; for
// bigger boxes (bw == 0) the projection and the exact tile tests are recomputed from `ms`.
template <class F>
__device__ __forceinline__ void for_each_tile(uint2 box, const float4& ms, const FrameParams& fp,
                                              F&& f) {
  const uint32_t bw = box.x >> 24;
  if (bw) {
    const uint32_t x0 = box.x & 0xFFFu, y0 = (box.x >> 12) & 0xFFFu;
    const uint32_t inv = (65536u + bw - 1u) / bw;  // exact floor(b / bw) for b < 32
    uint32_t m = box.y;
    while (m) {
      const uint32_t b = __ffs(m) - 1;
      m &= m - 1;
      const uint32_t r = (b * inv) >> 16;
      f((int)((y0 + r) * (uint32_t)fp.tiles_x + x0 + (b - r * bw)));
    }
    return;
  }
  const Proj p = project(ms, fp.cam);
  int x0, x1, y0, y1;
  if (!p.vis || !tile_bbox(p.u, p.v, p.s, fp.tiles_x, fp.tiles_y, x0, x1, y0, y1)) return;
  for (int ty = y0; ty <= y1; ++ty)
    for (int tx = x0; tx <= x1; ++tx)
      if (tile_hit(p.u, p.v, p.r2max, tx, ty, fp.cam.width, fp.cam.height))
        f(ty * fp.tiles_x + tx);
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

}  // namespace isg

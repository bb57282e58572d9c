// K6/K7 — per-16x16-tile alpha blending, forward and backward.
//
// K6 replaces composite_pixels (/root/reference/proj/src/splat3d.cpp:125-162) and the
// inclusion test covers(ScreenIso) (:108-114): instead of every pixel visiting every splat
// (O(W*H*N)), a CTA owns one tile and walks only that tile's depth-ordered list, staged in
// batches of 256 records into shared memory; each thread is one pixel, and the CTA stops as
// soon as every pixel's transmittance is <= t_min (__syncthreads_count).  The 3-sigma test is
// bit-identical to the FP32 oracle (explicit _rn arithmetic); exp uses ex2.approx.
//
// K7 is the backward the reference does not have: the same tile walk in
// reverse from each pixel's last processed entry, with the L2 loss gradient
// dL/dC = 2 w (C - target) / (3 W H) (mse, src/image.cpp:50-58) fused in the prologue, the
// transmittance recovered by division, and per-splat 2D gradients (du, dv, dsigma2d,
// dopacity, drgb) pre-reduced across the warp with shuffles before one vector atomic per warp.
#include "isg_math.cuh"

namespace isg {

namespace {
constexpr int kBlendThreads = kTilePixels;  // one pixel per thread
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ bool overflowed(const unsigned long long* total, int64_t cap) {
  return *total > (unsigned long long)cap;
}
}  // namespace

__global__ void __launch_bounds__(kBlendThreads) k_blend_fwd(
    FrameParams fp, const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
    const RenderRec* __restrict__ rec, const unsigned long long* __restrict__ total,
    int64_t key_cap, float* __restrict__ out, float* __restrict__ t_last,
    uint32_t* __restrict__ n_proc) {
  __shared__ float4 s_geo[kBlendThreads];
  __shared__ float4 s_col[kBlendThreads];
  if (overflowed(total, key_cap)) return;
  const int tile = blockIdx.x;
  const int tx = tile % fp.tiles_x, ty = tile / fp.tiles_x;
  const int x = tx * kTile + (threadIdx.x & (kTile - 1));
  const int y = ty * kTile + (threadIdx.x / kTile);
  const int W = fp.cam.width, H = fp.cam.height;
  const bool inside = x < W && y < H;
  const float px = (float)x + 0.5f, py = (float)y + 0.5f;
  const uint2 rg = ranges[tile];
  float T = 1.0f, Tl = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f;
  uint32_t np = 0;
  bool done = !inside;
  for (uint32_t b = rg.x; b < rg.y; b += kBlendThreads) {
    if (__syncthreads_count(done) == kBlendThreads) break;
    const uint32_t idx = b + threadIdx.x;
    if (idx < rg.y) {
      const RenderRec r = rec[vals[idx]];
      s_geo[threadIdx.x] = make_float4(r.geo.x, r.geo.y, -kLog2e / r.geo.z, r.geo.w);
      s_col[threadIdx.x] = r.col;
    }
    __syncthreads();
    if (!done) {
      const int cnt = (int)min((uint32_t)kBlendThreads, rg.y - b);
      for (int j = 0; j < cnt; ++j) {
        const float4 g = s_geo[j];
        const float r2 = dist2_rn(__fsub_rn(px, g.x), __fsub_rn(py, g.y));
        if (r2 > g.w) continue;
        const float e = fast_exp2(r2 * g.z);
        const float4 c = s_col[j];
        const float a = c.w * e;
        const float wgt = T * a;
        C0 += wgt * c.x;
        C1 += wgt * c.y;
        C2 += wgt * c.z;
        Tl = T;
        T = T * (1.0f - a);
        np = b - rg.x + (uint32_t)j + 1u;
        if (!(T > fp.t_min)) {
          done = true;
          break;
        }
      }
    }
  }
  if (inside) {
    const size_t pix = (size_t)y * W + x;
    out[3 * pix + 0] = C0 + T * fp.bg[0];
    out[3 * pix + 1] = C1 + T * fp.bg[1];
    out[3 * pix + 2] = C2 + T * fp.bg[2];
    t_last[pix] = Tl;
    n_proc[pix] = np;
  }
}

__global__ void __launch_bounds__(kBlendThreads) k_blend_bwd(
    FrameParams fp, const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
    const RenderRec* __restrict__ rec, const unsigned long long* __restrict__ total,
    int64_t key_cap, const float* __restrict__ img, const float* __restrict__ target,
    const float* __restrict__ t_last, const uint32_t* __restrict__ n_proc, float loss_scale,
    float4* __restrict__ grad2d, double* __restrict__ tile_loss) {
  __shared__ float4 s_geo[kBlendThreads];  // u, v, r2max, -log2e/s^2
  __shared__ float4 s_col[kBlendThreads];  // r, g, b, opacity
  __shared__ float2 s_aux[kBlendThreads];  // 2/s^2, 1/s
  __shared__ uint32_t s_rank[kBlendThreads];
  __shared__ float s_red[kBlendThreads / 32];
  __shared__ uint32_t s_max[kBlendThreads / 32];
  const int tile = blockIdx.x;
  if (overflowed(total, key_cap)) {
    if (threadIdx.x == 0) tile_loss[tile] = 0.0;
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tx = tile % fp.tiles_x, ty = tile / fp.tiles_x;
  const int x = tx * kTile + (threadIdx.x & (kTile - 1));
  const int y = ty * kTile + (threadIdx.x / kTile);
  const int W = fp.cam.width, H = fp.cam.height;
  const bool inside = x < W && y < H;
  const float px = (float)x + 0.5f, py = (float)y + 0.5f;
  const uint2 rg = ranges[tile];
  float G0 = 0.f, G1 = 0.f, G2 = 0.f, Tc = 0.f, dsq = 0.f;
  uint32_t np = 0;
  if (inside) {
    const size_t pix = (size_t)y * W + x;
    const float d0 = img[3 * pix + 0] - target[3 * pix + 0];
    const float d1 = img[3 * pix + 1] - target[3 * pix + 1];
    const float d2 = img[3 * pix + 2] - target[3 * pix + 2];
    dsq = d0 * d0 + d1 * d1 + d2 * d2;
    G0 = 2.0f * d0 * loss_scale;
    G1 = 2.0f * d1 * loss_scale;
    G2 = 2.0f * d2 * loss_scale;
    Tc = t_last[pix];
    np = n_proc[pix];
  }
  // tile loss partial and the tile's longest walk
  float wsum = dsq;
  uint32_t wmax = np;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
    wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
  }
  if (lane == 0) {
    s_red[warp] = wsum;
    s_max[warp] = wmax;
  }
  __syncthreads();
  uint32_t maxnp = 0;
  if (threadIdx.x == 0) {
    float tsum = 0.f;
    for (int i = 0; i < kBlendThreads / 32; ++i) tsum += s_red[i];
    tile_loss[tile] = (double)tsum;
  }
#pragma unroll
  for (int i = 0; i < kBlendThreads / 32; ++i) maxnp = max(maxnp, s_max[i]);

  float A0 = fp.bg[0], A1 = fp.bg[1], A2 = fp.bg[2];
  bool first = true;
  for (int hi = (int)maxnp; hi > 0; hi -= kBlendThreads) {
    const int lo = max(0, hi - kBlendThreads);
    __syncthreads();
    const int jl = (int)threadIdx.x;
    if (lo + jl < hi) {
      const uint32_t r = vals[rg.x + lo + jl];
      const RenderRec rr = rec[r];
      const float s2 = rr.geo.z;
      s_geo[jl] = make_float4(rr.geo.x, rr.geo.y, rr.geo.w, -kLog2e / s2);
      s_col[jl] = rr.col;
      s_aux[jl] = make_float2(2.0f / s2, rsqrtf(s2));
      s_rank[jl] = r;
    }
    __syncthreads();
    for (int j = hi - 1; j >= lo; --j) {
      const float4 g = s_geo[j - lo];
      float gu = 0.f, gv = 0.f, gs = 0.f, go = 0.f, gr = 0.f, gg = 0.f, gb = 0.f;
      bool contrib = false;
      if ((uint32_t)j < np) {
        const float dx = __fsub_rn(px, g.x), dy = __fsub_rn(py, g.y);
        const float r2 = dist2_rn(dx, dy);
        if (!(r2 > g.z)) {
          contrib = true;
          const float e = fast_exp2(r2 * g.w);
          const float4 c = s_col[j - lo];
          const float2 aux = s_aux[j - lo];
          const float a = c.w * e;
          const float T = first ? Tc : __fdividef(Tc, 1.0f - a);
          first = false;
          Tc = T;
          const float dLda = T * (G0 * (c.x - A0) + G1 * (c.y - A1) + G2 * (c.z - A2));
          const float Ta = T * a;
          gr = G0 * Ta;
          gg = G1 * Ta;
          gb = G2 * Ta;
          A0 = a * c.x + (1.0f - a) * A0;
          A1 = a * c.y + (1.0f - a) * A1;
          A2 = a * c.z + (1.0f - a) * A2;
          go = dLda * e;
          const float k2 = dLda * c.w * e * aux.x;
          gu = k2 * dx;
          gv = k2 * dy;
          gs = k2 * r2 * aux.y;
        }
      }
      if (__any_sync(0xffffffffu, contrib)) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          gu += __shfl_down_sync(0xffffffffu, gu, o);
          gv += __shfl_down_sync(0xffffffffu, gv, o);
          gs += __shfl_down_sync(0xffffffffu, gs, o);
          go += __shfl_down_sync(0xffffffffu, go, o);
          gr += __shfl_down_sync(0xffffffffu, gr, o);
          gg += __shfl_down_sync(0xffffffffu, gg, o);
          gb += __shfl_down_sync(0xffffffffu, gb, o);
        }
        if (lane == 0) {
          const uint32_t r = s_rank[j - lo];
          atomicAdd(&grad2d[2 * (size_t)r + 0], make_float4(gu, gv, gs, go));
          atomicAdd(&grad2d[2 * (size_t)r + 1], make_float4(gr, gg, gb, 0.f));
        }
      }
    }
  }
}

__global__ void k_loss_reduce(const double* __restrict__ tile_loss, int n_tiles, double scale,
                              double* __restrict__ loss) {
  __shared__ double s[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n_tiles; i += 256) acc += tile_loss[i];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    loss[0] += s[0] * scale;  // accumulated over views
    loss[1] = s[0] * scale;   // this view
  }
}

void launch_blend_fwd(const FrameParams& fp, const uint2* ranges, const uint32_t* vals,
                      const RenderRec* rec, const unsigned long long* total, int64_t key_cap,
                      float* out, float* t_last, uint32_t* n_proc, cudaStream_t st) {
  k_blend_fwd<<<fp.n_tiles, kBlendThreads, 0, st>>>(fp, ranges, vals, rec, total, key_cap, out,
                                                    t_last, n_proc);
}

void launch_blend_bwd(const FrameParams& fp, const uint2* ranges, const uint32_t* vals,
                      const RenderRec* rec, const unsigned long long* total, int64_t key_cap,
                      const float* img, const float* target, const float* t_last,
                      const uint32_t* n_proc, float loss_scale, float4* grad2d,
                      double* tile_loss, cudaStream_t st) {
  k_blend_bwd<<<fp.n_tiles, kBlendThreads, 0, st>>>(fp, ranges, vals, rec, total, key_cap, img,
                                                    target, t_last, n_proc, loss_scale, grad2d,
                                                    tile_loss);
}

void launch_loss_reduce(const double* tile_loss, int n_tiles, double scale, double* loss,
                        cudaStream_t st) {
  k_loss_reduce<<<1, 256, 0, st>>>(tile_loss, n_tiles, scale, loss);
}

}  // namespace isg

// K1 — per-splat preprocess.  Replaces the projection loop of render(iso)
// (/root/reference/proj/src/splat3d.cpp:176-188 -> project_iso :59-64) and the per-splat
// validation (IsoSplat3D::validate, splat3d.cpp:10-17).
//
// One thread per splat (grid-stride over one resident wave of blocks, the next splat
// prefetched), coalesced float4 SoA loads (32 B/splat read), writes the 32-B render record,
// the tile count (4 B) and, in radix binning mode, the depth key (4 B) plus the depth sort's
// digit histograms (radix_hist.cuh: one global publish per block, so the sort needs no
// histogram pass); in tile-bucket mode it instead bumps one per-tile counter per touched tile.  Isotropic shortcut: the screen
// radius is 3*sigma*f/z directly — no 3x3 covariance, no eigen-solve.  Splats that are culled
// (z <= near) or touch no tile get count 0 (and depth key 0xFFFFFFFF: they sort last and emit
// nothing).
#include <algorithm>

#include "isg_math.cuh"
#include "radix_hist.cuh"

namespace isg {

// 5 CTAs / SM (47 registers, no spills): C3 0.0389 vs 0.0391 ms, C5 0.391 vs 0.398 ms against
// ptxas's own 58; 6 / 8 spill and are slower
#ifndef ISG_K1_MINB
#define ISG_K1_MINB 5
#endif
#if ISG_K1_MINB > 0
#define ISG_K1_BOUNDS __launch_bounds__(256, ISG_K1_MINB)
#else
#define ISG_K1_BOUNDS __launch_bounds__(256)
#endif
template <bool kBucket>  // tile-bucket binning: also bump the per-tile counters
__global__ void ISG_K1_BOUNDS k_preprocess(const float4* __restrict__ ms,
                                                    const float4* __restrict__ co, int64_t n,
                                                    FrameParams fp, RenderRec* __restrict__ rec,
                                                    uint32_t* __restrict__ depth_key,
                                                    uint32_t* __restrict__ ntiles,
                                                    uint2* __restrict__ tilebox,
                                                    uint32_t* __restrict__ tile_cnt,
                                                    uint32_t* __restrict__ sc,
                                                    uint32_t* __restrict__ hist,
                                                    uint32_t* __restrict__ hist_done) {
  pdl_enter();
  // radix mode: the depth sort's 4 digit histograms (radix_hist.cuh)
  __shared__ uint32_t sh[kMaxPasses][256];
  if (hist) {
    hist_zero(sh);
    __syncthreads();
  }
  // sc: [1] 0xFFFFFFFF - first invalid splat (atomicMax, 0 = none: zero-initialised with the
  // other scalars), [2] visible splats, [4] n (device count)
  if (blockIdx.x == 0 && threadIdx.x == 0) sc[4] = (uint32_t)n;
  // grid-stride over block-sized chunks (one resident wave of blocks: each publishes its
  // histograms once); the next chunk's splat is loaded while this one is processed
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float4 a_nx = make_float4(0.f, 0.f, 0.f, 0.f), c_nx = a_nx;
  {
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i0 < n) {
      a_nx = ms[i0];
      c_nx = co[i0];
    }
  }
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t i = base + threadIdx.x;
    const float4 a = a_nx, c = c_nx;
    if (i + stride < n) {
      a_nx = ms[i + stride];
      c_nx = co[i + stride];
    }
    uint32_t count = 0;
    uint32_t key = 0xFFFFFFFFu;
    if (i < n) {
      uint2 box = make_uint2(0u, 0u);
      // IsoSplat3D::validate (splat3d.cpp:10-17): finite mu, sigma > 0 finite, finite color,
      // opacity in [0,1].  The host reports the first offending index with the reference message.
      const bool ok = isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && a.w > 0.0f &&
                      isfinite(a.w) && isfinite(c.x) && isfinite(c.y) && isfinite(c.z) &&
                      c.w >= 0.0f && c.w <= 1.0f;
      if (!ok) atomicMax(&sc[1], 0xFFFFFFFFu - (uint32_t)i);
      const Proj p = project(a, fp.cam);
      if (p.vis && ok) {
        int x0, x1, y0, y1;
        if (tile_bbox(p.u, p.v, p.s, fp.tiles_x, fp.tiles_y, x0, x1, y0, y1)) {
          const int bw = x1 - x0 + 1;
          const bool small = bw * (y1 - y0 + 1) <= 32 && bw < 256 && x0 < 4096 && y0 < 4096;
          uint32_t mask = 0;
          // tile_hit, separably (bit-identical decisions): the row's y term once per row and,
          // for boxes up to kCols tiles wide (all but the largest splats), every column's x
          // term once per splat instead of once per tile.  Columns past the box get an x term
          // of +inf (never hit), so a row's hits are one branch-free 8-bit mask.
          uint32_t bit = 1u;
          constexpr int kCols = 8;
          if (bw <= kCols) {
            float ax[kCols];
#pragma unroll
            for (int c = 0; c < kCols; ++c)
              ax[c] = c < bw ? axis_d2(p.u, x0 + c, fp.cam.width) : __int_as_float(0x7f800000);
            int sh = 0;
            for (int ty = y0; ty <= y1; ++ty, sh += bw) {
              const float ay = axis_d2(p.v, ty, fp.cam.height);
              uint32_t row = 0;
#pragma unroll
              for (int c = 0; c < kCols; ++c)
                row |= (__fadd_rn(ax[c], ay) > p.r2max ? 0u : 1u) << c;
              count += __popc(row);
              if (sh < 32) mask |= row << sh;  // (only meaningful when small: <= 32 tiles)
              if constexpr (kBucket) {
                for (uint32_t m = row; m; m &= m - 1)
                  atomicAdd(&tile_cnt[ty * fp.tiles_x + x0 + __ffs(m) - 1], 1u);
              }
            }
          } else {
            for (int ty = y0; ty <= y1; ++ty) {
              const float ay = axis_d2(p.v, ty, fp.cam.height);
              for (int tx = x0; tx <= x1; ++tx, bit <<= 1) {
                if (__fadd_rn(axis_d2(p.u, tx, fp.cam.width), ay) > p.r2max) continue;
                mask |= bit;
                ++count;
                if constexpr (kBucket) atomicAdd(&tile_cnt[ty * fp.tiles_x + tx], 1u);
              }
            }
          }
          // emission kernels iterate the hit bits instead of re-projecting; a bigger box
          // (bw == 0: re-project) carries the tile count instead, so one 8-B gather gives the
          // emission every splat's count (popc of the mask, or box.y)
          box = small ? make_uint2((uint32_t)x0 | ((uint32_t)y0 << 12) | ((uint32_t)bw << 24), mask)
                      : make_uint2(0u, count);
        }
      }
      tilebox[i] = box;
      RenderRec r;  // (u, v, r2max, -log2(e)/sigma2d^2), (r, g, b, log2 opacity)
      // -log2(e) / sigma2d^2 feeds only ex2.approx (no inclusion decision): a MUFU reciprocal
      float inv_s2;
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv_s2) : "f"(__fmul_rn(p.s, p.s)));
      r.geo = make_float4(p.u, p.v, p.r2max, -1.4426950408889634f * inv_s2);
      r.col = c;
      // log2(opacity): the blend kernels form alpha as one ex2(r2 g + log2 o).  Opacity is
      // floored at kOpacityFloor (2^-60) so that alpha / o stays defined for the backward: an
      // opacity-0 splat keeps its opacity gradient, and its alpha (<= 2^-60) leaves every
      // 1 - alpha at exactly 1
      asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r.col.w) : "f"(fmaxf(c.w, kOpacityFloor)));
      rec[i] = r;
      key = count ? __float_as_uint(p.zc) : 0xFFFFFFFFu;
      depth_key[i] = key;
      ntiles[i] = count;
    }
    // visible-splat count, one atomic per warp
    const unsigned vis = __ballot_sync(0xffffffffu, count > 0);
    if ((threadIdx.x & 31) == 0 && vis) atomicAdd(&sc[2], (uint32_t)__popc(vis));
    if (hist) hist_add_warp(sh, key, i < n, kMaxPasses);
  }
  if (hist) hist_publish(sh, kMaxPasses, hist, hist_done);
}

void launch_preprocess(const float4* ms, const float4* co, int64_t n, const FrameParams& fp,
                       RenderRec* rec, uint32_t* depth_key, uint32_t* ntiles, uint2* tilebox,
                       uint32_t* tile_cnt, uint32_t* sc, uint32_t* hist, uint32_t* hist_done,
                       cudaStream_t st) {
  // one resident wave (every block publishes its histograms once), the next splat prefetched:
  // 0.038 vs 0.042 ms at C3 (8 blocks per SM, no prefetch)
  static const int wave = [] {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_preprocess<false>, 256, 0);
    return sms * std::max(per_sm, 1);
  }();
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, wave));
  launch_pdl(tile_cnt ? k_preprocess<true> : k_preprocess<false>, dim3((unsigned)blocks),
             dim3(256), 0, st, ms, co, n, fp, rec,
             depth_key, ntiles, tilebox, tile_cnt, sc, hist, hist_done);
}

// Frame scratch reset (the two regions a frame needs zeroed), as a kernel so that it joins the
// programmatic-dependent-launch chain instead of breaking it like a memset node would.
__global__ void __launch_bounds__(256) k_zero2(unsigned char* __restrict__ a, size_t a_bytes,
                                               unsigned char* __restrict__ b, size_t b_bytes) {
  pdl_enter();
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t a16 = ((uintptr_t)a & 15) ? 0 : a_bytes / 16;
  for (size_t i = tid; i < a16; i += stride)
    reinterpret_cast<uint4*>(a)[i] = make_uint4(0u, 0u, 0u, 0u);
  for (size_t i = 16 * a16 + tid; i < a_bytes; i += stride) a[i] = 0;
  for (size_t i = tid; i < b_bytes; i += stride) b[i] = 0;
}

void launch_zero2(void* a, size_t a_bytes, void* b, size_t b_bytes, cudaStream_t st) {
  const size_t blocks = std::min<size_t>(std::max<size_t>((a_bytes / 16 + 255) / 256, 1), 148 * 4);
  launch_pdl(k_zero2, dim3((unsigned)blocks), dim3(256), 0, st, (unsigned char*)a, a_bytes,
             (unsigned char*)b, b_bytes);
}

// Parity hook: (tile << 32 | float_bits(depth)) and splat index for each sorted entry.
__global__ void k_debug_keys(const uint2* __restrict__ ranges, const uint2* __restrict__ sorted,
                             const float4* __restrict__ ms, FrameParams fp,
                             uint64_t* __restrict__ keys, uint32_t* __restrict__ gids) {
  const uint2 rg = ranges[blockIdx.x];
  for (uint32_t i = rg.x + threadIdx.x; i < rg.y; i += blockDim.x) {
    const uint32_t g = sorted[i].x;
    const Proj p = project(ms[g], fp.cam);
    keys[i] = ((uint64_t)blockIdx.x << 32) | __float_as_uint(p.zc);
    gids[i] = g;
  }
}

void launch_debug_keys(const uint2* ranges, const uint2* sorted, const float4* ms,
                       const FrameParams& fp, uint64_t* keys, uint32_t* gids, cudaStream_t st) {
  k_debug_keys<<<fp.n_tiles, 128, 0, st>>>(ranges, sorted, ms, fp, keys, gids);
}

}  // namespace isg

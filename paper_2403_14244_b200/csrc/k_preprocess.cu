// K1 — per-splat preprocess.  Replaces the projection loop of render(iso)
// (/root/reference/proj/src/splat3d.cpp:176-188 -> project_iso :59-64) and the per-splat
// validation (IsoSplat3D::validate, splat3d.cpp:10-17).
//
// One thread per splat, coalesced float4 SoA loads (32 B/splat read), writes
// rec_geo (16 B), depth key (4 B) and tile count (4 B).  Isotropic shortcut: the screen
// radius is 3*sigma*f/z directly — no 3x3 covariance, no eigen-solve.  Splats that are
// culled (z <= near) or touch no tile get the depth key 0xFFFFFFFF and count 0, so they sort
// last and emit nothing.
#include "isg_math.cuh"

namespace isg {

__global__ void __launch_bounds__(256) k_preprocess(const float4* __restrict__ ms,
                                                    const float4* __restrict__ co, int64_t n,
                                                    FrameParams fp, float4* __restrict__ rec_geo,
                                                    uint32_t* __restrict__ depth_key,
                                                    uint32_t* __restrict__ ntiles,
                                                    uint32_t* __restrict__ first_bad,
                                                    uint32_t* __restrict__ n_dev) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) *n_dev = (uint32_t)n;
  if (i >= n) return;
  const float4 a = ms[i];
  const float4 c = co[i];
  // IsoSplat3D::validate (splat3d.cpp:10-17): finite mu, sigma > 0 finite, finite color,
  // opacity in [0,1].  The host reports the first offending index with the reference message.
  const bool ok = isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && a.w > 0.0f &&
                  isfinite(a.w) && isfinite(c.x) && isfinite(c.y) && isfinite(c.z) &&
                  c.w >= 0.0f && c.w <= 1.0f;
  if (!ok) atomicMin(first_bad, (uint32_t)i);

  const Proj p = project(a, fp.cam);
  uint32_t count = 0;
  if (p.vis && ok) {
    int x0, x1, y0, y1;
    if (tile_bbox(p.u, p.v, p.s, fp.tiles_x, fp.tiles_y, x0, x1, y0, y1)) {
      for (int ty = y0; ty <= y1; ++ty)
        for (int tx = x0; tx <= x1; ++tx)
          count += tile_hit(p.u, p.v, p.r2max, tx, ty, fp.cam.width, fp.cam.height) ? 1u : 0u;
    }
  }
  rec_geo[i] = make_float4(p.u, p.v, p.s, p.r2max);
  depth_key[i] = count ? __float_as_uint(p.zc) : 0xFFFFFFFFu;
  ntiles[i] = count;
}

void launch_preprocess(const float4* ms, const float4* co, int64_t n, const FrameParams& fp,
                       float4* rec_geo, uint32_t* depth_key, uint32_t* ntiles,
                       uint32_t* first_bad, uint32_t* n_dev, cudaStream_t st) {
  const int64_t blocks = n > 0 ? (n + 255) / 256 : 1;
  k_preprocess<<<(unsigned)blocks, 256, 0, st>>>(ms, co, n, fp, rec_geo, depth_key, ntiles,
                                                 first_bad, n_dev);
}

// Parity hook: (tile << 32 | float_bits(depth)) and splat index for each sorted key.
__global__ void k_debug_keys(const uint32_t* __restrict__ tiles,
                             const uint32_t* __restrict__ slots,
                             const uint32_t* __restrict__ emit_rank,
                             const uint32_t* __restrict__ order, const float4* __restrict__ ms,
                             FrameParams fp, int64_t nkeys, uint64_t* __restrict__ keys,
                             uint32_t* __restrict__ gids) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nkeys) return;
  const uint32_t g = order[emit_rank[slots[i]]];
  const Proj p = project(ms[g], fp.cam);
  keys[i] = ((uint64_t)tiles[i] << 32) | __float_as_uint(p.zc);
  gids[i] = g;
}

void launch_debug_keys(const uint32_t* tiles, const uint32_t* slots, const uint32_t* emit_rank,
                       const uint32_t* order, const float4* ms, const FrameParams& fp,
                       int64_t nkeys, uint64_t* keys, uint32_t* gids, cudaStream_t st) {
  if (nkeys <= 0) return;
  k_debug_keys<<<(unsigned)((nkeys + 255) / 256), 256, 0, st>>>(tiles, slots, emit_rank, order,
                                                                 ms, fp, nkeys, keys, gids);
}

}  // namespace isg

// K6/K7 — per-16x16-tile alpha blending, forward and backward.
//
// K6 replaces composite_pixels (/root/reference/proj/src/splat3d.cpp:125-162) and the
// inclusion test covers(ScreenIso) (:108-114).  Instead of every pixel visiting every splat
// (O(W*H*N)), one CTA owns one tile and walks only that tile's depth-ordered list.
//
// Mapping (both kernels): 64 threads per tile; warp w covers the 16x8 half-tile w, each lane a
// 2x2 pixel quad, so one shared-memory record feeds four pixels and the squared distances
// share two dx^2 and two dy^2.  Per list entry the warp first tests the splat's 3-sigma circle
// against its half-tile rectangle (warp-uniform; skips ~half the entries at no divergence).
// Records are staged 64 at a time into shared memory with cp.async, double-buffered: the
// next batch's copy is in flight while the current one is blended.  The forward stops once
// every pixel of the tile has transmittance <= t_min (__syncthreads_count per batch).
//
// The 3-sigma test is bit-identical to the FP32 oracle (explicit _rn arithmetic); exp uses
// ex2.approx on a per-splat precomputed -log2(e)/sigma2d^2.
//
// K7 is the backward the reference does not have: the same walk in reverse from
// each pixel's last processed entry, the L2 gradient dL/dC = 2 w (C - target) / (3 W H)
// (mse, src/image.cpp:50-58) fused in the prologue, transmittance recovered by division, and
// the 7 per-splat 2D gradients (du, dv, dsigma2d, dopacity, drgb) summed per thread over its
// quad, reduce-scattered across the warp in 9 shuffles, combined across the two warps in
// shared memory and written (no atomics) to the (tile, splat) pair's own slot in emission
// order; K8 then sums each splat's slots in a fixed order -> deterministic gradients.
#include "isg_math.cuh"

namespace isg {

namespace {
constexpr int kBT = 64;     // threads per tile CTA (2 warps x 32 quads)
constexpr int kBatch = 64;  // records staged per batch
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

struct Stage {
  float4 geo[kBatch];  // u, v, r2max, -log2e / sigma2d^2
  float4 col[kBatch];  // r, g, b, opacity
  uint32_t slot[kBatch];  // emission index of the (tile, splat) pair
};

// Stage list entries [beg, beg+cnt) of the sorted key array into `st` (thread t: entry t).
__device__ __forceinline__ void stage_batch(Stage& st, const uint32_t* __restrict__ vals,
                                            const uint32_t* __restrict__ emit_rank,
                                            const RenderRec* __restrict__ rec, uint32_t beg,
                                            int cnt) {
  const int t = threadIdx.x;
  if (t < cnt) {
    const uint32_t e = vals[beg + t];
    const uint32_t r = emit_rank[e];
    st.slot[t] = e;
    cp_async16(&st.geo[t], &rec[r].geo);
    cp_async16(&st.col[t], &rec[r].col);
  }
  cp_async_commit();
}

// Per-thread quad geometry.
struct Quad {
  float px0, px1, py0, py1;
  bool valid[4];  // (x0,y0) (x1,y0) (x0,y1) (x1,y1)
  float wx0, wx1, wy0, wy1;  // pixel-centre rectangle of the warp's half tile (clipped)
  bool warp_empty;
  int x0, y0;
};

__device__ __forceinline__ Quad make_quad(const FrameParams& fp, int tile) {
  Quad q;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tx = tile % fp.tiles_x, ty = tile / fp.tiles_x;
  const int W = fp.cam.width, H = fp.cam.height;
  q.x0 = tx * kTile + 2 * (lane & 7);
  q.y0 = ty * kTile + w * 8 + 2 * (lane >> 3);
  q.px0 = (float)q.x0 + 0.5f;
  q.px1 = q.px0 + 1.0f;
  q.py0 = (float)q.y0 + 0.5f;
  q.py1 = q.py0 + 1.0f;
  q.valid[0] = q.x0 < W && q.y0 < H;
  q.valid[1] = q.x0 + 1 < W && q.y0 < H;
  q.valid[2] = q.x0 < W && q.y0 + 1 < H;
  q.valid[3] = q.x0 + 1 < W && q.y0 + 1 < H;
  const int wy = ty * kTile + w * 8;
  q.warp_empty = wy >= H;
  q.wx0 = (float)(tx * kTile) + 0.5f;
  q.wx1 = (float)(min(tx * kTile + kTile, W) - 1) + 0.5f;
  q.wy0 = (float)wy + 0.5f;
  q.wy1 = (float)(min(wy + 8, H) - 1) + 0.5f;
  return q;
}

// Does the 3-sigma circle reach the warp's pixel-centre rectangle?  (conservative, exact
// rounding like tile_hit, so no covered pixel is ever skipped)
__device__ __forceinline__ bool warp_hit(const Quad& q, float u, float v, float r2max) {
  const float cx = u < q.wx0 ? q.wx0 : (u > q.wx1 ? q.wx1 : u);
  const float cy = v < q.wy0 ? q.wy0 : (v > q.wy1 ? q.wy1 : v);
  return !(dist2_rn(__fsub_rn(cx, u), __fsub_rn(cy, v)) > r2max);
}

// reduce-scatter of 8 values over the warp in 9 shuffles: lane L returns the warp-wide sum of
// value (L >> 2) & 7.
__device__ __forceinline__ float reduce_scatter8(const float v[8]) {
  const int lane = threadIdx.x & 31;
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  float w[4], x[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = b4 ? v[i] : v[i + 4];
    const float keep = b4 ? v[i + 4] : v[i];
    w[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = b3 ? w[i] : w[i + 2];
    const float keep = b3 ? w[i + 2] : w[i];
    x[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  const float send = b2 ? x[0] : x[1];
  const float keep = b2 ? x[1] : x[0];
  float y = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  y += __shfl_xor_sync(0xffffffffu, y, 2);
  y += __shfl_xor_sync(0xffffffffu, y, 1);
  return y;
}

}  // namespace

// =============================================================================================
__global__ void __launch_bounds__(kBT) k_blend_fwd(
    FrameParams fp, const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
    const uint32_t* __restrict__ emit_rank, const RenderRec* __restrict__ rec,
    const unsigned long long* __restrict__ total, int64_t key_cap, float* __restrict__ out,
    float* __restrict__ t_last, uint32_t* __restrict__ n_proc) {
  __shared__ Stage st[2];
  if (overflowed(total, key_cap)) return;
  const int tile = blockIdx.x;
  const Quad q = make_quad(fp, tile);
  const uint2 rg = ranges[tile];
  const int n = (int)(rg.y - rg.x);

  float T[4], Tl[4], C[4][3];
  uint32_t np[4];
  bool done[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    T[p] = 1.0f;
    Tl[p] = 1.0f;
    C[p][0] = C[p][1] = C[p][2] = 0.0f;
    np[p] = 0;
    done[p] = !q.valid[p];
  }
  const float t_min = fp.t_min;
  if (n > 0) stage_batch(st[0], vals, emit_rank, rec, rg.x, min(kBatch, n));
  for (int b = 0, it = 0; b < n; b += kBatch, ++it) {
    Stage& cur = st[it & 1];
    cp_async_wait_all();
    const bool tdone = done[0] && done[1] && done[2] && done[3];
    if (__syncthreads_count(tdone) == kBT) break;  // barrier: batch visible, previous consumed
    if (b + kBatch < n) stage_batch(st[(it + 1) & 1], vals, emit_rank, rec, rg.x + b + kBatch,
                                    min(kBatch, n - b - kBatch));
    if (tdone || q.warp_empty) continue;
    const int cnt = min(kBatch, n - b);
    for (int j = 0; j < cnt; ++j) {
      const float4 g = cur.geo[j];
      if (!warp_hit(q, g.x, g.y, g.z)) continue;
      const float dx0 = __fsub_rn(q.px0, g.x), dx1 = __fsub_rn(q.px1, g.x);
      const float dy0 = __fsub_rn(q.py0, g.y), dy1 = __fsub_rn(q.py1, g.y);
      const float ax0 = __fmul_rn(dx0, dx0), ax1 = __fmul_rn(dx1, dx1);
      const float ay0 = __fmul_rn(dy0, dy0), ay1 = __fmul_rn(dy1, dy1);
      float r2[4];
      r2[0] = __fadd_rn(ax0, ay0);
      r2[1] = __fadd_rn(ax1, ay0);
      r2[2] = __fadd_rn(ax0, ay1);
      r2[3] = __fadd_rn(ax1, ay1);
      bool in[4];
      bool any = false;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        in[p] = !(r2[p] > g.z) && !done[p];
        any |= in[p];
      }
      if (!any) continue;
      const float4 c = cur.col[j];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        if (!in[p]) continue;
        const float e = fast_exp2(r2[p] * g.w);
        const float a = c.w * e;
        const float wgt = T[p] * a;
        C[p][0] += wgt * c.x;
        C[p][1] += wgt * c.y;
        C[p][2] += wgt * c.z;
        Tl[p] = T[p];
        T[p] = T[p] * (1.0f - a);
        np[p] = (uint32_t)(b + j + 1);
        done[p] = !(T[p] > t_min);
      }
      if (done[0] && done[1] && done[2] && done[3]) break;
    }
  }
  cp_async_wait_all();
  const int W = fp.cam.width;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    if (!q.valid[p]) continue;
    const size_t pix = (size_t)(q.y0 + (p >> 1)) * W + q.x0 + (p & 1);
    out[3 * pix + 0] = C[p][0] + T[p] * fp.bg[0];
    out[3 * pix + 1] = C[p][1] + T[p] * fp.bg[1];
    out[3 * pix + 2] = C[p][2] + T[p] * fp.bg[2];
    t_last[pix] = Tl[p];
    n_proc[pix] = np[p];
  }
}

// =============================================================================================
__global__ void __launch_bounds__(kBT) k_blend_bwd(
    FrameParams fp, const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
    const uint32_t* __restrict__ emit_rank, const RenderRec* __restrict__ rec,
    const unsigned long long* __restrict__ total, int64_t key_cap, const float* __restrict__ img,
    const float* __restrict__ target, const float* __restrict__ t_last,
    const uint32_t* __restrict__ n_proc, float loss_scale, float4* __restrict__ partial,
    double* __restrict__ tile_loss) {
  __shared__ Stage st[2];
  __shared__ float s_part[2][8][kBatch];  // [warp][value][entry]
  __shared__ float s_red[2];
  __shared__ uint32_t s_max[2];
  const int tile = blockIdx.x;
  if (overflowed(total, key_cap)) {
    if (threadIdx.x == 0) tile_loss[tile] = 0.0;
    return;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const Quad q = make_quad(fp, tile);
  const uint2 rg = ranges[tile];
  const int n = (int)(rg.y - rg.x);
  const int W = fp.cam.width;

  float G[4][3], T[4], A[4][3];
  uint32_t np[4];
  bool first[4];
  float dsq = 0.0f;
  uint32_t npmax = 0;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    G[p][0] = G[p][1] = G[p][2] = 0.0f;
    T[p] = 0.0f;
    np[p] = 0;
    first[p] = true;
    A[p][0] = fp.bg[0];
    A[p][1] = fp.bg[1];
    A[p][2] = fp.bg[2];
    if (q.valid[p]) {
      const size_t pix = (size_t)(q.y0 + (p >> 1)) * W + q.x0 + (p & 1);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float d = img[3 * pix + c] - target[3 * pix + c];
        dsq += d * d;
        G[p][c] = 2.0f * d * loss_scale;
      }
      T[p] = t_last[pix];
      np[p] = n_proc[pix];
      npmax = max(npmax, np[p]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dsq += __shfl_xor_sync(0xffffffffu, dsq, o);
    npmax = max(npmax, __shfl_xor_sync(0xffffffffu, npmax, o));
  }
  if (lane == 0) {
    s_red[w] = dsq;
    s_max[w] = npmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) tile_loss[tile] = (double)s_red[0] + (double)s_red[1];
  const int m = (int)max(s_max[0], s_max[1]);  // entries [0, m) are walked

  // entries never reached by any pixel get zero gradient slots
  for (int j = m + (int)threadIdx.x; j < n; j += kBT) {
    const uint32_t e = vals[rg.x + j];
    partial[2 * (size_t)e] = make_float4(0.f, 0.f, 0.f, 0.f);
    partial[2 * (size_t)e + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (m == 0) return;

  int hi = m;
  stage_batch(st[0], vals, emit_rank, rec, rg.x + max(0, hi - kBatch), min(kBatch, hi));
  for (int it = 0; hi > 0; ++it) {
    const int lo = max(0, hi - kBatch);
    const int cnt = hi - lo;
    Stage& cur = st[it & 1];
    cp_async_wait_all();
    __syncthreads();  // batch visible; previous batch's flush finished reading s_part
    if (lo > 0) {
      const int nlo = max(0, lo - kBatch);
      stage_batch(st[(it + 1) & 1], vals, emit_rank, rec, rg.x + nlo, lo - nlo);
    }
    for (int jj = cnt - 1; jj >= 0; --jj) {
      const int j = lo + jj;
      const float4 g = cur.geo[jj];
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      bool contrib = false;
      if (!q.warp_empty && warp_hit(q, g.x, g.y, g.z)) {
        const float dx[2] = {__fsub_rn(q.px0, g.x), __fsub_rn(q.px1, g.x)};
        const float dy[2] = {__fsub_rn(q.py0, g.y), __fsub_rn(q.py1, g.y)};
        const float ax[2] = {__fmul_rn(dx[0], dx[0]), __fmul_rn(dx[1], dx[1])};
        const float ay[2] = {__fmul_rn(dy[0], dy[0]), __fmul_rn(dy[1], dy[1])};
        bool act[4];
        float r2[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          r2[p] = __fadd_rn(ax[p & 1], ay[p >> 1]);
          act[p] = (uint32_t)j < np[p] && !(r2[p] > g.z);
          contrib |= act[p];
        }
        if (contrib) {
          const float4 c = cur.col[jj];
          const float two_inv_s2 = g.w * (-2.0f * kLn2);  // 2 / sigma2d^2
          const float inv_s = sqrtf(two_inv_s2 * 0.5f);   // 1 / sigma2d
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            if (!act[p]) continue;
            const float e = fast_exp2(r2[p] * g.w);
            const float a = c.w * e;
            const float Tk = first[p] ? T[p] : __fdividef(T[p], 1.0f - a);
            first[p] = false;
            T[p] = Tk;
            const float dLda =
                Tk * (G[p][0] * (c.x - A[p][0]) + G[p][1] * (c.y - A[p][1]) +
                      G[p][2] * (c.z - A[p][2]));
            const float Ta = Tk * a;
            acc[4] += G[p][0] * Ta;
            acc[5] += G[p][1] * Ta;
            acc[6] += G[p][2] * Ta;
            A[p][0] = a * c.x + (1.0f - a) * A[p][0];
            A[p][1] = a * c.y + (1.0f - a) * A[p][1];
            A[p][2] = a * c.z + (1.0f - a) * A[p][2];
            acc[3] += dLda * e;
            const float k2 = dLda * c.w * e * two_inv_s2;
            acc[0] += k2 * dx[p & 1];
            acc[1] += k2 * dy[p >> 1];
            acc[2] += k2 * r2[p] * inv_s;
          }
        }
      }
      if (__any_sync(0xffffffffu, contrib)) {
        const float y = reduce_scatter8(acc);
        if ((lane & 3) == 0) s_part[w][lane >> 2][jj] = y;
      } else if (lane < 8) {
        s_part[w][lane][jj] = 0.0f;
      }
    }
    __syncthreads();
    // combine the two warps and write each (tile, splat) pair's gradient slot
    if ((int)threadIdx.x < cnt) {
      const int jj = threadIdx.x;
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = s_part[0][k][jj] + s_part[1][k][jj];
      const size_t e = cur.slot[jj];
      partial[2 * e] = make_float4(v[0], v[1], v[2], v[3]);
      partial[2 * e + 1] = make_float4(v[4], v[5], v[6], 0.0f);
    }
    hi = lo;
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
                      const uint32_t* emit_rank, const RenderRec* rec,
                      const unsigned long long* total, int64_t key_cap, float* out, float* t_last,
                      uint32_t* n_proc, cudaStream_t st) {
  k_blend_fwd<<<fp.n_tiles, kBT, 0, st>>>(fp, ranges, vals, emit_rank, rec, total, key_cap, out,
                                          t_last, n_proc);
}

void launch_blend_bwd(const FrameParams& fp, const uint2* ranges, const uint32_t* vals,
                      const uint32_t* emit_rank, const RenderRec* rec,
                      const unsigned long long* total, int64_t key_cap, const float* img,
                      const float* target, const float* t_last, const uint32_t* n_proc,
                      float loss_scale, float4* partial, double* tile_loss, cudaStream_t st) {
  k_blend_bwd<<<fp.n_tiles, kBT, 0, st>>>(fp, ranges, vals, emit_rank, rec, total, key_cap, img,
                                          target, t_last, n_proc, loss_scale, partial, tile_loss);
}

void launch_loss_reduce(const double* tile_loss, int n_tiles, double scale, double* loss,
                        cudaStream_t st) {
  k_loss_reduce<<<1, 256, 0, st>>>(tile_loss, n_tiles, scale, loss);
}

}  // namespace isg

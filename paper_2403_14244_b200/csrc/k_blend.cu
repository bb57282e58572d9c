// K6/K7 — per-16x16-tile alpha blending, forward and backward.
//
// K6 replaces composite_pixels (/root/reference/proj/src/splat3d.cpp:125-162) and the
// inclusion test covers(ScreenIso) (:108-114).  Instead of every pixel visiting every splat
// (O(W*H*N)), one CTA owns one tile and walks only that tile's depth-ordered list.
//
// Mapping (both kernels): 128 threads per tile; warp w owns the 8x8 quarter-tile w and each
// lane a vertical pixel pair, so one shared-memory record feeds two pixels that share dx.
// Records are staged 128 at a time into shared memory with cp.async, double-buffered (the
// next batch's copy is in flight while the current one is blended).  The staging thread also
// tests the splat's 3-sigma circle against the four quarter-tiles (conservative closest-point
// test, exact rounding) and stores a 4-bit mask; each warp turns the masks into a 128-bit
// ballot and iterates only over the entries that can touch its quarter — culling costs ~nothing
// and non-overlapping entries cost no issue slots at all.  Compositing is branch-free.
// The forward stops once every pixel of the tile has transmittance <= t_min.
//
// The 3-sigma test is bit-identical to the FP32 oracle (explicit _rn arithmetic); exp uses
// ex2.approx on a per-splat precomputed -log2(e)/sigma2d^2.
//
// K7 is the backward the reference does not have: the same walk in reverse from
// each pixel's last processed entry, the L2 gradient dL/dC = 2 w (C - target) / (3 W H)
// (mse, src/image.cpp:50-58) fused in the prologue, transmittance recovered by division, and
// the 7 per-splat 2D gradients (du, dv, dsigma2d, dopacity, drgb) summed per thread over its two
// pixels, reduce-scattered across the warp in 9 shuffles, combined across the four warps in
// shared memory and written (no atomics) to the (tile, splat) pair's own slot in emission
// order; K8 then sums each splat's slots in a fixed order -> deterministic gradients.
#include "isg_math.cuh"

namespace isg {

namespace {
constexpr int kBT = 128;     // threads per tile CTA (4 warps x 32 pixel pairs)
constexpr int kBatch = 128;  // records staged per batch (one per thread)
constexpr int kWarps = kBT / 32;
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
  float4 geo[kBatch];     // u, v, r2max, -log2e / sigma2d^2
  float4 col[kBatch];     // r, g, b, opacity
  uint32_t slot[kBatch];  // emission index of the (tile, splat) pair
};

// Pixel-centre rectangle of this warp's quarter-tile, clipped to the image.
struct TileGeom {
  float qx0, qx1, qy0, qy1;
  bool qvalid;
};

__device__ __forceinline__ TileGeom tile_geom(const FrameParams& fp, int tile) {
  TileGeom t;
  const int w = threadIdx.x >> 5;
  const int tx = tile % fp.tiles_x, ty = tile / fp.tiles_x;
  const int W = fp.cam.width, H = fp.cam.height;
  const int x0 = tx * kTile + (w & 1) * 8, y0 = ty * kTile + (w >> 1) * 8;
  t.qvalid = x0 < W && y0 < H;
  t.qx0 = (float)x0 + 0.5f;
  t.qx1 = (float)(min(x0 + 8, W) - 1) + 0.5f;
  t.qy0 = (float)y0 + 0.5f;
  t.qy1 = (float)(min(y0 + 8, H) - 1) + 0.5f;
  return t;
}

// 3-sigma circle vs pixel-centre rectangle (conservative, exact rounding like tile_hit).
__device__ __forceinline__ bool rect_hit(float x0, float x1, float y0, float y1, float u, float v,
                                         float r2max) {
  const float cx = fminf(fmaxf(u, x0), x1);
  const float cy = fminf(fmaxf(v, y0), y1);
  return !(dist2_rn(__fsub_rn(cx, u), __fsub_rn(cy, v)) > r2max);
}

// Stage list entries [beg, beg+cnt) of the sorted (splat, slot) array into `st` (thread t:
// entry t).  The 32-B record gather is issued as cp.async.
__device__ __forceinline__ void stage_batch(Stage& st, const uint2* __restrict__ sorted,
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

// 128-bit relevance mask of the staged batch for warp w: bit j <=> entry j's 3-sigma circle can
// reach the warp's quarter-tile.  Lane l tests entries l, l+32, l+64, l+96.
__device__ __forceinline__ void warp_relevance(const Stage& st, const TileGeom& tg, int w,
                                               int cnt, uint32_t rel[4]) {
  (void)w;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int j = 32 * k + lane;
    bool hit = false;
    if (j < cnt && tg.qvalid) {
      const float4 g = st.geo[j];
      hit = rect_hit(tg.qx0, tg.qx1, tg.qy0, tg.qy1, g.x, g.y, g.z);
    }
    rel[k] = __ballot_sync(0xffffffffu, hit);
  }
}

// Compact the warp's relevant entries of the batch into `list` (ascending); returns the count.
// The blend loops then cost ~3 instructions per relevant entry for iteration.
__device__ __forceinline__ int warp_compact(const uint32_t rel[4], uint8_t* list) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  int base = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if ((rel[k] >> lane) & 1u) list[base + __popc(rel[k] & lt)] = (uint8_t)(32 * k + lane);
    base += __popc(rel[k]);
  }
  __syncwarp();
  return base;
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

struct PixPair {
  int x, y0;        // pixels (x, y0) and (x, y0 + 1)
  float px, py0, py1;
  bool valid0, valid1;
};

__device__ __forceinline__ PixPair pix_pair(const FrameParams& fp, int tile) {
  PixPair p;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tx = tile % fp.tiles_x, ty = tile / fp.tiles_x;
  p.x = tx * kTile + (w & 1) * 8 + (lane & 7);
  p.y0 = ty * kTile + (w >> 1) * 8 + 2 * (lane >> 3);
  p.px = (float)p.x + 0.5f;
  p.py0 = (float)p.y0 + 0.5f;
  p.py1 = p.py0 + 1.0f;
  p.valid0 = p.x < fp.cam.width && p.y0 < fp.cam.height;
  p.valid1 = p.x < fp.cam.width && p.y0 + 1 < fp.cam.height;
  return p;
}

}  // namespace

// =============================================================================================
__global__ void __launch_bounds__(kBT) k_blend_fwd(
    FrameParams fp, const uint2* __restrict__ ranges, const uint2* __restrict__ sorted,
    const RenderRec* __restrict__ rec,
    const unsigned long long* __restrict__ total, int64_t key_cap, float* __restrict__ out,
    float* __restrict__ t_last, uint32_t* __restrict__ n_proc) {
  __shared__ Stage st[2];
  __shared__ uint8_t s_list[kWarps][kBatch];
  if (overflowed(total, key_cap)) return;
  const int tile = blockIdx.x;
  const int w = threadIdx.x >> 5;
  const TileGeom tg = tile_geom(fp, tile);
  const PixPair pp = pix_pair(fp, tile);
  const uint2 rg = ranges[tile];
  const int n = (int)(rg.y - rg.x);
  const float t_min = fp.t_min;

  // invalid pixels start "terminated" (T = 0 <= t_min) and never contribute
  float T0 = pp.valid0 ? 1.0f : 0.0f, T1 = pp.valid1 ? 1.0f : 0.0f;
  float Tl0 = 1.0f, Tl1 = 1.0f;
  float C0r = 0.f, C0g = 0.f, C0b = 0.f, C1r = 0.f, C1g = 0.f, C1b = 0.f;
  uint32_t np0 = 0, np1 = 0;

  if (n > 0) stage_batch(st[0], sorted, rec, rg.x, min(kBatch, n));
  for (int b = 0, it = 0; b < n; b += kBatch, ++it) {
    Stage& cur = st[it & 1];
    cp_async_wait_all();
    const bool tdone = !(T0 > t_min) && !(T1 > t_min);
    if (__syncthreads_count(tdone) == kBT) break;  // barrier: batch visible, previous consumed
    if (b + kBatch < n)
      stage_batch(st[(it + 1) & 1], sorted, rec, rg.x + b + kBatch,
                  min(kBatch, n - b - kBatch));
    uint32_t rel[4];
    warp_relevance(cur, tg, w, min(kBatch, n - b), rel);
    const int nrel = warp_compact(rel, s_list[w]);
    {
      for (int i = 0; i < nrel; ++i) {
        const int jj = s_list[w][i];
        const float4 g = cur.geo[jj];
        const float4 c = cur.col[jj];
        const float dx = __fsub_rn(pp.px, g.x);
        const float ax = __fmul_rn(dx, dx);
        const float dy0 = __fsub_rn(pp.py0, g.y), dy1 = __fsub_rn(pp.py1, g.y);
        const float r20 = __fadd_rn(ax, __fmul_rn(dy0, dy0));
        const float r21 = __fadd_rn(ax, __fmul_rn(dy1, dy1));
        const bool in0 = !(r20 > g.z) && (T0 > t_min);
        const bool in1 = !(r21 > g.z) && (T1 > t_min);
        const uint32_t idx = (uint32_t)(b + jj + 1);
        const float a0 = in0 ? c.w * fast_exp2(r20 * g.w) : 0.0f;
        const float a1 = in1 ? c.w * fast_exp2(r21 * g.w) : 0.0f;
        const float w0 = T0 * a0, w1 = T1 * a1;
        C0r += w0 * c.x;
        C0g += w0 * c.y;
        C0b += w0 * c.z;
        C1r += w1 * c.x;
        C1g += w1 * c.y;
        C1b += w1 * c.z;
        Tl0 = in0 ? T0 : Tl0;
        Tl1 = in1 ? T1 : Tl1;
        np0 = in0 ? idx : np0;
        np1 = in1 ? idx : np1;
        T0 = T0 * (1.0f - a0);
        T1 = T1 * (1.0f - a1);
      }
    }
  }
  cp_async_wait_all();
  const int W = fp.cam.width;
  if (pp.valid0) {
    const size_t pix = (size_t)pp.y0 * W + pp.x;
    out[3 * pix + 0] = C0r + T0 * fp.bg[0];
    out[3 * pix + 1] = C0g + T0 * fp.bg[1];
    out[3 * pix + 2] = C0b + T0 * fp.bg[2];
    t_last[pix] = Tl0;
    n_proc[pix] = np0;
  }
  if (pp.valid1) {
    const size_t pix = (size_t)(pp.y0 + 1) * W + pp.x;
    out[3 * pix + 0] = C1r + T1 * fp.bg[0];
    out[3 * pix + 1] = C1g + T1 * fp.bg[1];
    out[3 * pix + 2] = C1b + T1 * fp.bg[2];
    t_last[pix] = Tl1;
    n_proc[pix] = np1;
  }
}

// =============================================================================================
// One pixel of the reverse walk (branch-free; inactive pixels contribute exact zeros).
struct BwdPix {
  float G0, G1, G2;  // dL/dC
  float T;           // transmittance before the most recently processed (later) entry
  float A0, A1, A2;  // colour behind, normalised
  uint32_t np;
  bool first;
};

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

// acc: [0] sum go*dx, [1] sum go*dy, [2] sum go*r2 (scaled per entry by the caller into
// du, dv, dsigma2d), [3] dopacity, [4..6] drgb;  go = dL/dalpha * g.
// An inactive pixel gets e = 0, hence a = 0: T is unchanged exactly (T * rcp(1) = T), A is
// unchanged (A + 0), and every contribution (Ta = T a, go = dL/da e) is an exact zero.
__device__ __forceinline__ void bwd_pixel(BwdPix& p, bool act, float dx, float dy, float r2,
                                          const float4 g, const float4 c, float acc[8]) {
  const float e = act ? fast_exp2(r2 * g.w) : 0.0f;
  const float a = c.w * e;
  const float Tk = p.first ? p.T : p.T * fast_rcp(1.0f - a);
  p.first = p.first && !act;
  p.T = Tk;
  const float d0 = c.x - p.A0, d1 = c.y - p.A1, d2 = c.z - p.A2;
  const float dLda = Tk * (p.G0 * d0 + p.G1 * d1 + p.G2 * d2);
  const float Ta = Tk * a;
  acc[4] += p.G0 * Ta;
  acc[5] += p.G1 * Ta;
  acc[6] += p.G2 * Ta;
  p.A0 += a * d0;  // A <- a c + (1 - a) A
  p.A1 += a * d1;
  p.A2 += a * d2;
  const float go = dLda * e;
  acc[3] += go;
  acc[0] += go * dx;
  acc[1] += go * dy;
  acc[2] += go * r2;
}

__global__ void __launch_bounds__(kBT) k_blend_bwd(
    FrameParams fp, const uint2* __restrict__ ranges, const uint2* __restrict__ sorted,
    const RenderRec* __restrict__ rec,
    const unsigned long long* __restrict__ total, int64_t key_cap, const float* __restrict__ img,
    const float* __restrict__ target, const float* __restrict__ t_last,
    const uint32_t* __restrict__ n_proc, float loss_scale, float4* __restrict__ partial,
    double* __restrict__ tile_loss) {
  __shared__ Stage st[2];
  // [warp][value][entry], rows padded by one word so the 8 values of one entry (written by
  // lanes 0,4,..,28 at once) fall in 8 different banks
  __shared__ float s_part[kWarps][8][kBatch + 1];
  __shared__ uint32_t s_rel[kWarps][4];
  __shared__ uint8_t s_list[kWarps][kBatch];
  __shared__ float s_red[kWarps];
  __shared__ uint32_t s_max[kWarps];
  const int tile = blockIdx.x;
  if (overflowed(total, key_cap)) {
    if (threadIdx.x == 0) tile_loss[tile] = 0.0;
    return;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const TileGeom tg = tile_geom(fp, tile);
  const PixPair pp = pix_pair(fp, tile);
  const uint2 rg = ranges[tile];
  const int n = (int)(rg.y - rg.x);
  const int W = fp.cam.width;

  BwdPix P[2];
  float dsq = 0.0f;
  uint32_t npmax = 0;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    BwdPix& p = P[q];
    p.G0 = p.G1 = p.G2 = 0.0f;
    p.T = 0.0f;
    p.np = 0;
    p.first = true;
    p.A0 = fp.bg[0];
    p.A1 = fp.bg[1];
    p.A2 = fp.bg[2];
    if (q == 0 ? pp.valid0 : pp.valid1) {
      const size_t pix = (size_t)(pp.y0 + q) * W + pp.x;
      const float d0 = img[3 * pix + 0] - target[3 * pix + 0];
      const float d1 = img[3 * pix + 1] - target[3 * pix + 1];
      const float d2 = img[3 * pix + 2] - target[3 * pix + 2];
      dsq += d0 * d0 + d1 * d1 + d2 * d2;
      p.G0 = 2.0f * d0 * loss_scale;
      p.G1 = 2.0f * d1 * loss_scale;
      p.G2 = 2.0f * d2 * loss_scale;
      p.T = t_last[pix];
      p.np = n_proc[pix];
      npmax = max(npmax, p.np);
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
  int m = 0;
#pragma unroll
  for (int i = 0; i < kWarps; ++i) m = max(m, (int)s_max[i]);
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < kWarps; ++i) t += (double)s_red[i];
    tile_loss[tile] = t;
  }
  // entries never reached by any pixel get zero gradient slots
  for (int j = m + (int)threadIdx.x; j < n; j += kBT) {
    const uint32_t e = sorted[rg.x + j].y;
    partial[2 * (size_t)e] = make_float4(0.f, 0.f, 0.f, 0.f);
    partial[2 * (size_t)e + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (m == 0) return;

  int hi = m;
  stage_batch(st[0], sorted, rec, rg.x + max(0, hi - kBatch), min(kBatch, hi));
  for (int it = 0; hi > 0; ++it) {
    const int lo = max(0, hi - kBatch);
    const int cnt = hi - lo;
    Stage& cur = st[it & 1];
    cp_async_wait_all();
    __syncthreads();  // batch visible; previous batch's flush finished reading s_part
    if (lo > 0) {
      const int nlo = max(0, lo - kBatch);
      stage_batch(st[(it + 1) & 1], sorted, rec, rg.x + nlo, lo - nlo);
    }
    uint32_t rel[4];
    warp_relevance(cur, tg, w, cnt, rel);
    const int nrel = warp_compact(rel, s_list[w]);
    {
      for (int i = nrel - 1; i >= 0; --i) {
        const int jj = s_list[w][i];
        const int j = lo + jj;
        const float4 g = cur.geo[jj];
        const float4 c = cur.col[jj];
        const float dx = __fsub_rn(pp.px, g.x);
        const float ax = __fmul_rn(dx, dx);
        const float dy0 = __fsub_rn(pp.py0, g.y), dy1 = __fsub_rn(pp.py1, g.y);
        const float r20 = __fadd_rn(ax, __fmul_rn(dy0, dy0));
        const float r21 = __fadd_rn(ax, __fmul_rn(dy1, dy1));
        const bool act0 = (uint32_t)j < P[0].np && !(r20 > g.z);
        const bool act1 = (uint32_t)j < P[1].np && !(r21 > g.z);
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        bwd_pixel(P[0], act0, dx, dy0, r20, g, c, acc);
        bwd_pixel(P[1], act1, dx, dy1, r21, g, c, acc);
        // kernels.hpp:219-220 closed forms: dg/du = g 2 dx/s^2, dg/ds = g 2 r^2/s^3, times opacity
        const float inv_s2 = g.w * -kLn2;          // 1 / sigma2d^2
        const float k = 2.0f * c.w * inv_s2;       // 2 o / s^2
        acc[0] *= k;
        acc[1] *= k;
        acc[2] *= k * fast_sqrt(inv_s2);           // 2 o / s^3
        const float y = reduce_scatter8(acc);
        if ((lane & 3) == 0) s_part[w][lane >> 2][jj] = y;
      }
    }
    // fix the relevance words: lanes 0..3 of warp w hold rel[k] only for k == lane
    if (lane < 4) {
      uint32_t r = rel[0];
      r = lane == 1 ? rel[1] : r;
      r = lane == 2 ? rel[2] : r;
      r = lane == 3 ? rel[3] : r;
      s_rel[w][lane] = r;
    }
    __syncthreads();
    // combine the warps and write each (tile, splat) pair's gradient slot
    if ((int)threadIdx.x < cnt) {
      const int jj = threadIdx.x;
      float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ww = 0; ww < kWarps; ++ww) {
        if (!((s_rel[ww][jj >> 5] >> (jj & 31)) & 1u)) continue;
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] += s_part[ww][k][jj];
      }
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

void launch_blend_fwd(const FrameParams& fp, const uint2* ranges, const uint2* sorted,
                      const RenderRec* rec, const unsigned long long* total, int64_t key_cap,
                      float* out, float* t_last, uint32_t* n_proc, cudaStream_t st) {
  k_blend_fwd<<<fp.n_tiles, kBT, 0, st>>>(fp, ranges, sorted, rec, total, key_cap, out, t_last,
                                          n_proc);
}

void launch_blend_bwd(const FrameParams& fp, const uint2* ranges, const uint2* sorted,
                      const RenderRec* rec, const unsigned long long* total, int64_t key_cap,
                      const float* img,
                      const float* target, const float* t_last, const uint32_t* n_proc,
                      float loss_scale, float4* partial, double* tile_loss, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_blend_bwd, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr = true;
  }
  k_blend_bwd<<<fp.n_tiles, kBT, 0, st>>>(fp, ranges, sorted, rec, total, key_cap, img,
                                          target, t_last, n_proc, loss_scale, partial, tile_loss);
}

void launch_loss_reduce(const double* tile_loss, int n_tiles, double scale, double* loss,
                        cudaStream_t st) {
  k_loss_reduce<<<1, 256, 0, st>>>(tile_loss, n_tiles, scale, loss);
}

}  // namespace isg

// K6 — per-16x16-tile front-to-back alpha blending (forward).
//
// Replaces composite_pixels (/root/reference/proj/src/splat3d.cpp:125-162) and the inclusion
// test covers(ScreenIso) (:108-114).  Instead of every pixel visiting every splat
// (O(W*H*N)), one CTA owns one tile and walks only that tile's depth-ordered list.
//
// Mapping: 64 threads per tile (2 warps).  Each four-lane group owns one 4x4 sub-quarter and
// each lane a 2x2 pixel quad, processed as two packed f32x2 pixel pairs (one row each), so one
// shared-memory record feeds four pixels.  Records are staged 128 at a time into shared memory
// with cp.async, double-buffered (the next batch's copy is in flight while the current one is
// blended).  After each batch barrier every warp tests the staged splats' 3-sigma circles
// against its eight sub-quarters (conservative closest-point tests sharing per-axis terms,
// exact rounding), ballots, and compacts eight relevance lists; the groups walk their own
// lists in lockstep, padded with a sentinel record to the warp's step count.  The 4x4 culling
// cuts the pixel-entry slots a circle does not cover (a circle of the typical 6-px 3-sigma
// radius covers a 4x4 region far better than an 8x8).  Compositing is branch-free; a
// sub-quarter whose pixels all terminated walks nothing, and the CTA stops once every pixel
// has transmittance <= t_min.
//
// The 3-sigma test is bit-identical to the FP32 oracle (explicit _rn arithmetic); exp uses
// ex2.approx of r2 * (-log2(e)/sigma2d^2) + log2(opacity), both precomputed per splat by K1.
#include "blend_common.cuh"

namespace isg {

namespace {
using namespace blend;

constexpr int kBT = 64;      // threads per tile CTA: 2 warps x 8 four-lane groups
#ifndef ISG_FWD_BATCH
#define ISG_FWD_BATCH 128
#endif
// Register budget: a 12-CTA/SM minimum (80 registers) measured fastest for the relevance-testing
// forward of a train step (0.259 vs 0.275 ms at 116 registers with a 1-CTA minimum; 8 and 10
// CTAs in between).
#ifndef ISG_FWD_MINB
#define ISG_FWD_MINB 12
#endif
#if ISG_FWD_MINB > 0
#define ISG_FWD_BOUNDS __launch_bounds__(kBT, ISG_FWD_MINB)
#else
#define ISG_FWD_BOUNDS __launch_bounds__(kBT)
#endif
// 4 walk steps per loop iteration: C2 0.2213 vs 0.2255 ms unrolled by 1 (render, t_min = 0);
// train frames equal
#ifndef ISG_FWD_UNROLL
#define ISG_FWD_UNROLL 4
#endif
constexpr int kUnroll = ISG_FWD_UNROLL;  // walk steps per loop iteration
constexpr int kBatch = ISG_FWD_BATCH;  // records staged per batch
constexpr int kWords = kBatch / 32;
static_assert(kBatch < 256, "u8 list entries, sentinel index kBatch");
constexpr int kListPitch = kBatch + 4;  // sub-quarter lists start in different banks

// One row of a lane's 2x2 pixel quad: two horizontally adjacent pixels as packed f32x2 lanes
// (.x = (x0, y), .y = (x0 + 1, y)); FFMA2/FMUL2/FADD2 issue once for both.
struct FwdPair {
  float2 T;           // transmittance
  float2 Cr, Cg, Cb;  // accumulated colour
  float2 Tl;          // transmittance before the last contributor (the rare re-walk only)
  uint32_t np0, np1;  // 1 + index of the last contributor (entries the backward walks)
};

__device__ __forceinline__ float2 bc(float v) { return make_float2(v, v); }

// kTrack: also record, per pixel, the index of the last contributor (where the backward starts
// its walk); a render-only frame skips it.  kTl: also record the transmittance *before* the last
// contributor (the backward's starting state for pixels whose final transmittance is not a
// normal float, see k_blend_fwd).
// kTerm = false (an untracked frame at t_min = 0): the per-pixel termination test is dropped —
// once T reaches 0 every later contribution T a c and T (1 - a) is an exact zero anyway, so the
// image is bit-identical.
template <bool kTrack, bool kTl, bool kTerm = true>
__device__ __forceinline__ void fwd_pair(FwdPair& p, float2 r2, const float4 g, const float4 c,
                                         float t_min, uint32_t idx) {
  const bool in0 = !(r2.x > g.z) && (!kTerm || p.T.x > t_min);
  const bool in1 = !(r2.y > g.z) && (!kTerm || p.T.y > t_min);
  // an excluded pixel's exponential is never evaluated (predicated MUFU into a zeroed pair), so
  // its alpha is an exact 0
  // c.w holds log2(opacity) (K1): alpha = o exp(-r2 / s^2) = ex2(r2 g.w + log2 o), one
  // fused op (the backward forms it the same way)
  const float2 q = __ffma2_rn(r2, bc(g.w), bc(c.w));
  const float2 a = make_float2(in0 ? fast_exp2(q.x) : 0.0f, in1 ? fast_exp2(q.y) : 0.0f);
  const float2 wgt = __fmul2_rn(p.T, a);
  p.Cr = __ffma2_rn(wgt, bc(c.x), p.Cr);
  p.Cg = __ffma2_rn(wgt, bc(c.y), p.Cg);
  p.Cb = __ffma2_rn(wgt, bc(c.z), p.Cb);
  if constexpr (kTl) p.Tl = make_float2(in0 ? p.T.x : p.Tl.x, in1 ? p.T.y : p.Tl.y);
  if constexpr (kTrack) {
    p.np0 = in0 ? idx : p.np0;
    p.np1 = in1 ? idx : p.np1;
  }
  // T (1 - a) as T - T a: one op on the product already formed (the backward recovers
  // T_k = T_{k+1} / (1 - a_k) up to the same rounding either way)
  p.T = __fadd2_rn(p.T, make_float2(-wgt.x, -wgt.y));
}

}  // namespace

template <bool kTrack, bool kTerm>
__global__ void ISG_FWD_BOUNDS k_blend_fwd(
    FrameParams fp, const uint2* __restrict__ ranges, const uint2* __restrict__ sorted,
    uint16_t* __restrict__ submask,
    const RenderRec* __restrict__ rec, unsigned long long* __restrict__ total,
    int64_t key_cap, float* __restrict__ out, float* __restrict__ t_last,
    uint32_t* __restrict__ n_proc) {
  // entry kBatch of each stage is a sentinel no pixel is inside (r2max = -1): the groups'
  // lists are padded with it to the warp's step count, so the walk needs no bounds test
  __shared__ Stage<kBatch + 1> st[2];
  __shared__ uint8_t s_list[16][kListPitch];
  pdl_enter();
  if (overflowed(total, key_cap)) {
    // sticky record for the host's next check (survives later frames' resets): the largest
    // key count any frame since then needed, and how many frames were skipped
    if (blockIdx.x == 0 && threadIdx.x == 0) note_overflow(total);
    return;
  }
  if (threadIdx.x < 2) {
    st[threadIdx.x].geo[kBatch] = make_float4(0.0f, 0.0f, -1.0f, 0.0f);
    st[threadIdx.x].col[kBatch] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  }
  const int tile = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gq = lane >> 2, l4 = lane & 3;  // four-lane group = one 4x4 sub-quarter
  const int sub = 8 * w + gq;
  const int q = sub >> 2, sq = sub & 3;
  const int tx = tile % fp.tiles_x, ty = tile / fp.tiles_x;
  const int W = fp.cam.width, H = fp.cam.height;
  const int x0 = tx * kTile + (q & 1) * 8 + (sq & 1) * 4 + 2 * (l4 & 1);
  const int y0 = ty * kTile + (q >> 1) * 8 + (sq >> 1) * 4 + 2 * (l4 >> 1);
  const float2 PX = make_float2((float)x0 + 0.5f, (float)x0 + 1.5f);
  const float2 PY = make_float2((float)y0 + 0.5f, (float)y0 + 1.5f);
  // the warp's 8 sub-quarters: 4 columns of the tile (x = 4c) x 2 rows (y = 8w + 4r)
  // Untracked frames give a column or row of sub-quarters outside the image the span 1e30:
  // the rounded square of the distance is +inf and no record tests relevant to it, so the
  // per-record tests need no validity predicates (render 0.1995 -> 0.1974 ms).  Tracked frames
  // keep the predicates (without them ptxas spills in that variant).
  float cx0[4], cx1[4], ry0[2], ry1[2];
  bool cv[4], rv[2];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int xs = tx * kTile + 4 * c;
    cv[c] = xs < W;
    cx0[c] = (kTrack || xs < W) ? (float)xs + 0.5f : 1e30f;
    cx1[c] = (kTrack || xs < W) ? (float)(min(xs + 4, W) - 1) + 0.5f : 1e30f;
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int ys = ty * kTile + 8 * w + 4 * r;
    rv[r] = ys < H;
    ry0[r] = (kTrack || ys < H) ? (float)ys + 0.5f : 1e30f;
    ry1[r] = (kTrack || ys < H) ? (float)(min(ys + 4, H) - 1) + 0.5f : 1e30f;
  }
  // tracked frames leave each entry's relevance bits for the backward: byte w of submask[e]
  uint8_t* const mask_bytes = reinterpret_cast<uint8_t*>(submask);
  const uint2 rg = ranges[tile];
  const int n = rg.x == kEmptyRange ? 0 : (int)(rg.y - rg.x);
  const float t_min = fp.t_min;

  const uint32_t lt = (1u << lane) - 1u;
  FwdPair P[2];
  // One walk over the tile's list.  kTl = false is every frame's walk; kTl = true the rare
  // re-walk of a tracked frame that also records the transmittance before the last contributor.
  auto walk = [&](auto tl_tag) {
  constexpr bool kTl = decltype(tl_tag)::value;
  // Invalid pixels start "terminated" (T = 0 <= t_min) and never contribute.
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    P[k].T = make_float2(x0 < W && y0 + k < H ? 1.0f : 0.0f,
                         x0 + 1 < W && y0 + k < H ? 1.0f : 0.0f);
    P[k].Cr = P[k].Cg = P[k].Cb = bc(0.0f);
    P[k].Tl = bc(1.0f);
    P[k].np0 = P[k].np1 = 0u;
  }

  if (n > 0) stage_batch<kBT, kBatch + 1, false, false>(st[0], sorted, submask, rec, rg.x, min(kBatch, n));
  for (int b = 0, it = 0; b < n; b += kBatch, ++it) {
    Stage<kBatch + 1>& cur = st[it & 1];
    cp_async_wait_all();
    const bool live = P[0].T.x > t_min || P[0].T.y > t_min || P[1].T.x > t_min ||
                      P[1].T.y > t_min;
    if (__syncthreads_count(live) == 0) break;  // barrier: batch visible, previous consumed
    if (b + kBatch < n)
      stage_batch<kBT, kBatch + 1, false, false>(st[(it + 1) & 1], sorted, submask, rec, rg.x + b + kBatch,
                       min(kBatch, n - b - kBatch));
    // relevance of the batch for the warp's 8 sub-quarters -> 8 compacted lists.  The tests
    // share their per-axis terms (rounded squares of the distances to the 4 columns and 2
    // rows) and add one pair exactly as dist2_rn would at the sub-quarter's closest pixel
    // centre (bit-identical decisions; a conservative superset of the per-pixel test).
    // a warp whose 128 pixels all terminated skips the tests (it still joins the barriers;
    // its mask bytes stay unwritten, which the backward tolerates: those pixels' walks ended
    // before the batch, so any bits only add entries that contribute exact zeros)
    const uint32_t alive = __ballot_sync(0xffffffffu, live);
    const int cnt = alive ? min(kBatch, n - b) : 0;
    int base[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int wd = 0; wd < kWords; ++wd) {
      if (32 * wd >= cnt) break;  // warp-uniform
      const int j = 32 * wd + lane;
      const bool in = j < cnt;
      // past the batch: the sentinel, never relevant (tracked frames test `in` explicitly)
      const float4 g = cur.geo[in ? j : (kTrack ? 0 : kBatch)];
      float ax4[4], ay2[2];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float d = __fsub_rn(fminf(fmaxf(g.x, cx0[c]), cx1[c]), g.x);
        ax4[c] = __fmul_rn(d, d);
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const float d = __fsub_rn(fminf(fmaxf(g.y, ry0[r]), ry1[r]), g.y);
        ay2[r] = __fmul_rn(d, d);
      }
      uint32_t mw = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {  // group k: quarter 2w + (k >> 2), sub (k & 3)
        const int c = (k >> 2) * 2 + (k & 1), r = (k >> 1) & 1;
        const bool hk = (!kTrack || (in && cv[c] && rv[r])) && !(__fadd_rn(ax4[c], ay2[r]) > g.z);
        mw |= (hk ? 1u : 0u) << k;
        const uint32_t mk = __ballot_sync(0xffffffffu, hk);
        if (hk) s_list[8 * w + k][base[k] + __popc(mk & lt)] = (uint8_t)j;
        base[k] += __popc(mk);
      }
      if (kTrack && !kTl && in) mask_bytes[2 * ((size_t)rg.x + b + j) + w] = (uint8_t)mw;
    }
    // a sub-quarter whose 16 pixels have all terminated walks nothing
    int steps = 0, my_cnt = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int ck = ((alive >> (4 * k)) & 0xFu) ? base[k] : 0;
      steps = max(steps, ck);
      if (k == gq) my_cnt = ck;
    }
    for (int e = my_cnt + l4; e < steps; e += 4) s_list[sub][e] = (uint8_t)kBatch;
    __syncwarp();
    const uint8_t* my_list = s_list[sub];
#pragma unroll kUnroll
    for (int i = 0; i < steps; ++i) {
      const int jj = my_list[i];
      const float4 g = cur.geo[jj], c = cur.col[jj];
      const float2 dx = __fadd2_rn(PX, bc(-g.x));
      const float2 dy = __fadd2_rn(PY, bc(-g.y));
      // r2 rounds exactly like the oracle's dist2_rn: dx^2 as fma(dx, dx, -0) = round(dx^2)
      // (an FMUL2 ptxas does not contract with the following add), dy^2 as a scalar mul.rn
      const float2 ax = __ffma2_rn(dx, dx, bc(-0.0f));
      const uint32_t idx = (uint32_t)(b + jj + 1);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float dyk = k ? dy.y : dy.x;
        const float2 r2 = __fadd2_rn(ax, bc(__fmul_rn(dyk, dyk)));
        fwd_pair<kTrack, kTl, kTerm>(P[k], r2, g, c, t_min, idx);
      }
    }
  }
  };
  walk(std::false_type{});
  // Tracked frames hand the backward each pixel's final transmittance, from which it recovers
  // T before every contributor by division (k_blend_bwd.cu).  A pixel whose final
  // transmittance is not a normal float (an opacity-1 splat at its centre gives T = 0; t_min = 0
  // lets T underflow) cannot be recovered that way: if the tile has one, it is walked again,
  // recording T before the last contributor, stored negated so the backward takes its slower,
  // select-based start for this tile.
  bool rewalk = false;
  if constexpr (kTrack) {
    bool bad = false;
#pragma unroll
    for (int k = 0; k < 2; ++k)
      bad |= (P[k].np0 != 0u && !(P[k].T.x >= kMinNormal)) ||
             (P[k].np1 != 0u && !(P[k].T.y >= kMinNormal));
    rewalk = __syncthreads_or(bad) != 0;
    if (rewalk) walk(std::true_type{});
  }
  cp_async_wait_all();
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int y = y0 + k;
    if (y >= H) continue;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int x = x0 + i;
      if (x >= W) continue;
      const float T = i ? P[k].T.y : P[k].T.x;
      const size_t pix = (size_t)y * W + x;
      out[3 * pix + 0] = (i ? P[k].Cr.y : P[k].Cr.x) + T * fp.bg[0];
      out[3 * pix + 1] = (i ? P[k].Cg.y : P[k].Cg.x) + T * fp.bg[1];
      out[3 * pix + 2] = (i ? P[k].Cb.y : P[k].Cb.x) + T * fp.bg[2];
      if constexpr (kTrack) {
        t_last[pix] = rewalk ? -(i ? P[k].Tl.y : P[k].Tl.x) : T;
        n_proc[pix] = i ? P[k].np1 : P[k].np0;
      }
    }
  }
}

// Measurement hook (bench.py's roofline): the algorithmic work of the last frame, counted the
// way the reference's per-pixel loop sees it -- every pixel walks its tile's list in depth
// order until its transmittance drops to t_min, counting the entries it evaluates and those
// inside their 3-sigma circle.  One thread per pixel, no culling; run outside timed regions.
__global__ void __launch_bounds__(kTilePixels) k_count_pairs(
    FrameParams fp, const uint2* __restrict__ ranges, const uint2* __restrict__ sorted,
    const RenderRec* __restrict__ rec, unsigned long long* __restrict__ out) {
  __shared__ unsigned long long s_ev[kTilePixels / 32], s_in[kTilePixels / 32];
  const int tile = blockIdx.x;
  const int tx = tile % fp.tiles_x, ty = tile / fp.tiles_x;
  const int x = tx * kTile + (threadIdx.x & (kTile - 1)), y = ty * kTile + threadIdx.x / kTile;
  unsigned long long ev = 0, in = 0;
  if (x < fp.cam.width && y < fp.cam.height) {
    const uint2 rg = ranges[tile];
    const uint32_t n = rg.x == kEmptyRange ? 0u : rg.y - rg.x;
    const float px = (float)x + 0.5f, py = (float)y + 0.5f;
    float T = 1.0f;
    for (uint32_t p = 0; p < n; ++p) {
      const RenderRec r = rec[sorted[rg.x + p].x];
      ++ev;
      const float r2 = dist2_rn(__fsub_rn(px, r.geo.x), __fsub_rn(py, r.geo.y));
      if (r2 > r.geo.z) continue;
      ++in;
      const float a = fast_exp2(__fmaf_rn(r2, r.geo.w, r.col.w));  // K6's alpha
      T = T * (1.0f - a);
      if (!(T > fp.t_min)) break;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ev += __shfl_xor_sync(0xffffffffu, ev, o);
    in += __shfl_xor_sync(0xffffffffu, in, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s_ev[threadIdx.x >> 5] = ev;
    s_in[threadIdx.x >> 5] = in;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long e = 0, i = 0;
    for (int w = 0; w < kTilePixels / 32; ++w) {
      e += s_ev[w];
      i += s_in[w];
    }
    atomicAdd(&out[0], e);
    atomicAdd(&out[1], i);
  }
}

void launch_count_pairs(const FrameParams& fp, const uint2* ranges, const uint2* sorted,
                        const RenderRec* rec, unsigned long long* out, cudaStream_t st) {
  k_count_pairs<<<fp.n_tiles, kTilePixels, 0, st>>>(fp, ranges, sorted, rec, out);
}

void launch_blend_fwd(const FrameParams& fp, const uint2* ranges, const uint2* sorted,
                      uint16_t* submask, const RenderRec* rec, unsigned long long* total,
                      int64_t key_cap, float* out, float* t_last, uint32_t* n_proc, bool track,
                      cudaStream_t st) {
  // a tracked frame needs the termination test (the last contributor it records); an untracked
  // one only when t_min > 0
  auto k = track ? k_blend_fwd<true, true>
                 : (fp.t_min > 0.0f ? k_blend_fwd<false, true> : k_blend_fwd<false, false>);
  launch_pdl(k, dim3(fp.n_tiles), dim3(kBT), 0, st,
             fp, ranges, sorted, submask, rec, total, key_cap, out, t_last, n_proc);
}

}  // namespace isg

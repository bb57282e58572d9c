// K6 — per-16x16-tile front-to-back alpha blending (forward).
//
// Replaces composite_pixels (/root/reference/proj/src/splat3d.cpp:125-162) and the inclusion
// test covers(ScreenIso) (:108-114).  Instead of every pixel visiting every splat
// (O(W*H*N)), one CTA owns one tile and walks only that tile's depth-ordered list.
//
// Mapping: 128 threads per tile; warp w owns the 8x8 quarter-tile w, each 8-lane group one 4x4
// sub-quarter and each lane a vertical pixel pair, so one shared-memory record feeds two pixels
// that share dx.  Records are staged 128 at a time into shared memory with cp.async,
// double-buffered (the next batch's copy is in flight while the current one is blended).
// After each batch barrier every warp tests the staged splats' 3-sigma circles against its
// quarter and then its four sub-quarters (conservative closest-point tests, exact rounding),
// ballots, and compacts the relevant entry indices into four lists; the groups walk their own
// lists in lockstep.  The 4x4 culling cuts the pixel-entry slots a circle does not cover
// (a circle of the typical 6-px 3-sigma radius covers a 4x4 region far better than an 8x8).
// Compositing is branch-free; the CTA stops once every pixel has transmittance <= t_min.
//
// The 3-sigma test is bit-identical to the FP32 oracle (explicit _rn arithmetic); exp uses
// ex2.approx on a per-splat precomputed -log2(e)/sigma2d^2.
#include "blend_common.cuh"

namespace isg {

namespace {
using namespace blend;

constexpr int kBT = 128;     // threads per tile CTA (4 warps x 32 pixel pairs)
constexpr int kBatch = 128;  // records staged per batch (one per thread)
constexpr int kListPitch = kBatch + 4;  // sub-quarter lists start in different banks

// Pixel-centre rectangle of a region, clipped to the image.
struct Region {
  float x0, x1, y0, y1;
  bool valid;
};

// 4x4 sub-quarter s (0..3) of quarter-tile w, pixel-centre rectangle clipped to the image.
__device__ __forceinline__ Region sub_rect(const FrameParams& fp, int tile, int w, int s) {
  Region g;
  const int tx = tile % fp.tiles_x, ty = tile / fp.tiles_x;
  const int W = fp.cam.width, H = fp.cam.height;
  const int x0 = tx * kTile + (w & 1) * 8 + (s & 1) * 4, y0 = ty * kTile + (w >> 1) * 8 + (s >> 1) * 4;
  g.valid = x0 < W && y0 < H;
  g.x0 = (float)x0 + 0.5f;
  g.x1 = (float)(min(x0 + 4, W) - 1) + 0.5f;
  g.y0 = (float)y0 + 0.5f;
  g.y1 = (float)(min(y0 + 4, H) - 1) + 0.5f;
  return g;
}

// Compact the batch's entries relevant to each of the warp's four 4x4 sub-quarters into
// list[s] (ascending); count[s] receives the lengths.  The four closest-point tests share their
// per-axis terms: the rounded squares of the x distances to the left / right sub-quarter
// columns and of the y distances to the top / bottom rows are computed once, and each test
// adds one pair exactly as dist2_rn (isg_math.cuh) would at the sub-quarter's closest pixel
// centre (bit-identical decisions; a conservative superset of the per-pixel 3-sigma test).
__device__ __forceinline__ void warp_relevant_lists(const Stage<kBatch>& st, const Region rs[4],
                                                    int cnt, uint8_t (*list)[kListPitch],
                                                    int count[4]) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  int base[4] = {0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < kBatch / 32; ++k) {
    const int j = 32 * k + lane;
    bool h[4] = {false, false, false, false};
    if (j < cnt) {
      const float4 g = st.geo[j];
      float ax[2], ay[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const float dx = __fsub_rn(fminf(fmaxf(g.x, rs[i].x0), rs[i].x1), g.x);
        const float dy = __fsub_rn(fminf(fmaxf(g.y, rs[2 * i].y0), rs[2 * i].y1), g.y);
        ax[i] = __fmul_rn(dx, dx);
        ay[i] = __fmul_rn(dy, dy);
      }
#pragma unroll
      for (int s = 0; s < 4; ++s) h[s] = rs[s].valid && !(__fadd_rn(ax[s & 1], ay[s >> 1]) > g.z);
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const uint32_t m = __ballot_sync(0xffffffffu, h[s]);
      if (h[s]) list[s][base[s] + __popc(m & lt)] = (uint8_t)j;
      base[s] += __popc(m);
    }
  }
  __syncwarp();
#pragma unroll
  for (int s = 0; s < 4; ++s) count[s] = base[s];
}

}  // namespace

__global__ void __launch_bounds__(kBT) k_blend_fwd(
    FrameParams fp, const uint2* __restrict__ ranges, const uint2* __restrict__ sorted,
    const RenderRec* __restrict__ rec, const unsigned long long* __restrict__ total,
    int64_t key_cap, float* __restrict__ out, float* __restrict__ t_last,
    uint32_t* __restrict__ n_proc) {
  __shared__ Stage<kBatch> st[2];
  __shared__ uint8_t s_list[kBT / 32][4][kListPitch];
  if (overflowed(total, key_cap)) return;
  const int tile = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int sq = lane >> 3, l8 = lane & 7;  // 8-lane group = 4x4 sub-quarter, lane = pixel pair
  Region sub[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) sub[s] = sub_rect(fp, tile, w, s);
  const int tx = tile % fp.tiles_x, ty = tile / fp.tiles_x;
  const int px_i = tx * kTile + (w & 1) * 8 + (sq & 1) * 4 + (l8 & 3);
  const int py_i = ty * kTile + (w >> 1) * 8 + (sq >> 1) * 4 + 2 * (l8 >> 2);  // (px, py+{0,1})
  const int W = fp.cam.width, H = fp.cam.height;
  const bool valid0 = px_i < W && py_i < H, valid1 = px_i < W && py_i + 1 < H;
  const float px = (float)px_i + 0.5f, py0 = (float)py_i + 0.5f, py1 = py0 + 1.0f;
  const uint2 rg = ranges[tile];
  const int n = (int)(rg.y - rg.x);
  const float t_min = fp.t_min;

  // The pixel pair is processed as packed f32x2 (FFMA2/FMUL2/FADD2: one issue slot for both
  // pixels); .x = pixel (px, py), .y = pixel (px, py + 1).  Every packed op rounds per lane
  // exactly like its scalar counterpart, so the 3-sigma test stays bit-identical to the oracle.
  // Invalid pixels start "terminated" (T = 0 <= t_min) and never contribute.
  const float2 PY = make_float2(py0, py1);
  float2 T = make_float2(valid0 ? 1.0f : 0.0f, valid1 ? 1.0f : 0.0f);
  float Tl0 = 1.0f, Tl1 = 1.0f;
  float2 Cr = make_float2(0.f, 0.f), Cg = Cr, Cb = Cr;
  uint32_t np0 = 0, np1 = 0;
  const float2 kOne = make_float2(1.0f, 1.0f);

  if (n > 0) stage_batch(st[0], sorted, rec, rg.x, min(kBatch, n));
  for (int b = 0, it = 0; b < n; b += kBatch, ++it) {
    Stage<kBatch>& cur = st[it & 1];
    cp_async_wait_all();
    const bool tdone = !(T.x > t_min) && !(T.y > t_min);
    if (__syncthreads_count(tdone) == kBT) break;  // barrier: batch visible, previous consumed
    if (b + kBatch < n)
      stage_batch(st[(it + 1) & 1], sorted, rec, rg.x + b + kBatch, min(kBatch, n - b - kBatch));
    int cnt[4];
    warp_relevant_lists(cur, sub, min(kBatch, n - b), s_list[w], cnt);
    // a sub-quarter whose 16 pixels have all terminated walks nothing
    const uint32_t alive = __ballot_sync(0xffffffffu, T.x > t_min || T.y > t_min);
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4)
      if (((alive >> (8 * q4)) & 0xFFu) == 0u) cnt[q4] = 0;
    const int steps = max(max(cnt[0], cnt[1]), max(cnt[2], cnt[3]));
    const int my_cnt = sq == 0 ? cnt[0] : (sq == 1 ? cnt[1] : (sq == 2 ? cnt[2] : cnt[3]));
    // the four 8-lane groups walk their own sub-quarter lists in lockstep
    const uint8_t* my_list = s_list[w][sq];
    for (int i = 0; i < steps; ++i) {
      const bool has = i < my_cnt;
      const int jj = has ? my_list[i] : 0;
      const float4 g = cur.geo[jj], c = cur.col[jj];
      const float dx = __fsub_rn(px, g.x);
      const float ax = __fmul_rn(dx, dx);
      const float2 dy = __fadd2_rn(PY, make_float2(-g.y, -g.y));
      // scalar: ptxas would contract a packed mul.rn + add.rn into FFMA2 (one rounding), and
      // the 3-sigma test must round exactly like the oracle's (and K1's) dist2_rn
      const float2 r2 = make_float2(__fadd_rn(ax, __fmul_rn(dy.x, dy.x)),
                                    __fadd_rn(ax, __fmul_rn(dy.y, dy.y)));
      const bool in0 = has && !(r2.x > g.z) && (T.x > t_min);
      const bool in1 = has && !(r2.y > g.z) && (T.y > t_min);
      const uint32_t idx = (uint32_t)(b + jj + 1);
      const float2 q = __fmul2_rn(r2, make_float2(g.w, g.w));
      const float2 e = __fmul2_rn(make_float2(c.w, c.w), make_float2(fast_exp2(q.x), fast_exp2(q.y)));
      const float2 a = make_float2(in0 ? e.x : 0.0f, in1 ? e.y : 0.0f);
      const float2 wgt = __fmul2_rn(T, a);
      Cr = __ffma2_rn(wgt, make_float2(c.x, c.x), Cr);
      Cg = __ffma2_rn(wgt, make_float2(c.y, c.y), Cg);
      Cb = __ffma2_rn(wgt, make_float2(c.z, c.z), Cb);
      Tl0 = in0 ? T.x : Tl0;
      Tl1 = in1 ? T.y : Tl1;
      np0 = in0 ? idx : np0;
      np1 = in1 ? idx : np1;
      T = __fmul2_rn(T, __fadd2_rn(kOne, make_float2(-a.x, -a.y)));  // T (1 - a)
    }
  }
  const float T0 = T.x, T1 = T.y;
  const float C0r = Cr.x, C0g = Cg.x, C0b = Cb.x, C1r = Cr.y, C1g = Cg.y, C1b = Cb.y;
  cp_async_wait_all();
  if (valid0) {
    const size_t pix = (size_t)py_i * W + px_i;
    out[3 * pix + 0] = C0r + T0 * fp.bg[0];
    out[3 * pix + 1] = C0g + T0 * fp.bg[1];
    out[3 * pix + 2] = C0b + T0 * fp.bg[2];
    t_last[pix] = Tl0;
    n_proc[pix] = np0;
  }
  if (valid1) {
    const size_t pix = (size_t)(py_i + 1) * W + px_i;
    out[3 * pix + 0] = C1r + T1 * fp.bg[0];
    out[3 * pix + 1] = C1g + T1 * fp.bg[1];
    out[3 * pix + 2] = C1b + T1 * fp.bg[2];
    t_last[pix] = Tl1;
    n_proc[pix] = np1;
  }
}

void launch_blend_fwd(const FrameParams& fp, const uint2* ranges, const uint2* sorted,
                      const RenderRec* rec, const unsigned long long* total, int64_t key_cap,
                      float* out, float* t_last, uint32_t* n_proc, cudaStream_t st) {
  k_blend_fwd<<<fp.n_tiles, kBT, 0, st>>>(fp, ranges, sorted, rec, total, key_cap, out, t_last,
                                          n_proc);
}

}  // namespace isg

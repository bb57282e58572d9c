// K6 — per-16x16-tile front-to-back alpha blending (forward).
//
// Replaces composite_pixels (/root/reference/proj/src/splat3d.cpp:125-162) and the inclusion
// test covers(ScreenIso) (:108-114).  Instead of every pixel visiting every splat
// (O(W*H*N)), one CTA owns one tile and walks only that tile's depth-ordered list.
//
// Mapping: 128 threads per tile; warp w owns the 8x8 quarter-tile w and each lane a vertical
// pixel pair, so one shared-memory record feeds two pixels that share dx.  Records are
// staged 128 at a time into shared memory with cp.async, double-buffered (the next batch's
// copy is in flight while the current one is blended).  After each batch barrier every warp
// tests the staged splats' 3-sigma circles against its quarter (conservative closest-point
// test, exact rounding), ballots, and compacts the relevant entry indices into a per-warp list
// — culling costs a few instructions per batch and irrelevant entries cost no issue slots.
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

// Compact the warp's relevant entries of the batch into `list` (ascending); returns the count.
__device__ __forceinline__ int warp_relevant_list(const Stage<kBatch>& st, const Region& rg,
                                                  int cnt, uint8_t* list) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  int base = 0;
#pragma unroll
  for (int k = 0; k < kBatch / 32; ++k) {
    const int j = 32 * k + lane;
    bool hit = false;
    if (j < cnt && rg.valid) {
      const float4 g = st.geo[j];
      hit = rect_hit(rg, g.x, g.y, g.z);
    }
    const uint32_t m = __ballot_sync(0xffffffffu, hit);
    if (hit) list[base + __popc(m & lt)] = (uint8_t)j;
    base += __popc(m);
  }
  __syncwarp();
  return base;
}

}  // namespace

__global__ void __launch_bounds__(kBT) k_blend_fwd(
    FrameParams fp, const uint2* __restrict__ ranges, const uint2* __restrict__ sorted,
    const RenderRec* __restrict__ rec, const unsigned long long* __restrict__ total,
    int64_t key_cap, float* __restrict__ out, float* __restrict__ t_last,
    uint32_t* __restrict__ n_proc) {
  __shared__ Stage<kBatch> st[2];
  __shared__ uint8_t s_list[kBT / 32][kBatch];
  if (overflowed(total, key_cap)) return;
  const int tile = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const Region reg = region_rect(fp, tile, w);
  const int tx = tile % fp.tiles_x, ty = tile / fp.tiles_x;
  const int px_i = tx * kTile + (w & 1) * 8 + (lane & 7);
  const int py_i = ty * kTile + (w >> 1) * 8 + 2 * (lane >> 3);  // pixels (px_i, py_i + {0,1})
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
  const float2 kOne = make_float2(1.0f, 1.0f), kMinusOne = make_float2(-1.0f, -1.0f);

  if (n > 0) stage_batch(st[0], sorted, rec, rg.x, min(kBatch, n));
  for (int b = 0, it = 0; b < n; b += kBatch, ++it) {
    Stage<kBatch>& cur = st[it & 1];
    cp_async_wait_all();
    const bool tdone = !(T.x > t_min) && !(T.y > t_min);
    if (__syncthreads_count(tdone) == kBT) break;  // barrier: batch visible, previous consumed
    if (b + kBatch < n)
      stage_batch(st[(it + 1) & 1], sorted, rec, rg.x + b + kBatch, min(kBatch, n - b - kBatch));
    const int nrel = warp_relevant_list(cur, reg, min(kBatch, n - b), s_list[w]);
    for (int i = 0; i < nrel; ++i) {
      const int jj = s_list[w][i];
      const float4 g = cur.geo[jj];
      const float4 c = cur.col[jj];
      const float dx = __fsub_rn(px, g.x);
      const float ax = __fmul_rn(dx, dx);
      const float2 dy = __fadd2_rn(PY, make_float2(-g.y, -g.y));
      // scalar: ptxas would contract a packed mul.rn + add.rn into FFMA2 (one rounding), and
      // the 3-sigma test must round exactly like the oracle's (and K1's) dist2_rn
      const float2 r2 = make_float2(__fadd_rn(ax, __fmul_rn(dy.x, dy.x)),
                                    __fadd_rn(ax, __fmul_rn(dy.y, dy.y)));
      const bool in0 = !(r2.x > g.z) && (T.x > t_min);
      const bool in1 = !(r2.y > g.z) && (T.y > t_min);
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
      T = __fmul2_rn(T, __ffma2_rn(a, kMinusOne, kOne));  // T (1 - a)
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

// K7 — per-16x16-tile backward of the alpha blend, with the L2 loss gradient fused in.
//
// The backward the reference does not have (its 2D analogue is loss_gradients,
// /root/reference/proj/src/loss.cpp:259-300).  Per pixel it walks the tile's depth-ordered
// list in reverse from the last contributor (n_proc - 1), recovering the transmittance
// T_k = T_{k+1} / (1 - a_k) from the pixel's final transmittance (a tile where that is not a
// normal float — alpha = 1 or underflow — gets T before the last contributor instead, see
// k_blend.cu, and does not divide for it), and accumulating with A = colour behind (SURVEY
// Appendix A):
//     dL/da_k = T_k G.(c_k - A_k),  dL/dc_k = G T_k a_k,  A <- a c + (1 - a) A
// with G = dL/dC = 2 w (C - target) / (3 W H) (mse, src/image.cpp:50-58) computed in the
// prologue — or, for the L1 + D-SSIM loss, read from the dL/dC image k_ssim.cu wrote — and the
// kernel closed forms of include/isosplat/kernels.hpp:208-222.
//
// Mapping: 64 threads per tile.  Each four-lane group owns one 4x4 sub-quarter and each lane a
// 2x2 pixel quad (two packed f32x2 pixel pairs).  Per staged batch (128 records in direct
// mode, 32 in slot mode) every warp turns the entries' sub-quarter masks (written by the
// forward) into 8 relevance lists by ballots; the 8 groups then walk their OWN lists in
// lockstep in reverse — eight different splats per warp step — so culling is at 4x4
// granularity (a typical 6-px 3-sigma circle covers a 4x4 region far better than an 8x8 one)
// and the per-entry reduction runs over only 4 lanes.  The 7 gradients of a pair are summed
// over the lane's 4 pixels and reduce-scattered over the group in 6 shuffles.  Direct mode
// (default): each lane adds its 2 values to the splat's 2D sums with one L2 reduction
// (red.global.add.v2.f32; the 4 lanes cover one 32-B sector).  Slot mode (deterministic): the
// 16 sub-quarters are combined in shared memory in a fixed order and written — no atomics —
// to the pair's gradient slot; K8 sums each splat's slots in a fixed order, so gradients are
// bitwise deterministic.
#include "blend_common.cuh"

namespace isg {

namespace {
using namespace blend;

constexpr int kBT = 64;      // threads per tile CTA: 2 warps x 8 four-lane groups
#ifndef ISG_BWD_BATCH
#define ISG_BWD_BATCH 160
#endif
// 4 walk steps per loop iteration (0.578 vs 0.595 ms unrolled by 1 at C3, direct mode)
#ifndef ISG_BWD_UNROLL
#define ISG_BWD_UNROLL 4
#endif
#ifndef ISG_LIST_PTX
#define ISG_LIST_PTX 1
#endif
constexpr int kUnroll = ISG_BWD_UNROLL;  // walk steps per loop iteration
// Records staged per batch.  The 8 groups of a warp walk a batch in lockstep, so a warp's step
// count per batch is the longest of its 8 relevance lists: larger batches pad less (C3 walk
// steps, tools/sim_bwd_lists.py / sim_bwd_trim.py: 3.36M at 32, 3.20M at 64, 3.08M at 128,
// 3.03M at 192), until the staging's shared memory costs resident CTAs: 0.485 ms at 128,
// 0.475 at 160, 0.488 at 192 (11 CTAs / SM), 0.491 at 224 (96 registers).  Slot mode keeps 32
// (its flush maps entry = lane).
constexpr int kBatchDirect = ISG_BWD_BATCH;
constexpr int kBatchSlot = 32;
static_assert(kBatchDirect % 32 == 0 && kBatchDirect < 256, "u8 list entries, sentinel index");
constexpr int kSubs = 16;    // 4x4 sub-quarters per tile (one per four-lane group)

// Two horizontally adjacent pixels (same row) as packed f32x2 lanes: .x = (x0, y), .y = (x0+1, y).
// Packed FFMA2/FMUL2/FADD2 issue once for both pixels.
struct BwdPair {
  float2 G0, G1, G2;  // dL/dC
  float2 T;           // transmittance before the most recently processed (later) entry
  float2 GA;          // G . A, A = colour behind (normalised): only its projection on G is used
  int np0, np1;       // list entries the forward processed for each pixel
};

__device__ __forceinline__ float2 bc(float v) { return make_float2(v, v); }

// acc: [2] sum go*r2, [4..6] drgb, summed per lane of the pair; go = dL/dalpha * alpha is
// returned per pixel (the caller forms [0] sum go*dx, [1] sum go*dy and [3] sum go = o dL/do
// from the quad's row and column sums).  alpha = ex2(r2 g.w + log2 o) exactly as the forward
// formed it (c.w = log2 o, K1).
//   dL/da_k = T_k G.(c_k - A_k);  A <- a c + (1 - a) A  =>  G.A <- G.A + a (G.c - G.A)
// so the colour behind is carried as the single scalar G.A per pixel.  An inactive pixel gets
// e = 0, hence a = 0: T and G.A stay exactly unchanged and every contribution is an exact zero.
// kFast: p.T starts as the pixel's final transmittance and every contributor divides it back
// up, T_k = T_{k+1} / (1 - a_k).  Otherwise (a tile the forward re-walked, k_blend.cu) p.T
// starts as the transmittance before the last contributor, which therefore does not divide.
template <bool kFast>
__device__ __forceinline__ void bwd_pair(BwdPair& p, bool act0, bool act1, int j, float2 r2,
                                         const float4 g, const float4 c, float2 acc[8],
                                         float2& go) {
  const float2 q = __ffma2_rn(r2, bc(g.w), bc(c.w));
  const float2 a = make_float2(act0 ? fast_exp2(q.x) : 0.0f, act1 ? fast_exp2(q.y) : 0.0f);
  const float2 om = __fadd2_rn(bc(1.0f), make_float2(-a.x, -a.y));  // 1 - a (FADD2 imm)
  const float2 Tr = __fmul2_rn(p.T, make_float2(fast_rcp(om.x), fast_rcp(om.y)));
  float2 Tk = Tr;
  if constexpr (!kFast)
    Tk = make_float2(j == p.np0 - 1 ? p.T.x : Tr.x, j == p.np1 - 1 ? p.T.y : Tr.y);
  p.T = Tk;
  const float2 Gc = __ffma2_rn(p.G2, bc(c.z), __ffma2_rn(p.G1, bc(c.y), __fmul2_rn(p.G0, bc(c.x))));
  const float2 gd = __fadd2_rn(Gc, make_float2(-p.GA.x, -p.GA.y));  // G.(c - A)
  p.GA = __ffma2_rn(a, gd, p.GA);
  const float2 dLda = __fmul2_rn(Tk, gd);
  const float2 Ta = __fmul2_rn(Tk, a);
  acc[4] = __ffma2_rn(p.G0, Ta, acc[4]);
  acc[5] = __ffma2_rn(p.G1, Ta, acc[5]);
  acc[6] = __ffma2_rn(p.G2, Ta, acc[6]);
  go = __fmul2_rn(dLda, a);  // the caller sums the two rows' go into acc[3]
  acc[2] = __ffma2_rn(go, r2, acc[2]);
}

// reduce-scatter of 8 values (v[7] == 0) over a 4-lane group in 6 shuffles: lane l (l4 = l & 3)
// returns the group sums of values 4*(l4>>1) + 2*(l4&1) + {0, 1} in out[0], out[1].
__device__ __forceinline__ void reduce_scatter8_quad(const float v[8], float out[2]) {
  const int lane = threadIdx.x & 31;
  const bool b1 = lane & 2, b0 = lane & 1;
  float w[4];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float send = b1 ? v[i] : v[i + 4];
    const float keep = b1 ? v[i + 4] : v[i];
    w[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  {  // value 7 is zero: the upper lanes' share of this pair is 0, the lower lanes add v[3]
    const float t = __shfl_xor_sync(0xffffffffu, v[3], 2);
    w[3] = b1 ? 0.0f : v[3] + t;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = b0 ? w[i] : w[i + 2];
    const float keep = b0 ? w[i + 2] : w[i];
    out[i] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
  }
}

}  // namespace

#ifndef ISG_BWD_MINB
#define ISG_BWD_MINB 0
#endif
#if ISG_BWD_MINB > 0
#define ISG_BWD_BOUNDS __launch_bounds__(kBT, ISG_BWD_MINB)
#else
#define ISG_BWD_BOUNDS __launch_bounds__(kBT)
#endif
template <bool kGivenG, bool kDirect>
// (a minimum-blocks bound that caps registers for more resident warps — 10, 12, 14 or 16 CTAs
// per SM — measured 12-27% slower: ptxas then trades ILP for registers)
__global__ void ISG_BWD_BOUNDS k_blend_bwd(
    FrameParams fp, const uint2* __restrict__ ranges, const uint2* __restrict__ sorted,
    const uint16_t* __restrict__ submask,
    const RenderRec* __restrict__ rec, const unsigned long long* __restrict__ total,
    int64_t key_cap, const float* __restrict__ img, const float* __restrict__ target,
    const float* __restrict__ t_last, const uint32_t* __restrict__ n_proc, float loss_scale,
    float4* __restrict__ partial, double* __restrict__ tile_loss, float* __restrict__ grad2d) {
  constexpr int kB = kDirect ? kBatchDirect : kBatchSlot;
  constexpr int kW = kB / 32;
  constexpr int kListPitch = kB + 4;  // sub-quarter lists start in different banks
  // entry kB of each stage is a sentinel no pixel is inside (r2max = -1): the groups'
  // lists are padded with it to the warp's step count, so the walk needs no bounds test
  __shared__ Stage<kB + 1> st[2];
  // [sub-quarter][value][entry]; rows padded so one entry's 8 values hit 8 different banks
  // (slot mode only: the direct mode reduces into grad2d in L2 instead)
  // (direct mode: one-element placeholders, no shared memory spent)
  __shared__ float s_part[kDirect ? 1 : kSubs][kDirect ? 1 : 8][kDirect ? 1 : kB + 1];
  __shared__ uint32_t s_rel[kDirect ? 1 : kSubs][kDirect ? 1 : kW];  // relevance ballots
  __shared__ uint8_t s_list[kSubs][kListPitch];
  __shared__ float s_red[2];
  __shared__ int s_max[2];
  __shared__ __align__(16) int s_sqmax[kSubs];  // per sub-quarter: max entries processed over its 16 pixels
  const int tile = blockIdx.x;
  pdl_enter();
  if (overflowed(total, key_cap)) {
    if (threadIdx.x == 0) tile_loss[tile] = 0.0;
    return;
  }
  if (threadIdx.x < 2) {
    st[threadIdx.x].geo[kB] = make_float4(0.0f, 0.0f, -1.0f, 0.0f);
    st[threadIdx.x].col[kB] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gq = lane >> 2, l4 = lane & 3;  // four-lane group = one 4x4 sub-quarter
  const int sub = 8 * w + gq;               // q = sub >> 2 (quarter), sub & 3 within it
  const int q = sub >> 2, sq = sub & 3;
  const int tx = tile % fp.tiles_x, ty = tile / fp.tiles_x;
  const int W = fp.cam.width, H = fp.cam.height;
  const int x0 = tx * kTile + (q & 1) * 8 + (sq & 1) * 4 + 2 * (l4 & 1);
  const int y0 = ty * kTile + (q >> 1) * 8 + (sq >> 1) * 4 + 2 * (l4 >> 1);
  const float2 PX = make_float2((float)x0 + 0.5f, (float)x0 + 1.5f);
  const float2 PY = make_float2((float)y0 + 0.5f, (float)y0 + 1.5f);
  const uint2 rg = ranges[tile];
  const int n = rg.x == kEmptyRange ? 0 : (int)(rg.y - rg.x);

  BwdPair P[2];  // P[k]: the quad's row k
  float dsq = 0.0f;
  bool slow_px = false;
  int npmax = 0;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    float G[2][3] = {}, T[2] = {0.f, 0.f};
    int np[2] = {0, 0};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int x = x0 + i, y = y0 + k;
      if (x < W && y < H) {
        const size_t pix = (size_t)y * W + x;
        if (kGivenG) {  // `target` holds dL/dC (e.g. L1 + D-SSIM, k_ssim.cu)
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) G[i][ch] = target[3 * pix + ch] * loss_scale;
        } else {
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const float d = img[3 * pix + ch] - target[3 * pix + ch];
            dsq += d * d;
            G[i][ch] = 2.0f * d * loss_scale;
          }
        }
        const float tl = t_last[pix];  // negative: the tile's select-based start (k_blend.cu)
        slow_px |= tl < 0.0f;
        T[i] = fabsf(tl);
        np[i] = (int)n_proc[pix];
        npmax = max(npmax, np[i]);
      }
    }
    BwdPair& s = P[k];
    s.G0 = make_float2(G[0][0], G[1][0]);
    s.G1 = make_float2(G[0][1], G[1][1]);
    s.G2 = make_float2(G[0][2], G[1][2]);
    s.T = make_float2(T[0], T[1]);
    s.np0 = np[0];
    s.np1 = np[1];
    s.GA = make_float2(G[0][0] * fp.bg[0] + G[0][1] * fp.bg[1] + G[0][2] * fp.bg[2],
                       G[1][0] * fp.bg[0] + G[1][1] * fp.bg[1] + G[1][2] * fp.bg[2]);
  }
  // the sub-quarter's own last entry: entries at or past it are exact zeros for all of its
  // pixels, so its lists stop there (dense scenes terminate sub-quarters at very different
  // depths within one tile)
  npmax = max(npmax, __shfl_xor_sync(0xffffffffu, npmax, 1));
  npmax = max(npmax, __shfl_xor_sync(0xffffffffu, npmax, 2));
  if (l4 == 0) s_sqmax[sub] = npmax;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dsq += __shfl_xor_sync(0xffffffffu, dsq, o);
    if (o >= 4) npmax = max(npmax, __shfl_xor_sync(0xffffffffu, npmax, o));
  }
  if (lane == 0) {
    s_red[w] = dsq;
    s_max[w] = npmax;
  }
  const bool slow = __syncthreads_or(slow_px) != 0;
  const int m = max(s_max[0], s_max[1]);  // entries [0, m) are walked
  if (threadIdx.x == 0) tile_loss[tile] = (double)s_red[0] + (double)s_red[1];
  // entries never reached by any pixel get zero gradient slots (slot mode)
  for (int j = m + (int)threadIdx.x; !kDirect && j < n; j += kBT) {
    const uint32_t e = sorted[rg.x + j].y;
    partial[2 * (size_t)e] = make_float4(0.f, 0.f, 0.f, 0.f);
    partial[2 * (size_t)e + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (m == 0) return;

  const uint32_t gt = ~((2u << lane) - 1u);  // lanes above this one
  int hi = m;
  stage_batch<kBT, kB + 1, kDirect>(st[0], sorted, submask, rec, rg.x + max(0, hi - kB),
                                        min(kB, hi));
  for (int it = 0; hi > 0; ++it) {
    const int lo = max(0, hi - kB);
    const int cnt = hi - lo;
    Stage<kB + 1>& cur = st[it & 1];
    cp_async_wait_all();
    __syncthreads();  // batch visible; previous batch's flush finished reading s_part
    if (lo > 0) {
      const int nlo = max(0, lo - kB);
      stage_batch<kBT, kB + 1, kDirect>(st[(it + 1) & 1], sorted, submask, rec, rg.x + nlo,
                                            lo - nlo);
    }
    // relevance of the batch for the warp's 8 sub-quarters -> 8 compacted lists, from the
    // pairs' precomputed sub-quarter masks (sub_mask16, the binning's closest-point tests)
    int my_cnt = 0, steps = 0;
    int base[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // (re-read per batch: two broadcast loads, no registers held across the walk)
    const int4 sq0 = reinterpret_cast<const int4*>(s_sqmax)[2 * w];
    const int4 sq1 = reinterpret_cast<const int4*>(s_sqmax)[2 * w + 1];
    const int sqm[8] = {sq0.x, sq0.y, sq0.z, sq0.w, sq1.x, sq1.y, sq1.z, sq1.w};
    // words from the last to the first and, within a word, lanes from high to low: the lists
    // come out in reverse depth order
#pragma unroll
    for (int wd = kW - 1; wd >= 0; --wd) {
      if (32 * wd >= cnt) continue;  // warp-uniform: the batch's partial end
      const int j = 32 * wd + lane;
      const uint32_t mw = j < cnt ? ((uint32_t)cur.mask[j] >> (8 * w)) & 0xFFu : 0u;
#pragma unroll
      for (int k = 0; k < 8; ++k) {  // group k = sub-quarter 8 w + k
#if ISG_LIST_PTX
        // the mask bit as a predicate (ptxas sets them together with R2P) and-ed into the
        // trim compare, then the ballot: three instructions where the C++ form takes five
        uint32_t mk, hku;
        asm("{\n\t.reg .pred p, q;\n\t.reg .b32 t;\n\t"
            "and.b32 t, %2, %3;\n\t"
            "setp.ne.u32 p, t, 0;\n\t"
            "setp.lt.and.s32 q, %4, %5, p;\n\t"
            "vote.sync.ballot.b32 %0, q, 0xffffffff;\n\t"
            "selp.u32 %1, 1, 0, q;\n\t}"
            : "=r"(mk), "=r"(hku)
            : "r"(mw), "r"(1u << k), "r"(lo + j), "r"(sqm[k]));
        const bool hk = hku != 0u;
#else
        const bool hk = ((mw >> k) & 1u) && lo + j < sqm[k];
        const uint32_t mk = __ballot_sync(0xffffffffu, hk);
#endif
        if (hk) s_list[8 * w + k][base[k] + __popc(mk & gt)] = (uint8_t)j;
        if (!kDirect && lane == 0) s_rel[8 * w + k][wd] = mk;
        base[k] += __popc(mk);
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      steps = max(steps, base[k]);
      if (k == gq) my_cnt = base[k];
    }
    for (int e = my_cnt + l4; e < steps; e += 4) s_list[sub][e] = (uint8_t)kB;
    __syncwarp();
    const uint8_t* my_list = s_list[sub];
    // kNp: some pixel of the warp has its last entry inside this batch, so each pixel tests
    // j < n_proc; below every pixel's last entry (most batches) the test is dropped
    auto walk = [&](auto fast_tag, auto np_tag) {
    constexpr bool kFast = decltype(fast_tag)::value;
    constexpr bool kNp = decltype(np_tag)::value;
#pragma unroll kUnroll
    for (int s = 0; s < steps; ++s) {
      // reverse depth order; the sentinel has a = 0 for every pixel, so T (T / 1) and G.A stay
      // exactly unchanged whatever j is, and its s_part column kB is padding
      const int jj = my_list[s];
      const int j = lo + jj;
      const float4 g = cur.geo[jj];
      const float4 c = cur.col[jj];
      const float2 dx = __fadd2_rn(PX, bc(-g.x));
      const float2 dy = __fadd2_rn(PY, bc(-g.y));
      // r2 keeps the oracle's rounding: dx^2 as fma(dx, dx, -0) = round(dx^2), which ptxas
      // emits as an FMUL2 it does not contract with the following add (a packed mul.rn +
      // add.rn pair it would contract into one FFMA2)
      const float2 ax = __ffma2_rn(dx, dx, bc(-0.0f));
      float2 acc2[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) acc2[k] = bc(0.0f);
      float2 go[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float dyk = k ? dy.y : dy.x;
        const float ay = __fmul_rn(dyk, dyk);
        const float2 r2 = __fadd2_rn(ax, bc(ay));
        const bool act0 = (!kNp || j < P[k].np0) && !(r2.x > g.z);
        const bool act1 = (!kNp || j < P[k].np1) && !(r2.y > g.z);
        bwd_pair<kFast>(P[k], act0, act1, j, r2, g, c, acc2, go[k]);
      }
      acc2[3] = __fadd2_rn(go[0], go[1]);
      // sum go dx and sum go dy over the 2x2 quad from its row and column sums: the right
      // column's dx and the bottom row's dy are the top-left pixel's + 1, so
      //   sum go dx = dx00 sum go + sum_right go,  sum go dy = dy00 sum go + sum_bottom go
      const float s_go = acc2[3].x + acc2[3].y;
      float acc[8];
#pragma unroll
      for (int k = 2; k < 8; ++k) acc[k] = k == 3 ? s_go : acc2[k].x + acc2[k].y;
      acc[0] = __fmaf_rn(dx.x, s_go, go[0].y + go[1].y);
      acc[1] = __fmaf_rn(dy.x, s_go, go[1].x + go[1].y);
      float y[2];
      reduce_scatter8_quad(acc, y);
      // the lane holds values vb, vb + 1 (vb = 4 (l4 >> 1) + 2 (l4 & 1)); the per-splat
      // scale factors are applied once per entry in the flush (slot mode) or per splat by K8
      const int vb = 4 * (l4 >> 1) + 2 * (l4 & 1);
      if constexpr (kDirect) {
        // the sub-quarter's pre-reduced share goes straight to the splat's 2D gradient in L2
        // (4 lanes = one 32-B sector); the sentinel sends nothing
// (skipping exact-zero shares saves L2 reductions but costs three instructions per step:
// 0.4559 vs 0.4516 ms without the test)
#ifndef ISG_RED_SKIP_ZERO
#define ISG_RED_SKIP_ZERO 0
#endif
        red_add_v2_if(jj < kB && (!ISG_RED_SKIP_ZERO || y[0] != 0.0f || y[1] != 0.0f),
                      grad2d + 8 * (size_t)cur.slot[jj] + vb, y[0], y[1]);
      } else {
        s_part[sub][vb][jj] = y[0];  // the sentinel writes the padding column
        s_part[sub][vb + 1][jj] = y[1];
      }
    }
    };
    const bool np_in = !__all_sync(0xffffffffu, P[0].np0 >= hi && P[0].np1 >= hi &&
                                                  P[1].np0 >= hi && P[1].np1 >= hi);
    if (slow)
      walk(std::false_type{}, std::true_type{});
    else if (np_in)
      walk(std::true_type{}, std::true_type{});
    else
      walk(std::true_type{}, std::false_type{});
    if constexpr (kDirect) {
      hi = lo;  // the next batch's barrier orders the staging buffers
      continue;
    }
    __syncthreads();
    // combine the sub-quarters in a fixed order and write each (tile, splat) pair's slot:
    // warp h sums values 4h .. 4h+3 of entry `lane` (h = 1: drgb; value 7 is unused)
    static_assert(kDirect || (kB == 32 && kBT == 64), "flush maps entry = lane, half = warp");
    if (lane < cnt) {
      const int jj = lane;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
      for (int r = 0; r < kSubs; ++r) {
        if (!((s_rel[r][0] >> jj) & 1u)) continue;
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] += s_part[r][4 * w + k][jj];
      }
      const size_t e = cur.slot[jj];
      if (w == 0) {
        // kernels.hpp:219-220: dg/du = g 2 dx / s^2, dg/ds = g 2 r^2 / s^3 (go already carries
        // the opacity): (du, dv) scale by 2 / s^2, dsigma2d by 2 / s^3
        const float inv_s2 = cur.geo[jj].w * -kLn2;  // 1 / sigma2d^2
        const float k2 = 2.0f * inv_s2;
        partial[2 * e] = make_float4(v[0] * k2, v[1] * k2, v[2] * (k2 * fast_sqrt(inv_s2)), v[3]);
      } else {
        partial[2 * e + 1] = make_float4(v[0], v[1], v[2], 0.0f);
      }
    }
    hi = lo;
  }
}

// Loss without gradients (evaluation): per-tile sum of squared differences, same tiling and
// summation order as the backward's prologue.
__global__ void __launch_bounds__(kTilePixels) k_l2_tiles(FrameParams fp,
                                                          const float* __restrict__ img,
                                                          const float* __restrict__ target,
                                                          double* __restrict__ tile_loss) {
  __shared__ float s_red[kTilePixels / 32];
  const int tile = blockIdx.x;
  const int tx = tile % fp.tiles_x, ty = tile / fp.tiles_x;
  const int x = tx * kTile + (threadIdx.x & (kTile - 1)), y = ty * kTile + threadIdx.x / kTile;
  float d2 = 0.0f;
  if (x < fp.cam.width && y < fp.cam.height) {
    const size_t pix = (size_t)y * fp.cam.width + x;
    for (int c = 0; c < 3; ++c) {
      const float d = img[3 * pix + c] - target[3 * pix + c];
      d2 += d * d;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d2 += __shfl_xor_sync(0xffffffffu, d2, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = d2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < kTilePixels / 32; ++i) t += (double)s_red[i];
    tile_loss[tile] = t;
  }
}

// scale * sum(tile_loss) in a fixed order: added to *accum (if not null), stored to *set.
constexpr int kReduceThreads = 1024;
__global__ void __launch_bounds__(kReduceThreads) k_loss_reduce(
    const double* __restrict__ tile_loss, int n_tiles, double scale, double* __restrict__ accum,
    double* __restrict__ set) {
  pdl_enter();
  __shared__ double s[kReduceThreads / 32];
  // fixed order: thread t sums tiles t, t + 1024, ... (8 loads in flight), then a fixed
  // shuffle tree and a fixed sum over the warps
  double acc = 0.0;
  for (int i0 = 0; i0 < n_tiles; i0 += 8 * kReduceThreads) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * kReduceThreads + (int)threadIdx.x;
      v[u] = i < n_tiles ? tile_loss[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kReduceThreads / 32; ++w) t += s[w];
    if (accum) *accum += t * scale;
    *set = t * scale;
  }
}

void launch_blend_bwd(const FrameParams& fp, const uint2* ranges, const uint2* sorted,
                      const uint16_t* submask, const RenderRec* rec,
                      const unsigned long long* total, int64_t key_cap,
                      const float* img, const float* target, const float* t_last,
                      const uint32_t* n_proc, float loss_scale, float4* partial,
                      double* tile_loss, bool given_dldc, float* grad2d, cudaStream_t st) {
  auto k = grad2d ? (given_dldc ? k_blend_bwd<true, true> : k_blend_bwd<false, true>)
                  : (given_dldc ? k_blend_bwd<true, false> : k_blend_bwd<false, false>);
  launch_pdl(k, dim3(fp.n_tiles), dim3(kBT), 0, st, fp, ranges, sorted, submask, rec, total,
             key_cap, img, target, t_last, n_proc, loss_scale, partial, tile_loss, grad2d);
}

void launch_loss_reduce(const double* tile_loss, int n_tiles, double scale, double* accum,
                        double* set, cudaStream_t st) {
  launch_pdl(k_loss_reduce, dim3(1), dim3(kReduceThreads), 0, st, (const double*)tile_loss,
             n_tiles, scale, accum, set);
}

void launch_l2_tiles(const FrameParams& fp, const float* img, const float* target,
                     double* tile_loss, cudaStream_t st) {
  k_l2_tiles<<<fp.n_tiles, kTilePixels, 0, st>>>(fp, img, target, tile_loss);
}

}  // namespace isg

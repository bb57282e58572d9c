// K8 — projection backward and the fused Adam step.
//
// Each splat's 2D gradient (du, dv, dsigma2d, dopacity, drgb) is the sum of its (tile, splat)
// gradient slots written by K7.  Splat g's slots are listed at slot_of[slot_off[g] + k],
// k < ntiles[g], in emission (row-major tile) order — or are the contiguous range
// [slot_off[g], + ntiles[g]) when slot_of is null (radix binning) — and are summed in that
// fixed order, so gradients are bitwise deterministic (no atomics anywhere).
//
// Projection backward: chain rule through u = f x/z + cx, v = f y/z + cy, s = sigma f/z
// (Jacobian: projection_jacobian, /root/reference/proj/src/splat3d.cpp:39-47; closed forms of
// the kernel gradient: include/isosplat/kernels.hpp:208-222), rotated back to world space with
// R^T.  Optimizer slot: update_step (src/optimize.cpp:78-108) — sigma moves in log space
// (:93,:105), updates with a non-finite gradient are skipped and counted (:87-90) — with the
// Adam rule of torch.optim.Adam on (mu, log sigma, rgb, logit opacity).
//
// One thread per splat; params, moments and 3D grads are float4 SoA, coalesced.
#include <algorithm>
#include <cstdlib>

#include "isg_math.cuh"

namespace isg {

namespace {

// MUFU approximations (~2 ulp) for K8's arithmetic: the optimizer and the chain rule are
// compared with tolerances, never bit for bit (and nothing is binned from them)
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void sum_slots(const float4* __restrict__ partial,
                                          const uint32_t* __restrict__ slot_of, uint32_t off,
                                          uint32_t cnt, float4& a, float4& b) {
  a = make_float4(0.f, 0.f, 0.f, 0.f);
  b = make_float4(0.f, 0.f, 0.f, 0.f);
  // kUnroll slots' loads in flight at once, then summed in slot order (same order as a plain
  // loop, so the result is unchanged and deterministic)
  constexpr uint32_t kUnroll = 4;
  for (uint32_t k0 = 0; k0 < cnt; k0 += kUnroll) {
    float4 x[kUnroll], y[kUnroll];
#pragma unroll
    for (uint32_t u = 0; u < kUnroll; ++u) {
      if (k0 + u < cnt) {
        const size_t e = slot_of ? slot_of[off + k0 + u] : (size_t)(off + k0 + u);
        x[u] = partial[2 * e];
        y[u] = partial[2 * e + 1];
      }
    }
#pragma unroll
    for (uint32_t u = 0; u < kUnroll; ++u) {
      if (k0 + u < cnt) {
        a.x += x[u].x;
        a.y += x[u].y;
        a.z += x[u].z;
        a.w += x[u].w;
        b.x += y[u].x;
        b.y += y[u].y;
        b.z += y[u].z;
      }
    }
  }
}

// Splat i's 2D gradient sums of one view: its gradient slots (slot mode, already scaled by
// K7's flush) or, in direct mode (grad2d != null), the dense L2-reduced sums, read and zeroed
// for the next view (the caller scales them, see grad3d_of).
__device__ __forceinline__ void load_2d(int64_t i, float* __restrict__ grad2d,
                                        const float4* __restrict__ partial,
                                        const uint32_t* __restrict__ slot_of,
                                        const uint32_t* __restrict__ slot_off,
                                        const uint32_t* __restrict__ ntiles, bool skip,
                                        float4& a, float4& b) {
  if (grad2d) {
    float4* g = reinterpret_cast<float4*>(grad2d) + 2 * i;
    a = g[0];
    b = g[1];
    g[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    g[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  } else {
    sum_slots(partial, slot_of, slot_off[i], skip ? 0u : ntiles[i], a, b);
  }
}

// a = (sum go dx, sum go dy, sum go r2, sum go) with go = dL/dalpha * alpha (K7), so alpha's
// opacity factor is already in: sum go = o dL/do.  Direct mode (!scaled): kernels.hpp:219-220,
// dg/du = g 2 dx / s^2, dg/ds = g 2 r^2 / s^3, so (du, dv) scale by 2 / s^2 and dsigma2d by
// 2 / s^3 (s = sigma2d of this projection); slot mode: K7's flush scaled them.
// The chain rule needs only the camera-space centre and 1 / z: no exact-rounding projection
// here (nothing is binned from it), one fast reciprocal instead of K1's three IEEE divisions.
__device__ __forceinline__ void grad3d_of(const float4 ms, const isg_camera& cam, float4 a,
                                          float4 b, float out[8], float opacity, bool scaled) {
  const float xc = cam.R[0] * ms.x + cam.R[1] * ms.y + cam.R[2] * ms.z + cam.t[0];
  const float yc = cam.R[3] * ms.x + cam.R[4] * ms.y + cam.R[5] * ms.z + cam.t[1];
  const float zc = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(cam.R[6], ms.x), __fmul_rn(cam.R[7], ms.y)),
                                       __fmul_rn(cam.R[8], ms.z)),
                             cam.t[2]);  // K1's rounding: the same near-plane decision
  if (!(zc > kNearPlane)) {
#pragma unroll
    for (int j = 0; j < 8; ++j) out[j] = 0.f;
    return;
  }
  const float iz = rcp_approx(zc);
  const float fz = cam.focal * iz;
  if (!scaled) {
    // s = sigma f / z; (du, dv) scale by 2 / s^2, dsigma2d by 2 / s^3
    const float inv_s = rcp_approx(ms.w * fz);
    const float k2 = 2.0f * inv_s * inv_s;
    a.x *= k2;
    a.y *= k2;
    a.z *= k2 * inv_s;
  }
  const float gx = a.x * fz, gy = a.y * fz;
  const float gz = -(((a.x * xc + a.y * yc) + a.z * ms.w) * fz) * iz;
  out[0] = (cam.R[0] * gx + cam.R[3] * gy) + cam.R[6] * gz;
  out[1] = (cam.R[1] * gx + cam.R[4] * gy) + cam.R[7] * gz;
  out[2] = (cam.R[2] * gx + cam.R[5] * gy) + cam.R[8] * gz;
  out[3] = a.z * fz;
  out[4] = b.x;
  out[5] = b.y;
  out[6] = b.z;
  out[7] = a.w * rcp_approx(fmaxf(opacity, kOpacityFloor));  // K1's floored opacity
}

// Optimizer space (torch.optim.Adam on the parameters (mu, log sigma, rgb, logit opacity)):
// log sigma and logit opacity live in `raw` (float2 per splat) and persist across steps, so
// sigma = exp(raw.x) and opacity = sigmoid(raw.y) are never re-derived from the rendered
// values (no log/exp round-trip drift; an opacity of exactly 0 or 1 is entered into the open
// interval once, by k_raw_init).  A parameter whose update is exactly zero keeps its stored
// value bit for bit (a zero-gradient step from zero moments is a no-op).
//
// A splat's optimizer inputs, loaded together up front (every load in flight at once: the
// kernels are HBM streams whose only limit is memory-level parallelism).
struct AdamIn {
  float4 P0, P1;          // (mu, sigma), (rgb, opacity)
  float2 R;               // (log sigma, logit opacity)
  float4 M0, M1, V0, V1;  // moments
};
__device__ __forceinline__ AdamIn adam_load(const float4* __restrict__ ms,
                                            const float4* __restrict__ co,
                                            const float2* __restrict__ raw,
                                            const float4* __restrict__ m,
                                            const float4* __restrict__ v, int64_t i) {
  AdamIn a;
  a.P0 = ms[i];
  a.P1 = co[i];
  a.R = raw[i];
  a.M0 = m[2 * i];
  a.M1 = m[2 * i + 1];
  a.V0 = v[2 * i];
  a.V1 = v[2 * i + 1];
  return a;
}

__device__ __forceinline__ void adam_apply(const AdamIn& in, float4* __restrict__ ms,
                                           float4* __restrict__ co, float2* __restrict__ raw,
                                           float4* __restrict__ m, float4* __restrict__ v,
                                           int64_t i, const float gr[8], const AdamParams& ap,
                                           unsigned long long* skipped) {
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 8; ++j) ok &= isfinite(gr[j]);
  if (!ok) {
    atomicAdd(skipped, 1ull);
    return;
  }
  const float sigma = in.P0.w;
  const float s = rcp_approx(1.0f + __expf(-in.R.y));  // sigmoid(logit) of the optimizer state
  float p[8] = {in.P0.x, in.P0.y, in.P0.z, in.R.x, in.P1.x, in.P1.y, in.P1.z, in.R.y};
  const float g[8] = {gr[0], gr[1], gr[2], gr[3] * sigma,
                      gr[4], gr[5], gr[6], gr[7] * s * (1.0f - s)};
  float mm[8] = {in.M0.x, in.M0.y, in.M0.z, in.M0.w, in.M1.x, in.M1.y, in.M1.z, in.M1.w};
  float vv[8] = {in.V0.x, in.V0.y, in.V0.z, in.V0.w, in.V1.x, in.V1.y, in.V1.z, in.V1.w};
  const int group[8] = {0, 0, 0, 1, 2, 2, 2, 3};
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    mm[j] = mm[j] + (1.0f - ap.b1) * (g[j] - mm[j]);
    vv[j] = ap.b2 * vv[j] + (1.0f - ap.b2) * g[j] * g[j];
    // MUFU square root and reciprocal (~2 ulp; the oracle's IEEE forms agree to ~1e-7 rel)
    const float denom = sqrt_approx(vv[j]) * ap.inv_bc2_sqrt + ap.eps;
    // m == 0 moves nothing (also with eps == 0 and v == 0, where m / denom would be 0 / 0)
    const float upd = mm[j] == 0.0f ? 0.0f : mm[j] * rcp_approx(denom);
    p[j] = p[j] - ap.step_size[group[j]] * upd;
  }
  m[2 * i] = make_float4(mm[0], mm[1], mm[2], mm[3]);
  m[2 * i + 1] = make_float4(mm[4], mm[5], mm[6], mm[7]);
  v[2 * i] = make_float4(vv[0], vv[1], vv[2], vv[3]);
  v[2 * i + 1] = make_float4(vv[4], vv[5], vv[6], vv[7]);
  raw[i] = make_float2(p[3], p[7]);
  ms[i] = make_float4(p[0], p[1], p[2], p[3] == in.R.x ? sigma : __expf(p[3]));
  co[i] = make_float4(p[4], p[5], p[6],
                      p[7] == in.R.y ? in.P1.w : rcp_approx(1.0f + __expf(-p[7])));
}

}  // namespace

// One thread: step counter, bias corrections (torch.optim.Adam: step_size = lr / (1 - b1^t),
// denominator sqrt(v) / sqrt(1 - b2^t) + eps) and the loss hand-over of the step.
__global__ void k_adam_tick(AdamParams in, AdamState* __restrict__ st, double* __restrict__ loss,
                            const unsigned long long* __restrict__ total) {
  pdl_enter();
  loss[2] = loss[0];
  loss[0] = 0.0;
  // a view of this step was skipped (key-capacity overflow): the whole step is a no-op, the
  // host reports it at its next check and the caller re-runs the step
  if (total[kTotalOverflowMax] != 0ull) return;
  const long long t = st->t + 1;
  st->t = t;
  const double bc1 = 1.0 - pow((double)in.b1, (double)t);
  const double bc2 = 1.0 - pow((double)in.b2, (double)t);
  AdamParams p = in;
  for (int i = 0; i < 4; ++i) p.step_size[i] = (float)((double)in.lr[i] / bc1);
  p.bc2_sqrt = (float)sqrt(bc2);
  p.inv_bc2_sqrt = (float)(1.0 / sqrt(bc2));
  st->p = p;
}

// Optimizer state of freshly set splats: raw = (log sigma, logit opacity), the opacity taken
// into [kOpacityEps, 1 - kOpacityEps] first (logit(0) and logit(1) are infinite).
__global__ void __launch_bounds__(256) k_raw_init(const float4* __restrict__ ms,
                                                  const float4* __restrict__ co, int64_t n,
                                                  float2* __restrict__ raw) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float op = fminf(fmaxf(co[i].w, kOpacityEps), 1.0f - kOpacityEps);
  raw[i] = make_float2(logf(ms[i].w), logf(op) - log1pf(-op));
}

__global__ void __launch_bounds__(256) k_project_backward(
    const float4* __restrict__ ms, const float4* __restrict__ co, int64_t n, FrameParams fp,
    const uint32_t* __restrict__ slot_off, const uint32_t* __restrict__ slot_of,
    const uint32_t* __restrict__ ntiles, const float4* __restrict__ partial,
    float* __restrict__ grad2d, const unsigned long long* __restrict__ total, int64_t cap,
    float4* __restrict__ grad3d, bool first, int64_t begin) {
  const int64_t i = begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const bool ov = *total > (unsigned long long)cap;  // frame was skipped: contributes nothing
  const float4 P0 = ms[i];
  const float op = co[i].w;
  float4 a, b;
  load_2d(i, grad2d, partial, slot_of, slot_off, ntiles, ov, a, b);
  float o[8];
  grad3d_of(P0, fp.cam, a, b, o, op, !grad2d);
  float4 g0 = make_float4(o[0], o[1], o[2], o[3]), g1 = make_float4(o[4], o[5], o[6], o[7]);
  if (!first) {
    const float4 h0 = grad3d[2 * i], h1 = grad3d[2 * i + 1];
    g0 = make_float4(g0.x + h0.x, g0.y + h0.y, g0.z + h0.z, g0.w + h0.w);
    g1 = make_float4(g1.x + h1.x, g1.y + h1.y, g1.z + h1.z, g1.w + h1.w);
  }
  grad3d[2 * i] = g0;
  grad3d[2 * i + 1] = g1;
}

#ifndef ISG_ADAM_MINB
#define ISG_ADAM_MINB 0
#endif
#if ISG_ADAM_MINB > 0
#define ISG_ADAM_BOUNDS __launch_bounds__(256, ISG_ADAM_MINB)
#else
#define ISG_ADAM_BOUNDS __launch_bounds__(256)
#endif
__global__ void ISG_ADAM_BOUNDS k_project_adam(
    float4* __restrict__ ms, float4* __restrict__ co, int64_t n, FrameParams fp,
    const uint32_t* __restrict__ slot_off, const uint32_t* __restrict__ slot_of,
    const uint32_t* __restrict__ ntiles, const float4* __restrict__ partial,
    float* __restrict__ grad2d, unsigned long long* __restrict__ total,
    float2* __restrict__ raw, float4* __restrict__ m, float4* __restrict__ v,
    const AdamState* __restrict__ state) {
  pdl_enter();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // an overflowed frame since the last host check: no update (the host re-runs the step);
  // the direct-mode sums are consumed (zeroed) either way
  const bool skip = total[kTotalOverflowMax] != 0ull;
  const AdamIn in = adam_load(ms, co, raw, m, v, i);
  float4 a, b;
  load_2d(i, grad2d, partial, slot_of, slot_off, ntiles, skip, a, b);
  if (skip) return;
  const AdamParams ap = state->p;
  float o[8];
  grad3d_of(in.P0, fp.cam, a, b, o, in.P1.w, !grad2d);
  adam_apply(in, ms, co, raw, m, v, i, o, ap, total + kTotalSkipped);
}

// ---- the optimizer-side kernels as persistent HBM streams -----------------------------------
// K8 and its multi-view / multi-GPU halves are pure streams (K8: 136 B read + 136 B written per
// splat) whose speed is set by how many bytes are in flight.  Each CTA owns chunks of kAS
// splats; one thread issues 1D bulk copies (cp.async.bulk, TMA) of a chunk's input arrays into a
// shared-memory stage that completes on an mbarrier, two stages deep, so the next chunk is in
// flight while the current one is computed and stored (one splat per thread, coalesced float4
// stores).  The partial last chunk is read directly.
constexpr int kAS = 128;  // splats per chunk = threads per CTA

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Stream `nfull` full chunks of NA arrays (array a: src[a], bpe[a] bytes per splat, laid out one
// after another in a stage) through the two stages at `smem`.  Per chunk c (owned by this CTA)
// `load(stage, a_off)` reads the thread's inputs from the stage into registers, the stage is
// refilled, then `compute(regs, c)` runs while the refill is in flight.
template <int NA, class Load, class Compute>
__device__ __forceinline__ void stream_chunks(unsigned char* smem, uint64_t* bar,
                                              const unsigned char* const (&src)[NA],
                                              const uint32_t (&bpe)[NA], int64_t nfull,
                                              Load&& load, Compute&& compute) {
  uint32_t off[NA], sb = 0;
#pragma unroll
  for (int a = 0; a < NA; ++a) {
    off[a] = sb;
    sb += kAS * bpe[a];
  }
  const int64_t G = gridDim.x;
  auto issue = [&](int s, int64_t c) {  // one thread: chunk c into stage s
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])),
                 "r"(sb)
                 : "memory");
#pragma unroll
    for (int a = 0; a < NA; ++a)
      bulk_load(smem + s * sb + off[a], src[a] + c * kAS * bpe[a], kAS * bpe[a], &bar[s]);
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar[0]);
    mbar_init(&bar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (blockIdx.x < nfull) issue(0, blockIdx.x);
    if (blockIdx.x + G < nfull) issue(1, blockIdx.x + G);
  }
  __syncthreads();
  uint32_t phase = 0;  // bit s: parity of stage s's next completion
  int it = 0;
  for (int64_t c = blockIdx.x; c < nfull; c += G, ++it) {
    const int s = it & 1;
    mbar_wait(&bar[s], (phase >> s) & 1u);
    phase ^= 1u << s;
    auto regs = load(smem + s * sb, off);
    // stage s consumed: refill it with the chunk two ahead (the generic-proxy reads of the
    // stage are ordered before the async-proxy writes of the refill)
    __syncthreads();
    if (threadIdx.x == 0 && c + 2 * G < nfull) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(s, c + 2 * G);
    }
    compute(regs, c);
  }
}

template <class T>
__device__ __forceinline__ const T* at(const unsigned char* stage, uint32_t off) {
  return reinterpret_cast<const T*>(stage + off);
}

// Adam over splats [0, n) of the (offset) arrays.  kProject: g is the view's 2D gradient sums
// (direct mode; read, zeroed, projected: K8).  Otherwise g is the summed 3D gradient (the
// multi-view / multi-GPU step after the projection backward and the all-reduce).
template <bool kProject>
__global__ void __launch_bounds__(kAS) k_adam_stream(
    float4* __restrict__ ms, float4* __restrict__ co, int64_t n, FrameParams fp,
    float4* __restrict__ g, unsigned long long* __restrict__ total, float2* __restrict__ raw,
    float4* __restrict__ m, float4* __restrict__ v, const AdamState* __restrict__ state) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bar[2];
  const int tid = threadIdx.x;
  if constexpr (kProject) pdl_enter();
  // an overflowed frame since the last host check: no update (the host re-runs the step);
  // K8's direct-mode sums are consumed (zeroed) either way
  if (total[kTotalOverflowMax] != 0ull) {
    if constexpr (kProject)
      for (int64_t i = (int64_t)blockIdx.x * kAS + tid; i < n; i += (int64_t)gridDim.x * kAS) {
        g[2 * i] = make_float4(0.f, 0.f, 0.f, 0.f);
        g[2 * i + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    return;
  }
  const AdamParams ap = state->p;
  struct Regs {
    AdamIn in;
    float4 a, b;
  };
  auto step = [&](const Regs& r, int64_t i) {
    float o[8];
    if constexpr (kProject) {
      g[2 * i] = make_float4(0.f, 0.f, 0.f, 0.f);
      g[2 * i + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
      grad3d_of(r.in.P0, fp.cam, r.a, r.b, o, r.in.P1.w, false);
    } else {
      o[0] = r.a.x; o[1] = r.a.y; o[2] = r.a.z; o[3] = r.a.w;
      o[4] = r.b.x; o[5] = r.b.y; o[6] = r.b.z; o[7] = r.b.w;
    }
    adam_apply(r.in, ms, co, raw, m, v, i, o, ap, total + kTotalSkipped);
  };
  const unsigned char* const src[6] = {
      reinterpret_cast<const unsigned char*>(ms), reinterpret_cast<const unsigned char*>(co),
      reinterpret_cast<const unsigned char*>(m), reinterpret_cast<const unsigned char*>(v),
      reinterpret_cast<const unsigned char*>(g), reinterpret_cast<const unsigned char*>(raw)};
  constexpr uint32_t bpe[6] = {16, 16, 32, 32, 32, 8};
  const int64_t nfull = n / kAS;
  stream_chunks<6>(
      smem_raw, bar, src, bpe, nfull,
      [&](const unsigned char* st, const uint32_t* off) {
        Regs r;
        r.in.P0 = at<float4>(st, off[0])[tid];
        r.in.P1 = at<float4>(st, off[1])[tid];
        r.in.M0 = at<float4>(st, off[2])[2 * tid];
        r.in.M1 = at<float4>(st, off[2])[2 * tid + 1];
        r.in.V0 = at<float4>(st, off[3])[2 * tid];
        r.in.V1 = at<float4>(st, off[3])[2 * tid + 1];
        r.a = at<float4>(st, off[4])[2 * tid];
        r.b = at<float4>(st, off[4])[2 * tid + 1];
        r.in.R = at<float2>(st, off[5])[tid];
        return r;
      },
      [&](const Regs& r, int64_t c) { step(r, c * kAS + tid); });
  // the partial last chunk: the CTA that would own it reads it directly
  if (nfull % gridDim.x == blockIdx.x) {
    const int64_t i = nfull * kAS + tid;
    if (i < n) {
      Regs r;
      r.in = adam_load(ms, co, raw, m, v, i);
      r.a = g[2 * i];
      r.b = g[2 * i + 1];
      step(r, i);
    }
  }
}

// Projection backward of one view for splats [begin, end): grad3d (+)= J^T grad2d, grad2d
// zeroed for the next view (direct mode).  Streams ms, co, grad2d and, unless first, grad3d.
template <bool kFirst>
__global__ void __launch_bounds__(kAS) k_project_stream(
    const float4* __restrict__ ms, const float4* __restrict__ co, int64_t begin, int64_t end,
    FrameParams fp, float4* __restrict__ g2, float4* __restrict__ grad3d) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bar[2];
  const int tid = threadIdx.x;
  struct Regs {
    float4 P0, a, b, h0, h1;
    float op;
  };
  auto step = [&](const Regs& r, int64_t i) {
    g2[2 * i] = make_float4(0.f, 0.f, 0.f, 0.f);
    g2[2 * i + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
    float o[8];
    grad3d_of(r.P0, fp.cam, r.a, r.b, o, r.op, false);
    float4 q0 = make_float4(o[0], o[1], o[2], o[3]), q1 = make_float4(o[4], o[5], o[6], o[7]);
    if constexpr (!kFirst) {
      q0 = make_float4(q0.x + r.h0.x, q0.y + r.h0.y, q0.z + r.h0.z, q0.w + r.h0.w);
      q1 = make_float4(q1.x + r.h1.x, q1.y + r.h1.y, q1.z + r.h1.z, q1.w + r.h1.w);
    }
    grad3d[2 * i] = q0;
    grad3d[2 * i + 1] = q1;
  };
  constexpr int NA = kFirst ? 3 : 4;
  const unsigned char* src[NA];
  uint32_t bpe[NA];
  src[0] = reinterpret_cast<const unsigned char*>(ms + begin);
  bpe[0] = 16;
  src[1] = reinterpret_cast<const unsigned char*>(co + begin);
  bpe[1] = 16;
  src[2] = reinterpret_cast<const unsigned char*>(g2 + 2 * begin);
  bpe[2] = 32;
  if constexpr (!kFirst) {
    src[NA - 1] = reinterpret_cast<const unsigned char*>(grad3d + 2 * begin);
    bpe[NA - 1] = 32;
  }
  const int64_t nfull = (end - begin) / kAS;
  stream_chunks<NA>(
      smem_raw, bar, src, bpe, nfull,
      [&](const unsigned char* st, const uint32_t* off) {
        Regs r;
        r.P0 = at<float4>(st, off[0])[tid];
        r.op = at<float4>(st, off[1])[tid].w;
        r.a = at<float4>(st, off[2])[2 * tid];
        r.b = at<float4>(st, off[2])[2 * tid + 1];
        if constexpr (!kFirst) {
          r.h0 = at<float4>(st, off[NA - 1])[2 * tid];
          r.h1 = at<float4>(st, off[NA - 1])[2 * tid + 1];
        }
        return r;
      },
      [&](const Regs& r, int64_t c) { step(r, begin + c * kAS + tid); });
  if (nfull % gridDim.x == blockIdx.x) {
    const int64_t i = begin + nfull * kAS + tid;
    if (i < end) {
      Regs r;
      r.P0 = ms[i];
      r.op = co[i].w;
      r.a = g2[2 * i];
      r.b = g2[2 * i + 1];
      if constexpr (!kFirst) {
        r.h0 = grad3d[2 * i];
        r.h1 = grad3d[2 * i + 1];
      }
      step(r, i);
    }
  }
}

// Resident CTAs of a stream kernel on the whole GPU (its dynamic shared memory set up once).
template <class K>
int stream_grid_max(K kernel, size_t smem) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kAS, smem);
  return std::max(1, sms * std::max(1, per_sm));
}
constexpr size_t kAdamStreamSmem = 2 * kAS * 136;
bool use_stream() {
  static const bool on = [] {
    const char* e = std::getenv("ISG_K8_STREAM");
    return !(e && e[0] == '0');
  }();
  return on;
}

__global__ void __launch_bounds__(256) k_adam(float4* __restrict__ ms, float4* __restrict__ co,
                                              int64_t n, const float4* __restrict__ grad3d,
                                              float2* __restrict__ raw, float4* __restrict__ m,
                                              float4* __restrict__ v,
                                              const AdamState* __restrict__ state,
                                              unsigned long long* __restrict__ total) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (total[kTotalOverflowMax] != 0ull) return;  // a view of the step was skipped
  const AdamIn in = adam_load(ms, co, raw, m, v, i);
  const float4 g0 = grad3d[2 * i], g1 = grad3d[2 * i + 1];
  const AdamParams ap = state->p;
  const float o[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
  adam_apply(in, ms, co, raw, m, v, i, o, ap, total + kTotalSkipped);
}

void launch_project_backward(const float4* ms, const float4* co, int64_t n,
                             const FrameParams& fp, const uint32_t* slot_off,
                             const uint32_t* slot_of, const uint32_t* ntiles,
                             const float4* partial, float* grad2d,
                             const unsigned long long* total, int64_t cap, float4* grad3d,
                             bool first, cudaStream_t st, int64_t begin, int64_t end) {
  if (end < 0 || end > n) end = n;
  if (end <= begin) return;
  if (grad2d && use_stream() && begin % kAS == 0) {
    static const int gmax[2] = {stream_grid_max(k_project_stream<true>, 2 * kAS * 64),
                                stream_grid_max(k_project_stream<false>, 2 * kAS * 96)};
    const int64_t chunks = (end - begin + kAS - 1) / kAS;
    auto k = first ? k_project_stream<true> : k_project_stream<false>;
    k<<<(unsigned)std::min<int64_t>(chunks, gmax[first ? 0 : 1]), kAS,
        first ? 2 * kAS * 64 : 2 * kAS * 96, st>>>(ms, co, begin, end, fp,
                                                   reinterpret_cast<float4*>(grad2d), grad3d);
    return;
  }
  k_project_backward<<<(unsigned)((end - begin + 255) / 256), 256, 0, st>>>(
      ms, co, end, fp, slot_off, slot_of, ntiles, partial, grad2d, total, cap, grad3d, first,
      begin);
}

// ---- multi-GPU exchange: the step's loss and overflow state ride in the gradient all-reduce --
// slots[r] = (hi, mid, lo, overflowed) for rank r, zero for every other rank: after the sum
// every rank holds every rank's values unchanged (x + 0 = x), and hi + mid + lo reconstructs
// the rank's double loss exactly (24 + 24 + <= 5 significant bits).
__global__ void k_loss_pack(const double* __restrict__ loss,
                            const unsigned long long* __restrict__ total, float4* __restrict__ slots,
                            int rank, int nranks) {
  const int r = threadIdx.x;
  if (r >= nranks) return;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (r == rank) {
    const double L = loss[0];
    const float hi = (float)L;
    const double r1 = L - (double)hi;
    const float mid = (float)r1;
    s = make_float4(hi, mid, (float)(r1 - (double)mid),
                    total[kTotalOverflowMax] != 0ull ? 1.0f : 0.0f);
  }
  slots[r] = s;
}

// After the exchange: loss[0] = the sum of the ranks' losses in rank order (identical on every
// rank; k_adam_tick hands it over to loss[2]); any rank's overflow makes every rank skip the
// step (replicas stay identical), recorded like a local overflow for the host's next check.
__global__ void k_loss_unpack(double* __restrict__ loss, unsigned long long* __restrict__ total,
                              const float4* __restrict__ slots, int nranks) {
  double sum = 0.0;
  bool ovf = false;
  for (int r = 0; r < nranks; ++r) {
    const float4 s = slots[r];
    sum += ((double)s.x + (double)s.y) + (double)s.z;
    ovf |= s.w != 0.0f;
  }
  loss[0] = sum;
  if (ovf && total[kTotalOverflowMax] == 0ull) {
    total[kTotalOverflowMax] = total[kTotalKeys];
    total[kTotalOverflowFrames] += 1ull;
  }
}

void launch_loss_pack(const double* loss, const unsigned long long* total, float4* slots,
                      int rank, int nranks, cudaStream_t st) {
  k_loss_pack<<<1, 64, 0, st>>>(loss, total, slots, rank, nranks);
}
void launch_loss_unpack(double* loss, unsigned long long* total, const float4* slots, int nranks,
                        cudaStream_t st) {
  k_loss_unpack<<<1, 1, 0, st>>>(loss, total, slots, nranks);
}

void launch_project_adam(float4* ms, float4* co, int64_t n, const FrameParams& fp,
                         const uint32_t* slot_off, const uint32_t* slot_of,
                         const uint32_t* ntiles, const float4* partial, float* grad2d,
                         unsigned long long* total, float2* raw, float4* m, float4* v,
                         const AdamState* ap, cudaStream_t st) {
  if (n <= 0) return;
  if (grad2d && use_stream()) {
    static const int grid_max = stream_grid_max(k_adam_stream<true>, kAdamStreamSmem);
    const int64_t chunks = (n + kAS - 1) / kAS;
    launch_pdl(k_adam_stream<true>, dim3((unsigned)std::min<int64_t>(chunks, grid_max)),
               dim3(kAS), kAdamStreamSmem, st, ms, co, n, fp, reinterpret_cast<float4*>(grad2d),
               total, raw, m, v, ap);
    return;
  }
  launch_pdl(k_project_adam, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, ms, co, n,
             fp, slot_off, slot_of, ntiles, partial, grad2d, total, raw, m, v, ap);
}

void launch_adam(float4* ms, float4* co, int64_t n, const float4* grad3d, float2* raw, float4* m,
                 float4* v, const AdamState* ap, unsigned long long* total, cudaStream_t st) {
  if (n <= 0) return;
  // (the plain one-thread-per-splat kernel already streams at ~7 TB/s: C4 0.115 ms vs 0.129 ms
  // through k_adam_stream<false>)
  k_adam<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ms, co, n, grad3d, raw, m, v, ap, total);
}

void launch_raw_init(const float4* ms, const float4* co, int64_t n, float2* raw, cudaStream_t st) {
  if (n <= 0) return;
  k_raw_init<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ms, co, n, raw);
}

void launch_adam_tick(const float lr[4], float b1, float b2, float eps, AdamState* st_dev,
                      double* loss, const unsigned long long* total, cudaStream_t st) {
  AdamParams in{};
  for (int i = 0; i < 4; ++i) in.lr[i] = lr[i];
  in.b1 = b1;
  in.b2 = b2;
  in.eps = eps;
  launch_pdl(k_adam_tick, dim3(1), dim3(1), 0, st, in, st_dev, loss, total);
}

}  // namespace isg

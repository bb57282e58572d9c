// L1 + D-SSIM image loss and its pixel gradient, the paper's loss
// (1 - lambda) L1 + lambda (1 - SSIM), lambda = 0.2 by default.
//
// Semantics follow /root/reference/proj/src/loss.cpp:
//   window       11 taps, sigma 1.5, normalised Gaussian, separable            :16-35
//   statistics   m1, m2, sigma11, sigma22, sigma12 from zero-padded filtering  :49-102
//   ssim         mean of (2 m1 m2 + C1)(2 s12 + C2) / ((m1^2 + m2^2 + C1)(s11 + s22 + C2)) over
//                the VALID window positions [5, dim-6] of every channel        :119-141
//   gradient     per valid window dS/d(m2, t2, t12), filtered back (zero padded) and combined
//                as norm (F1 + 2 fhat F2 + f F3)                               :143-182
//   loss         (1-l) l1 + l (1 - ssim); lambda == 0 skips SSIM entirely      :184-190
//   dL/dfhat     (1-l)/N sign(fhat - f) - l dSSIM/dfhat, sign(0) = 0           :201-213
// with f = target, fhat = rendered image; everything here is scaled by the view weight w.
//
// Two kernels over 32x32-pixel output tiles (all three channels per CTA, one at a time):
//   k_ssim_fwd  stages the tile's 42x42 halo region of both images in shared memory (RGB
//               interleaved, as in HBM), runs the 11-tap horizontal then vertical pass for the
//               five moments (each thread 4 consecutive outputs per pass, register-blocked),
//               and at every valid position evaluates S and the three gradient coefficients
//               (written as 9 planes, zero outside the valid region); per-CTA partial sums of
//               |f - fhat| and S go to `part` (reduced in a fixed order, deterministic).
//   k_ssim_bwd  filters the coefficient planes back (same 11-tap separable pass) and writes
//               dL/dfhat (HWC3), which K7 (k_blend_bwd<true>) consumes as G.
// The moments are FP32 (the reference is FP64); for images in [0,1] the cancellation in
// t - m^2 is ~1e-7 against C2 = 9e-4, well inside the loss/gradient tolerances of the tests.
#include <algorithm>
#include <cmath>

#include "isg_internal.cuh"

namespace isg {

namespace {

constexpr int kT = 32;  // output tile kT x kT, all three channels
constexpr int kHalf = kSsimHalf, kWin = 2 * kSsimHalf + 1;
constexpr int kR = kT + 2 * kHalf;  // 42: halo region side
constexpr int kThreads = 256;       // 8 warps
constexpr int kG = 4;               // outputs per thread in each 1D pass (register blocking)
constexpr int kIn = kG + kWin - 1;  // 14 inputs cover kG outputs
constexpr int kHItems = kR * (kT / kG);  // horizontal-pass work items per plane (336)
// Shared-memory pitches (odd / +1 so that lanes walking different rows hit different banks)
constexpr int kPitchI = 3 * kR + 1;  // interleaved RGB rows of the images (127)
constexpr int kPitchP = kR + 1;      // planar coefficient rows (43)
constexpr int kPitchH = kT + 1;      // horizontal-pass results (33)
constexpr float kC1 = 0.01f * 0.01f, kC2 = 0.03f * 0.03f;

struct Taps {
  float w[kWin];
};

Taps make_taps() {  // loss.cpp:22-35, in FP64 then rounded
  double t[kWin], sum = 0.0;
  for (int i = 0; i < kWin; ++i) {
    const double d = i - kHalf;
    t[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
    sum += t[i];
  }
  Taps tp;
  for (int i = 0; i < kWin; ++i) tp.w[i] = (float)(t[i] / sum);
  return tp;
}

__device__ __forceinline__ float sgn(float r) { return r > 0.0f ? 1.0f : (r < 0.0f ? -1.0f : 0.0f); }

// 4-byte asynchronous global->shared copy; src_ok == false zero-fills (src not read).
__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool src_ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src),
               "r"(src_ok ? 4 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Block-wide sum of two floats per thread into double2 (fixed order).
__device__ void block_sum2(float a, float b, double2* out) {
  __shared__ float s[2][kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s[0][threadIdx.x >> 5] = a;
    s[1][threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) {
      x += (double)s[0][i];
      y += (double)s[1][i];
    }
    *out = make_double2(x, y);
  }
}

// lambda == 0: the L1 term alone (loss.cpp:188) and, with dldc, its sign gradient.
__global__ void __launch_bounds__(kThreads) k_l1(int W, int H, const float* __restrict__ fhat,
                                                 const float* __restrict__ f, float w1,
                                                 double2* __restrict__ part,
                                                 float* __restrict__ dldc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gx = blockIdx.x * kT + lane;
  float l1 = 0.0f;
#pragma unroll
  for (int o = 0; o < kG; ++o) {
    const int gy = blockIdx.y * kT + warp * kG + o;
    if (gx < W && gy < H) {
      const size_t p = 3 * ((size_t)gy * W + gx);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float r = fhat[p + c] - f[p + c];
        l1 += fabsf(r);
        if (dldc) dldc[p + c] = w1 * sgn(r);
      }
    }
  }
  block_sum2(l1, 0.0f, part + blockIdx.y * gridDim.x + blockIdx.x);
}

struct FwdSmem {
  float a[kR][kPitchI];  // target f, interleaved RGB, halo region
  float b[kR][kPitchI];  // render fhat
  float h[5][kR][kPitchH];
};

// Moments of one channel -> S and the gradient coefficients at the tile's valid positions.
template <bool kGrad>
__global__ void __launch_bounds__(kThreads) k_ssim_fwd(int W, int H, const float* __restrict__ fhat,
                                                       const float* __restrict__ f, Taps tp,
                                                       float* __restrict__ coef,
                                                       double2* __restrict__ part) {
  extern __shared__ float4 smem_raw[];
  FwdSmem& S = *reinterpret_cast<FwdSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bx = blockIdx.x * kT, by = blockIdx.y * kT;
  const size_t HW = (size_t)W * H;
  const int row_len = 3 * W;
  // stage the halo region as it lies in HBM (interleaved RGB rows), all copies in flight at
  // once; zero outside the image
  for (int r = warp; r < kR; r += kThreads / 32) {
    const int gy = by - kHalf + r;
    const bool row_ok = gy >= 0 && gy < H;
    const size_t roff = row_ok ? (size_t)gy * row_len : 0;
#pragma unroll
    for (int k0 = 0; k0 < 3 * kR; k0 += 32) {
      const int k = k0 + lane;
      if (k < 3 * kR) {
        const int gx3 = 3 * (bx - kHalf) + k;
        const bool ok = row_ok && gx3 >= 0 && gx3 < row_len;
        const size_t o = ok ? roff + gx3 : 0;
        cp_async4(&S.a[r][k], f + o, ok);
        cp_async4(&S.b[r][k], fhat + o, ok);
      }
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  // L1 over the tile's own pixels (thread: column lane, rows warp*kG ..)
  float l1 = 0.0f, ssum = 0.0f;
  const int x = lane, y0 = warp * kG;
#pragma unroll
  for (int o = 0; o < kG; ++o)
    if (bx + x < W && by + y0 + o < H) {
#pragma unroll
      for (int c = 0; c < 3; ++c)
        l1 += fabsf(S.a[y0 + o + kHalf][3 * (x + kHalf) + c] - S.b[y0 + o + kHalf][3 * (x + kHalf) + c]);
    }
  for (int c = 0; c < 3; ++c) {
    // horizontal pass: item = (row, kG consecutive outputs); lanes walk different rows
    for (int i = tid; i < kHItems; i += kThreads) {
      const int g = i / kR, r = i - g * kR;
      const float* pa = &S.a[r][3 * g * kG + c];
      const float* pb = &S.b[r][3 * g * kG + c];
      // (m1, m2) and (t1, t2) as packed f32x2 pairs (FFMA2), t12 scalar
      float2 am[kG], at[kG];
      float ax[kG];
#pragma unroll
      for (int o = 0; o < kG; ++o) {
        am[o] = at[o] = make_float2(0.0f, 0.0f);
        ax[o] = 0.0f;
      }
#pragma unroll
      for (int j = 0; j < kIn; ++j) {
        const float2 ab = make_float2(pa[3 * j], pb[3 * j]);
        const float2 sq = __fmul2_rn(ab, ab);
        const float x12 = ab.x * ab.y;
#pragma unroll
        for (int o = 0; o < kG; ++o) {
          const int d = j - o;
          if (d >= 0 && d < kWin) {
            const float2 wd = make_float2(tp.w[d], tp.w[d]);
            am[o] = __ffma2_rn(wd, ab, am[o]);
            at[o] = __ffma2_rn(wd, sq, at[o]);
            ax[o] = fmaf(tp.w[d], x12, ax[o]);
          }
        }
      }
#pragma unroll
      for (int o = 0; o < kG; ++o) {
        S.h[0][r][g * kG + o] = am[o].x;
        S.h[1][r][g * kG + o] = am[o].y;
        S.h[2][r][g * kG + o] = at[o].x;
        S.h[3][r][g * kG + o] = at[o].y;
        S.h[4][r][g * kG + o] = ax[o];
      }
    }
    __syncthreads();
    // vertical pass: thread = (column lane, kG consecutive output rows)
    float2 vm[kG], vt[kG];
    float vx[kG];
#pragma unroll
    for (int o = 0; o < kG; ++o) {
      vm[o] = vt[o] = make_float2(0.0f, 0.0f);
      vx[o] = 0.0f;
    }
#pragma unroll
    for (int j = 0; j < kIn; ++j) {
      const float2 hm = make_float2(S.h[0][y0 + j][x], S.h[1][y0 + j][x]);
      const float2 ht = make_float2(S.h[2][y0 + j][x], S.h[3][y0 + j][x]);
      const float hx = S.h[4][y0 + j][x];
#pragma unroll
      for (int o = 0; o < kG; ++o) {
        const int d = j - o;
        if (d >= 0 && d < kWin) {
          const float2 wd = make_float2(tp.w[d], tp.w[d]);
          vm[o] = __ffma2_rn(wd, hm, vm[o]);
          vt[o] = __ffma2_rn(wd, ht, vt[o]);
          vx[o] = fmaf(tp.w[d], hx, vx[o]);
        }
      }
    }
    float acc[kG][5];
#pragma unroll
    for (int o = 0; o < kG; ++o) {
      acc[o][0] = vm[o].x;
      acc[o][1] = vm[o].y;
      acc[o][2] = vt[o].x;
      acc[o][3] = vt[o].y;
      acc[o][4] = vx[o];
    }
    const int gx = bx + x;
#pragma unroll
    for (int o = 0; o < kG; ++o) {
      const int gy = by + y0 + o;
      if (gx >= W || gy >= H) continue;
      const bool valid = gx >= kHalf && gx < W - kHalf && gy >= kHalf && gy < H - kHalf;
      float g_m2 = 0.f, g_t2 = 0.f, g_t12 = 0.f;
      if (valid) {
        const float m1 = acc[o][0], m2 = acc[o][1];
        const float s11 = acc[o][2] - m1 * m1, s22 = acc[o][3] - m2 * m2;
        const float s12 = acc[o][4] - m1 * m2;
        const float nl = 2.0f * m1 * m2 + kC1, dl = m1 * m1 + m2 * m2 + kC1;
        const float nc = 2.0f * s12 + kC2, dc = s11 + s22 + kC2;
        const float idl = rcp_approx(dl), idc = rcp_approx(dc);
        const float lum = nl * idl, cs = nc * idc;
        ssum += lum * cs;
        if (kGrad) {  // loss.cpp:164-170
          const float d_s22 = -lum * cs * idc;
          const float d_s12 = 2.0f * lum * idc;
          const float d_lum_m2 = 2.0f * (m1 * dl - nl * m2) * (idl * idl);
          g_m2 = cs * d_lum_m2 - 2.0f * m2 * d_s22 - m1 * d_s12;
          g_t2 = d_s22;
          g_t12 = d_s12;
        }
      }
      if (kGrad) {
        const size_t p = (size_t)gy * W + gx;
        coef[(3 * c + 0) * HW + p] = g_m2;
        coef[(3 * c + 1) * HW + p] = g_t2;
        coef[(3 * c + 2) * HW + p] = g_t12;
      }
    }
    __syncthreads();  // S.h is rewritten by the next channel
  }
  block_sum2(l1, ssum, part + blockIdx.y * gridDim.x + blockIdx.x);
}

#ifndef ISG_SSIM_BWD_BUFS
#define ISG_SSIM_BWD_BUFS 1
#endif
// ISG_SSIM_BWD_BUFS channel buffers of coefficient planes: 3 = all channels in flight at once
// (82 KB, 2 CTAs/SM); 1 = one channel at a time, the next one streaming in during the
// vertical pass (38 KB, 5 CTAs/SM; measured 4% faster)
struct BwdSmem {
  float c[ISG_SSIM_BWD_BUFS][3][kR][kPitchP];  // [channel buffer][coefficient] planes, halo
  float h[3][kR][kPitchH];
};

// dL/dfhat = w1 sign(fhat - f) - wln (F1 + 2 fhat F2 + f F3), F = window-filtered coefficients.
__global__ void __launch_bounds__(kThreads) k_ssim_bwd(int W, int H, const float* __restrict__ fhat,
                                                       const float* __restrict__ f,
                                                       const float* __restrict__ coef, Taps tp,
                                                       float w1, float wln,
                                                       float* __restrict__ dldc) {
  extern __shared__ float4 smem_raw[];
  BwdSmem& S = *reinterpret_cast<BwdSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bx = blockIdx.x * kT, by = blockIdx.y * kT;
  const size_t HW = (size_t)W * H;
  const int x = lane, y0 = warp * kG;
  // coefficient planes of channel c into buffer c % ISG_SSIM_BWD_BUFS, one commit group each
  auto stage_channel = [&](int c) {
    for (int rr = warp; rr < 3 * kR; rr += kThreads / 32) {
      const int k = rr / kR, r = rr - k * kR;
      const int gy = by - kHalf + r;
      const bool row_ok = gy >= 0 && gy < H;
      const float* src = coef + (3 * c + k) * HW + (row_ok ? (size_t)gy * W : 0);
#pragma unroll
      for (int px0 = 0; px0 < kR; px0 += 32) {
        const int px = px0 + lane;
        if (px < kR) {
          const int gx = bx - kHalf + px;
          const bool ok = row_ok && gx >= 0 && gx < W;
          cp_async4(&S.c[c % ISG_SSIM_BWD_BUFS][k][r][px], ok ? src + gx : coef, ok);
        }
      }
    }
    cp_async_commit();
  };
  for (int c = 0; c < ISG_SSIM_BWD_BUFS; ++c) stage_channel(c);
  // the thread's output pixels of both images, loaded while the planes stream in
  float fa[kG][3], fb[kG][3];
  {
    const int gx = bx + x;
#pragma unroll
    for (int o = 0; o < kG; ++o) {
      const int gy = by + y0 + o;
      const bool ok = gx < W && gy < H;
      const size_t p = ok ? 3 * ((size_t)gy * W + gx) : 0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        fa[o][c] = ok ? f[p + c] : 0.0f;
        fb[o][c] = ok ? fhat[p + c] : 0.0f;
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    if (ISG_SSIM_BWD_BUFS == 3 && c == 0) cp_async_wait<2>();
    else if (ISG_SSIM_BWD_BUFS == 3 && c == 1) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    // coefficients 0 and 1 as a packed f32x2 pair (FFMA2, same per-lane rounding as fmaf),
    // coefficient 2 scalar
    for (int i = tid; i < kHItems; i += kThreads) {
      const int g = i / kR, r = i - g * kR;
      float2 a01[kG];
      float a2[kG];
#pragma unroll
      for (int o = 0; o < kG; ++o) {
        a01[o] = make_float2(0.0f, 0.0f);
        a2[o] = 0.0f;
      }
#pragma unroll
      for (int j = 0; j < kIn; ++j) {
        const float2 v01 = make_float2(S.c[c % ISG_SSIM_BWD_BUFS][0][r][g * kG + j],
                                       S.c[c % ISG_SSIM_BWD_BUFS][1][r][g * kG + j]);
        const float v2 = S.c[c % ISG_SSIM_BWD_BUFS][2][r][g * kG + j];
#pragma unroll
        for (int o = 0; o < kG; ++o) {
          const int d = j - o;
          if (d >= 0 && d < kWin) {
            a01[o] = __ffma2_rn(make_float2(tp.w[d], tp.w[d]), v01, a01[o]);
            a2[o] = fmaf(tp.w[d], v2, a2[o]);
          }
        }
      }
#pragma unroll
      for (int o = 0; o < kG; ++o) {
        S.h[0][r][g * kG + o] = a01[o].x;
        S.h[1][r][g * kG + o] = a01[o].y;
        S.h[2][r][g * kG + o] = a2[o];
      }
    }
    __syncthreads();
    // one buffer: the planes of channel c are consumed, the next channel's stream in during
    // the vertical pass
    if (ISG_SSIM_BWD_BUFS == 1 && c + 1 < 3) stage_channel(c + 1);
    float2 b01[kG];
    float b2[kG];
#pragma unroll
    for (int o = 0; o < kG; ++o) {
      b01[o] = make_float2(0.0f, 0.0f);
      b2[o] = 0.0f;
    }
#pragma unroll
    for (int j = 0; j < kIn; ++j) {
      const float2 v01 = make_float2(S.h[0][y0 + j][x], S.h[1][y0 + j][x]);
      const float v2 = S.h[2][y0 + j][x];
#pragma unroll
      for (int o = 0; o < kG; ++o) {
        const int d = j - o;
        if (d >= 0 && d < kWin) {
          b01[o] = __ffma2_rn(make_float2(tp.w[d], tp.w[d]), v01, b01[o]);
          b2[o] = fmaf(tp.w[d], v2, b2[o]);
        }
      }
    }
    float acc[kG][3];
#pragma unroll
    for (int o = 0; o < kG; ++o) {
      acc[o][0] = b01[o].x;
      acc[o][1] = b01[o].y;
      acc[o][2] = b2[o];
    }
    const int gx = bx + x;
#pragma unroll
    for (int o = 0; o < kG; ++o) {
      const int gy = by + y0 + o;
      if (gx >= W || gy >= H) continue;
      const size_t p = 3 * ((size_t)gy * W + gx) + c;
      const float a = fa[o][c], b = fb[o][c];
      const float g = acc[o][0] + 2.0f * b * acc[o][1] + a * acc[o][2];
      dldc[p] = w1 * sgn(b - a) - wln * g;
    }
    __syncthreads();  // S.h is rewritten by the next channel
  }
}

// loss = l1_scale * sum|f - fhat| + wl - ssim_scale * sum S  (fixed order over CTAs)
__global__ void k_ssim_reduce(const double2* __restrict__ part, int n, double l1_scale, double wl,
                              double ssim_scale, const unsigned long long* __restrict__ total,
                              int64_t key_cap, double* __restrict__ accum,
                              double* __restrict__ set) {
  __shared__ double s[2][256];
  if (total && *total > (unsigned long long)key_cap) {  // the frame was skipped (regrow + re-run)
    if (threadIdx.x == 0) *set = 0.0;
    return;
  }
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) {
    a += part[i].x;
    b += part[i].y;
  }
  s[0][threadIdx.x] = a;
  s[1][threadIdx.x] = b;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      s[0][threadIdx.x] += s[0][threadIdx.x + o];
      s[1][threadIdx.x] += s[1][threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double loss = l1_scale * s[0][0] + (wl - ssim_scale * s[1][0]);
    if (accum) *accum += loss;
    *set = loss;
  }
}

dim3 ssim_grid(int W, int H) { return dim3((W + kT - 1) / kT, (H + kT - 1) / kT); }

__global__ void k_l2_grad(int64_t n, const float* __restrict__ fhat, const float* __restrict__ f,
                          float scale, float* __restrict__ dldc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dldc[i] = scale * (fhat[i] - f[i]);
}

}  // namespace

void launch_l2_grad(int W, int H, const float* fhat, const float* target, float scale,
                    float* dldc, cudaStream_t st) {
  const int64_t n = 3 * (int64_t)W * H;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_l2_grad<<<blocks, 256, 0, st>>>(n, fhat, target, scale, dldc);
}

int64_t ssim_part_count(int W, int H) {
  const dim3 g = ssim_grid(W, H);
  return (int64_t)g.x * g.y;
}

int launch_image_loss(int W, int H, const float* fhat, const float* target, float lambda,
                       double weight, bool grad, float* coef, double2* part, float* dldc,
                       const unsigned long long* total, int64_t key_cap, double* accum,
                       double* set, cudaStream_t st) {
  static const Taps tp = make_taps();
  static const bool attr = [] {
    cudaFuncSetAttribute(k_ssim_fwd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(FwdSmem));
    cudaFuncSetAttribute(k_ssim_fwd<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(FwdSmem));
    cudaFuncSetAttribute(k_ssim_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(BwdSmem));
    return true;
  }();
  (void)attr;
  const dim3 grid = ssim_grid(W, H);
  const bool ssim = lambda != 0.0f;
  const double N = 3.0 * W * (double)H;
  const double valid = ssim ? 3.0 * (W - 2 * kHalf) * (double)(H - 2 * kHalf) : 1.0;
  const double lam = (double)lambda;
  const float w1 = (float)(weight * (1.0 - lam) / N);
  const float wln = (float)(weight * lam / valid);
  if (!ssim) {
    k_l1<<<grid, kThreads, 0, st>>>(W, H, fhat, target, w1, part, grad ? dldc : nullptr);
  } else if (grad) {
    k_ssim_fwd<true><<<grid, kThreads, sizeof(FwdSmem), st>>>(W, H, fhat, target, tp, coef, part);
    k_ssim_bwd<<<grid, kThreads, sizeof(BwdSmem), st>>>(W, H, fhat, target, coef, tp, w1, wln,
                                                         dldc);
  } else {
    k_ssim_fwd<false><<<grid, kThreads, sizeof(FwdSmem), st>>>(W, H, fhat, target, tp, coef, part);
  }
  k_ssim_reduce<<<1, 256, 0, st>>>(part, (int)(grid.x * grid.y), weight * (1.0 - lam) / N,
                                   ssim ? weight * lam : 0.0, ssim ? weight * lam / valid : 0.0,
                                   total, key_cap, accum, set);
  return (ssim && grad) ? 3 : 2;
}

}  // namespace isg

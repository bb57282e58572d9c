// L2 reduction throughput on B200: red.global.add.v2/v4.f32 to pseudo-random splat records of a
// 1M x 32 B gradient buffer (the access pattern of per-sub-quarter gradient accumulation in
// the blend backward), vs plain stores.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned hash(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
template <int MODE>
__global__ void k(float* g, unsigned n_splat, unsigned iters, int coherent) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  for (unsigned i = 0; i < iters; ++i) {
    // 4 consecutive lanes hit the same splat (one sub-quarter group), groups random
    const unsigned grp = coherent ? (t >> 2) : t;
    const unsigned s = hash(grp * 1315423911u + i) % n_splat;
    float* p = g + 8 * (size_t)s;
    if (MODE == 0) {  // v2 per lane: lane l of the group adds values 2l, 2l+1
      float* q = p + 2 * (t & 3);
      asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(q), "f"(1.0f), "f"(2.0f) : "memory");
    } else if (MODE == 1) {  // v4 per lane pair
      if ((t & 1) == 0) {
        float* q = p + 4 * ((t >> 1) & 1);
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(q), "f"(1.0f), "f"(2.0f),
                     "f"(3.0f), "f"(4.0f) : "memory");
      }
    } else {  // plain v2 stores (no atomics)
      float* q = p + 2 * (t & 3);
      *reinterpret_cast<float2*>(q) = make_float2(1.0f, (float)i);
    }
  }
}

int main() {
  const unsigned n_splat = 1u << 20;
  float* g;
  cudaMalloc(&g, sizeof(float) * 8 * n_splat);
  cudaMemset(g, 0, sizeof(float) * 8 * n_splat);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = 148 * 16, threads = 256;
  const unsigned iters = 64;
  const double lanes = (double)blocks * threads * iters;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<blocks, threads>>>(g, n_splat, iters, 1);
      if (mode == 1) k<1><<<blocks, threads>>>(g, n_splat, iters, 1);
      if (mode == 2) k<2><<<blocks, threads>>>(g, n_splat, iters, 1);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = mode == 1 ? lanes / 2 : lanes;
      if (rep == 2)
        printf("%s: %.0f M ops in %.3f ms -> %.1f G ops/s (%.1f GB/s payload)\n",
               mode == 0 ? "red.v2.f32" : mode == 1 ? "red.v4.f32" : "st.v2.f32", ops / 1e6, ms,
               ops / ms / 1e6, ops * (mode == 1 ? 16 : 8) / ms / 1e6);
    }
  }
  return 0;
}

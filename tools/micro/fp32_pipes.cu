// Microbenchmark: per-SM throughput of FFMA (3-reg), FFMA2 (packed f32x2), FMUL2 and MUFU.EX2
// on this GPU.  Each thread runs 8 independent chains; results written to keep the code live.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp32_pipes.cu -o fp32_pipes && ./fp32_pipes
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void ffma(float* out, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  float bb = b + threadIdx.x * 1e-9f;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, bb);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}

__global__ void ffma2(float* out, float a, float b) {
  unsigned long long x[8];
  for (int i = 0; i < 8; ++i) x[i] = pk(threadIdx.x + i, i);
  const unsigned long long aa = pk(a, a), bb = pk(b + threadIdx.x * 1e-9f, b);
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(aa), "l"(bb));
  float s = 0;
  for (int i = 0; i < 8; ++i) {
    float p, q;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(p), "=f"(q) : "l"(x[i]));
    s += p + q;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ex2(float* out, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = (threadIdx.x + i) * 1e-3f;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

typedef void (*Kern)(float*, float, float);
float run(Kern k, float* out, int blocks, int threads) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<blocks, threads>>>(out, 0.999f, 1e-3f);
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(out, 0.999f, 1e-3f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256;
  float* out;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  const double ops = (double)blocks * threads * kIters * 8;  // per-thread ops
  const double warp_ops = ops / 32;
  float t1 = run(ffma, out, blocks, threads);
  float t2 = run(ffma2, out, blocks, threads);
  float t3 = run(ex2, out, blocks, threads);
  const double cyc = clk * 1e3;  // Hz
  auto per = [&](float ms) { return warp_ops / (ms * 1e-3 * cyc * sms * 4); };
  printf("sms %d clock %.0f MHz\n", sms, clk / 1e3);
  printf("FFMA : %.3f ms  %.3f warp-instr/clk/SMSP  %.1f TFLOP/s\n", t1, per(t1), 2 * ops / t1 / 1e9);
  printf("FFMA2: %.3f ms  %.3f warp-instr/clk/SMSP  %.1f TFLOP/s\n", t2, per(t2), 4 * ops / t2 / 1e9);
  printf("EX2  : %.3f ms  %.3f warp-instr/clk/SMSP\n", t3, per(t3));
  return 0;
}

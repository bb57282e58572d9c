// Microbenchmark: issue rates of the instruction classes K6/K7 are made of, alone and mixed, in
// warp-instructions per clock per SM sub-partition (SMSP).  8 independent chains per thread,
// 8 CTAs x 256 threads per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 pipes2.cu -o pipes2 && ./pipes2
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 2048;

__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float unpk(unsigned long long v) {
  float p, q;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(p), "=f"(q) : "l"(v));
  return p + q;
}

#define KERNEL(name, decl, fin, ...)                                        \
  __global__ void name(float* out, float a, float b) {                        \
    decl;                                                                     \
    for (int it = 0; it < kIters; ++it) {                                     \
      _Pragma("unroll") for (int i = 0; i < 8; ++i) { __VA_ARGS__; }          \
    }                                                                         \
    float s = 0;                                                              \
    for (int i = 0; i < 8; ++i) s += fin;                                     \
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;                           \
  }
#define FFMA(x) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x) : "f"(a), "f"(c))
#define FADD(x) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x) : "f"(c))
#define FFMA2(x) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(aa), "l"(bb))
#define FADD2(x) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(bb))
#define FSEL(x) asm volatile("{.reg .pred p; setp.gt.f32 p, %1, 0f00000000; selp.f32 %0, %0, %1, p;}" : "+f"(x) : "f"(c))
#define FSETP(y, x) asm volatile("{.reg .pred p; setp.gt.f32 p, %1, %2; selp.u32 %0, 1, 0, p;}" : "=r"(y) : "f"(x), "f"(c))
#define EX2(x) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x))
#define RCP(x) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(x))
#define ISEL(x) asm volatile("{.reg .pred p; setp.lt.s32 p, %0, %1; selp.s32 %0, %0, %1, p;}" : "+r"(x) : "r"(ic))
#define D1 float x[8]; float z[8]; float c = b + threadIdx.x * 1e-9f; int ic = threadIdx.x; \
  unsigned long long X[8]; unsigned y[8]; const unsigned long long aa = pk(a, a);            \
  const unsigned long long bb = pk(b + threadIdx.x * 1e-9f, b);                            \
  int iv[8]; \
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x + i; z[i] = i * 1e-3f; X[i] = pk(threadIdx.x + i, i); y[i] = 0; iv[i] = i * 7; }
#define FIN (x[i] + z[i] + unpk(X[i]) + (float)y[i] + (float)iv[i])

KERNEL(k_ffma, D1, FIN, FFMA(x[i]))
KERNEL(k_fadd, D1, FIN, FADD(x[i]))
KERNEL(k_ffma2, D1, FIN, FFMA2(X[i]))
KERNEL(k_fadd2, D1, FIN, FADD2(X[i]))
KERNEL(k_fsel, D1, FIN, FSEL(x[i]))
KERNEL(k_fsetp_only, D1, FIN, FSETP(y[i], x[i]); x[i] += 1.0f)
KERNEL(k_ffma2_fsel, D1, FIN, FFMA2(X[i]); FSEL(z[i]))
KERNEL(k_ffma2_fadd, D1, FIN, FFMA2(X[i]); FADD(z[i]))
KERNEL(k_ffma_fadd, D1, FIN, FFMA(x[i]); FADD(z[i]))
KERNEL(k_shfl, D1, FIN, x[i] = __shfl_xor_sync(0xffffffffu, x[i], 1 + (i & 1)))
KERNEL(k_ffma2_shfl, D1, FIN, FFMA2(X[i]); z[i] = __shfl_xor_sync(0xffffffffu, z[i], 1 + (i & 1)))
KERNEL(k_ex2, D1, FIN, EX2(z[i]))
KERNEL(k_rcp, D1, FIN, RCP(x[i]))
KERNEL(k_ffma2_ex2, D1, FIN, FFMA2(X[i]); EX2(z[i]))
KERNEL(k_isetp_sel, D1, FIN, ISEL(iv[i]))
KERNEL(k_ffma2_x2_fsel, D1, FIN, FFMA2(X[i]); FFMA2(X[i ^ 1]); FSEL(z[i]))

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
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256;
  float* out;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  const double warp_steps = (double)blocks * threads / 32 * kIters * 8;
  const double hz = clk * 1e3;
  struct {
    const char* name;
    Kern k;
    int instr;  // warp-instructions per chain step
  } ks[] = {{"FFMA", k_ffma, 1},          {"FADD", k_fadd, 1},
            {"FFMA2", k_ffma2, 1},        {"FADD2", k_fadd2, 1},
            {"FSETP+FSEL", k_fsel, 2},    {"FSETP+SEL+FADD", k_fsetp_only, 3},
            {"FFMA2+FSETP+FSEL", k_ffma2_fsel, 3}, {"FFMA2+FADD", k_ffma2_fadd, 2},
            {"FFMA+FADD", k_ffma_fadd, 2}, {"SHFL", k_shfl, 1},
            {"FFMA2+SHFL", k_ffma2_shfl, 2}, {"EX2", k_ex2, 1},
            {"RCP", k_rcp, 1},            {"FFMA2+EX2", k_ffma2_ex2, 2},
            {"ISETP+SEL", k_isetp_sel, 2}, {"2FFMA2+FSETP+FSEL", k_ffma2_x2_fsel, 4}};
  printf("sms %d clock %.0f MHz (steps: chain steps; rate: warp-instr/clk/SMSP of the step's instructions)\n",
         sms, clk / 1e3);
  for (auto& e : ks) {
    const float ms = run(e.k, out, blocks, threads);
    const double steps_per_clk = warp_steps / (ms * 1e-3 * hz * sms * 4);
    printf("%-18s %8.3f ms  steps/clk/SMSP %.3f  instr/clk/SMSP %.3f\n", e.name, ms, steps_per_clk,
           steps_per_clk * e.instr);
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return 0;
}

// Microbenchmark: per-tile stable sort of (depth key, splat) lists in shared memory, one CTA per
// tile (the segmented alternative to the global depth sort + depth-order emission).  8160
// segments (1080p tiles) of ~411 entries (C3), keys = float bits of depths in [2, 10], values in
// increasing order (stability = index order).  Checks against std::stable_sort.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 segsort_bench.cu -o segsort_bench
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include <cuda_runtime.h>

constexpr int kT = 256;          // threads per CTA
constexpr int kCap = 2048;       // entries sorted in shared memory
constexpr int kItems = kCap / kT;

__device__ __forceinline__ uint32_t warp_match9(uint32_t d) {
  uint32_t peers = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < 9; ++b) {
    const bool bit = (d >> b) & 1u;
    const uint32_t m = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? m : ~m;
  }
  return peers;
}

struct SegSmem {
  uint32_t key[2][kCap];
  uint32_t val[2][kCap];
  uint32_t wcnt[kT / 32][257];
  uint32_t dstart[256];
  uint32_t wtmp[8];
  uint32_t red[2];
};

__global__ void __launch_bounds__(kT) k_segsort(const uint2* __restrict__ ranges,
                                                const uint32_t* __restrict__ in_val,
                                                const uint32_t* __restrict__ depth_key,
                                                uint32_t* __restrict__ out_val) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SegSmem& S = *reinterpret_cast<SegSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint2 rg = ranges[blockIdx.x];
  const int L = (int)(rg.y - rg.x);
  if (L <= 0 || L > kCap) return;
  // items per thread for this segment; warp w owns items [w*32*K, (w+1)*32*K)
  const int K = (L + kT - 1) / kT;
  uint32_t kor = 0, kand = 0xffffffffu;
  for (int i = tid; i < L; i += kT) {
    const uint32_t v = in_val[rg.x + i];
    const uint32_t k = depth_key[v];
    S.key[0][i] = k;
    S.val[0][i] = v;
    kor |= k;
    kand &= k;
  }
  // bits that vary across the segment: passes over constant digits are skipped
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    kor |= __shfl_xor_sync(0xffffffffu, kor, o);
    kand &= __shfl_xor_sync(0xffffffffu, kand, o);
  }
  if (tid == 0) { S.red[0] = 0; S.red[1] = 0xffffffffu; }
  __syncthreads();
  if (lane == 0) { atomicOr(&S.red[0], kor); atomicAnd(&S.red[1], kand); }
  __syncthreads();
  const uint32_t vary = S.red[0] & ~S.red[1];
  const uint32_t lt = (1u << lane) - 1u;
  int cur = 0;
  for (int shift = 0; shift < 32; shift += 8) {
    if (((vary >> shift) & 255u) == 0) continue;  // block-uniform
    for (int i = tid; i < (kT / 32) * 257; i += kT) (&S.wcnt[0][0])[i] = 0;
    __syncthreads();
    uint32_t dig[kItems], rank[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      if (j >= K) break;  // block-uniform
      const int i = w * 32 * K + j * 32 + lane;
      const uint32_t d = i < L ? (S.key[cur][i] >> shift) & 255u : 256u;
      dig[j] = d;
      const uint32_t peers = warp_match9(d);
      const int leader = __ffs(peers) - 1;
      uint32_t before = 0;
      if (lane == leader) before = S.wcnt[w][d];
      before = __shfl_sync(0xffffffffu, before, leader);
      rank[j] = before + __popc(peers & lt);
      if (lane == leader) S.wcnt[w][d] = before + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // per digit (thread = digit): exclusive prefix over warps, then over digits
    uint32_t cnt = 0;
#pragma unroll
    for (int ww = 0; ww < kT / 32; ++ww) {
      const uint32_t c = S.wcnt[ww][tid];
      S.wcnt[ww][tid] = cnt;
      cnt += c;
    }
    {
      uint32_t x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) S.wtmp[w] = x;
      __syncthreads();
      uint32_t wpre = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) wpre += i < w ? S.wtmp[i] : 0u;
      S.dstart[tid] = wpre + x - cnt;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      if (j >= K) break;
      const int i = w * 32 * K + j * 32 + lane;
      const uint32_t d = dig[j];
      if (d < 256u) {
        const uint32_t pos = S.dstart[d] + S.wcnt[w][d] + rank[j];
        S.key[cur ^ 1][pos] = S.key[cur][i];
        S.val[cur ^ 1][pos] = S.val[cur][i];
      }
    }
    __syncthreads();
    cur ^= 1;
  }
  for (int i = tid; i < L; i += kT) out_val[rg.x + i] = S.val[cur][i];
}

int main() {
  const int tiles = 8160;
  std::mt19937 rng(1);
  std::poisson_distribution<int> pl(411);
  std::vector<uint2> ranges(tiles);
  uint32_t total = 0;
  for (int t = 0; t < tiles; ++t) {
    const int L = std::min(pl(rng), kCap);
    ranges[t] = make_uint2(total, total + L);
    total += L;
  }
  const uint32_t nsplat = 1000000;
  std::vector<uint32_t> key(nsplat), val(total);
  std::uniform_real_distribution<float> uz(2.0f, 10.0f);
  for (auto& k : key) {
    const float z = uz(rng);
    std::memcpy(&k, &z, 4);
  }
  std::uniform_int_distribution<uint32_t> us(0, nsplat - 1);
  for (int t = 0; t < tiles; ++t) {  // each tile: splat ids in increasing order
    std::vector<uint32_t> s(ranges[t].y - ranges[t].x);
    for (auto& x : s) x = us(rng);
    std::sort(s.begin(), s.end());
    std::copy(s.begin(), s.end(), val.begin() + ranges[t].x);
  }
  uint2* d_r;
  uint32_t *d_in, *d_key, *d_out;
  cudaMalloc(&d_r, sizeof(uint2) * tiles);
  cudaMalloc(&d_in, 4 * total);
  cudaMalloc(&d_out, 4 * total);
  cudaMalloc(&d_key, 4 * nsplat);
  cudaMemcpy(d_r, ranges.data(), sizeof(uint2) * tiles, cudaMemcpyHostToDevice);
  cudaMemcpy(d_in, val.data(), 4 * total, cudaMemcpyHostToDevice);
  cudaMemcpy(d_key, key.data(), 4 * nsplat, cudaMemcpyHostToDevice);
  const size_t smem = sizeof(SegSmem);
  cudaFuncSetAttribute(k_segsort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_segsort, kT, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) k_segsort<<<tiles, kT, smem>>>(d_r, d_in, d_key, d_out);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int rep = 0; rep < reps; ++rep) k_segsort<<<tiles, kT, smem>>>(d_r, d_in, d_key, d_out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<uint32_t> out(total);
  cudaMemcpy(out.data(), d_out, 4 * total, cudaMemcpyDeviceToHost);
  size_t bad = 0;
  for (int t = 0; t < tiles; ++t) {
    std::vector<uint32_t> s(val.begin() + ranges[t].x, val.begin() + ranges[t].y);
    std::stable_sort(s.begin(), s.end(), [&](uint32_t a, uint32_t b) { return key[a] < key[b]; });
    for (size_t i = 0; i < s.size(); ++i) bad += s[i] != out[ranges[t].x + i];
  }
  printf("segments %d entries %u smem %zu B, %d CTAs/SM: %.2f us per sort, mismatches %zu (%s)\n",
         tiles, total, smem, per_sm, 1000.0 * ms / reps, bad,
         cudaGetErrorString(cudaGetLastError()));
  return bad != 0;
}

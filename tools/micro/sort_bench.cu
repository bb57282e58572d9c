// Standalone timing of the onesweep radix sort (k_sort.cu) on the two C3 binning workloads:
//   depth: 1M float-bit depth keys (z ~ U[2,10]) + iota values, 32 bits
//   tile : 3.36M tile ids (8160 tiles, 13 bits) + values, stable
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//   tools/micro/sort_bench.cu paper_2403_14244_b200/csrc/k_sort.cu -o tools/micro/sort_bench
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "../../paper_2403_14244_b200/csrc/isg_internal.cuh"

static void run(const char* name, std::vector<uint32_t>& hk, bool iota, int bits, int reps) {
  const int64_t n = (int64_t)hk.size();
  const int64_t cap = n + n / 2;
  uint32_t *k[2], *v[2], *ndev;
  for (int i = 0; i < 2; ++i) {
    cudaMalloc(&k[i], cap * 4);
    cudaMalloc(&v[i], cap * 4);
  }
  cudaMalloc(&ndev, 4);
  uint32_t nn = (uint32_t)n;
  cudaMemcpy(ndev, &nn, 4, cudaMemcpyHostToDevice);
  std::vector<uint32_t> hv(n);
  for (int64_t i = 0; i < n; ++i) hv[i] = (uint32_t)i;
  isg::SortScratch s{};
  const int64_t tiles = isg::sort_tiles_for(cap);
  cudaMalloc(&s.hist, isg::kMaxPasses * 256 * 4);
  cudaMalloc(&s.counters, (isg::kMaxPasses + 1) * 4);
  cudaMalloc(&s.lookback, (size_t)isg::kMaxPasses * 256 * tiles * 4);
  s.max_tiles = tiles;
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9, sum = 0;
  int out = 0;
  for (int r = 0; r < reps; ++r) {
    cudaMemcpyAsync(k[0], hk.data(), n * 4, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(v[0], hv.data(), n * 4, cudaMemcpyHostToDevice, st);
    int64_t launches = 0;
    cudaEventRecord(e0, st);
    out = isg::radix_sort_pairs(k, v, iota, ndev, cap, bits, s, st, &launches);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0) {
      best = std::min(best, ms);
      sum += ms;
    }
  }
  // verify stable sort
  std::vector<uint32_t> ok(n), ov(n);
  cudaMemcpy(ok.data(), k[out], n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(ov.data(), v[out], n * 4, cudaMemcpyDeviceToHost);
  std::vector<uint32_t> idx(n);
  for (int64_t i = 0; i < n; ++i) idx[i] = (uint32_t)i;
  const uint32_t mask = bits >= 32 ? 0xFFFFFFFFu : ((1u << bits) - 1);
  std::stable_sort(idx.begin(), idx.end(),
                   [&](uint32_t a, uint32_t b) { return (hk[a] & mask) < (hk[b] & mask); });
  int64_t bad = 0;
  for (int64_t i = 0; i < n; ++i) bad += (ov[i] != idx[i]);
  printf("%-6s n=%lld bits=%d  best %.1f us  mean %.1f us  mismatches %lld\n", name,
         (long long)n, bits, best * 1e3, sum / (reps - 1) * 1e3, (long long)bad);
}

int main() {
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<float> uz(2.0f, 10.0f);
  std::vector<uint32_t> depth(1000000);
  for (auto& d : depth) {
    float z = uz(rng);
    std::memcpy(&d, &z, 4);
  }
  for (int64_t m : {32768L, 131072L, 262144L, 1000000L}) {
    std::vector<uint32_t> d(depth.begin(), depth.begin() + m);
    char name[32];
    snprintf(name, sizeof name, "d%lld", (long long)m);
    run(name, d, true, 32, 20);
  }
  // tile ids in depth order: each splat touches a few neighbouring tiles
  std::vector<uint32_t> tile;
  std::uniform_int_distribution<int> ut(0, 8159), nt(1, 7);
  while (tile.size() < 3360000) {
    int t = ut(rng), c = nt(rng);
    for (int j = 0; j < c && tile.size() < 3360000; ++j) tile.push_back((t + (j & 1) + 120 * (j >> 1)) % 8160);
  }
  run("tile", tile, false, 13, 20);
  if (getenv("SORT_BIG")) {  // C5-sized tile sort: 33M keys over 32400 tiles (15 bits)
    std::vector<uint32_t> big;
    std::uniform_int_distribution<int> ub(0, 32399);
    while (big.size() < 33000000) {
      int t = ub(rng), c = nt(rng);
      for (int j = 0; j < c && big.size() < 33000000; ++j) big.push_back((t + (j & 1) + 240 * (j >> 1)) % 32400);
    }
    run("big", big, false, 15, 5);
  }
  return 0;
}

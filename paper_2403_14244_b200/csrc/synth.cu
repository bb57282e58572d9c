// synth.cu — the synthetic workload "isg-synth v1", host side.
//
// Counter-based RNG (splitmix64 finaliser of seed*phi + 8*i + j, top 24 bits) so a splat's
// parameters depend only on (seed, index): the CPU oracle, the GPU host and any rank generate
// bit-identical scenes without communication.
#include <cmath>
#include <cstdint>

#include "../../include/isg.h"

namespace {
inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline double u01(uint64_t seed, uint64_t i, int j) {
  return (double)(mix64(seed * 0x9E3779B97F4A7C15ull + 8 * i + (uint64_t)j) >> 40) *
         (1.0 / 16777216.0);
}
}  // namespace

extern "C" {

isg_status isg_synth_camera(int32_t W, int32_t H, int32_t view, int32_t n_views, isg_camera* c) {
  if (!c || W <= 0 || H <= 0 || n_views < 1 || view < 0 || view >= n_views) return ISG_E_ARG;
  const double k = view - 0.5 * (n_views - 1);
  const double th = k * 1.5 * M_PI / 180.0;
  const double cs = std::cos(th), sn = std::sin(th);
  const double R[9] = {cs, 0, sn, 0, 1, 0, -sn, 0, cs};
  for (int i = 0; i < 9; ++i) c->R[i] = (float)R[i];
  c->t[0] = (float)(0.05 * k);
  c->t[1] = 0.0f;
  c->t[2] = 0.0f;
  c->focal = (float)(1000.0 * W / 1920.0);
  c->cx = (float)(0.5 * W);
  c->cy = (float)(0.5 * H);
  c->width = W;
  c->height = H;
  return ISG_OK;
}

// Per splat: z ~ U[2,10]; screen position u ~ U[-5%,105%] W, v ~ U[-5%,105%] H back-projected
// through the identity camera; sigma_2d ~ logU[0.5, 8] px so sigma = sigma_2d z / f;
// opacity ~ U[0.05, 0.95]; rgb ~ U[0,1]^3.
isg_status isg_synth_scene(uint64_t seed, int64_t n, int32_t W, int32_t H, float* ms, float* co) {
  if (n < 0 || W <= 0 || H <= 0 || (n > 0 && (!ms || !co))) return ISG_E_ARG;
  const double f = 1000.0 * W / 1920.0, cx = 0.5 * W, cy = 0.5 * H;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const double z = 2.0 + 8.0 * u01(seed, i, 0);
    const double u = W * (-0.05 + 1.1 * u01(seed, i, 1));
    const double v = H * (-0.05 + 1.1 * u01(seed, i, 2));
    const double s2d = 0.5 * std::pow(16.0, u01(seed, i, 3));
    ms[4 * i + 0] = (float)((u - cx) * z / f);
    ms[4 * i + 1] = (float)((v - cy) * z / f);
    ms[4 * i + 2] = (float)z;
    ms[4 * i + 3] = (float)(s2d * z / f);
    co[4 * i + 0] = (float)u01(seed, i, 5);
    co[4 * i + 1] = (float)u01(seed, i, 6);
    co[4 * i + 2] = (float)u01(seed, i, 7);
    co[4 * i + 3] = (float)(0.05 + 0.9 * u01(seed, i, 4));
  }
  return ISG_OK;
}

}  // extern "C"

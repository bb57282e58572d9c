// ref_capi.cpp — extern "C" wrappers around the REFERENCE's own hot-path code, compiled from
// /root/reference/proj/src/{splat3d,image,loss,reconstruct,optimize}.cpp by oracle/build_ref.sh into
// oracle/_ref/libisosplat_ref.so.  TEST INFRASTRUCTURE ONLY (checker / CPU baseline).
//
// The calls go through the reference's public API unchanged:
//   isosplat::render(std::span<const IsoSplat3D>, const Camera&, const RenderOptions&)
//       include/isosplat/splat3d.hpp:96-97, src/splat3d.cpp:173-194
//   isosplat::project_iso   splat3d.hpp:74, splat3d.cpp:59-64
//   isosplat::composite     splat3d.hpp:85, splat3d.cpp:76-87
//   isosplat::mse           image.hpp:40, image.cpp:50-58
//   isosplat::loss / ssim / l1_term / ssim_gradient_wrt_second
//                           loss.hpp:12-24, loss.cpp:112-190
//   isosplat::adaptive_control (IsoParticle2D)   optimize.cpp:221-284
// Exceptions (std::domain_error) become a non-zero return plus the message.
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <utility>
#include <vector>

#include "isosplat/image.hpp"
#include "isosplat/loss.hpp"
#include "isosplat/optimize.hpp"
#include "isosplat/splat3d.hpp"

namespace {
isosplat::Camera make_camera(const double* c, int w, int h) {
  isosplat::Camera cam;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) cam.rotation(i, j) = c[3 * i + j];
  for (int i = 0; i < 3; ++i) cam.translation[i] = c[9 + i];
  cam.focal = c[12];
  cam.principal_point[0] = c[13];
  cam.principal_point[1] = c[14];
  cam.width = w;
  cam.height = h;
  return cam;
}

std::vector<isosplat::IsoSplat3D> make_splats(int64_t n, const double* s) {
  std::vector<isosplat::IsoSplat3D> v(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    const double* r = s + 8 * i;
    v[i].mu = Eigen::Vector3d(r[0], r[1], r[2]);
    v[i].sigma = r[3];
    v[i].color = Eigen::Vector3d(r[4], r[5], r[6]);
    v[i].opacity = r[7];
  }
  return v;
}

int report(const std::exception& e, char* err, int len) {
  if (err && len > 0) {
    std::strncpy(err, e.what(), static_cast<size_t>(len) - 1);
    err[len - 1] = 0;
  }
  return dynamic_cast<const std::domain_error*>(&e) ? 1 : 2;
}
}  // namespace

extern "C" {

// cam: R (row-major 9), t (3), focal, cx, cy.  out: H x W x 3 doubles.
int ref_render(int64_t n, const double* splats, const double* cam, int w, int h, const double* bg,
               int threads, double* out, char* err, int errlen) {
  try {
    const auto sp = make_splats(n, splats);
    isosplat::RenderOptions opt;
    opt.background = Eigen::Vector3d(bg[0], bg[1], bg[2]);
    opt.threads = threads;
    const isosplat::ImageGrid img =
        isosplat::render(std::span<const isosplat::IsoSplat3D>(sp), make_camera(cam, w, h), opt);
    std::memcpy(out, img.data.data(), sizeof(double) * img.data.size());
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, errlen);
  }
}

// Returns 1 and (u, v, sigma2d, depth) when visible, 0 when culled, -1 on domain error.
int ref_project_iso(const double* splat, const double* cam, double* out, char* err, int errlen) {
  try {
    const auto sp = make_splats(1, splat);
    const auto p = isosplat::project_iso(sp[0], make_camera(cam, 1, 1));
    if (!p) return 0;
    out[0] = p->mu2d[0];
    out[1] = p->mu2d[1];
    out[2] = p->sigma2d;
    out[3] = p->depth;
    return 1;
  } catch (const std::exception& e) {
    report(e, err, errlen);
    return -1;
  }
}

int ref_composite(int64_t n, const double* rgba, double* out, char* err, int errlen) {
  try {
    std::vector<std::pair<Eigen::Vector3d, double>> v;
    for (int64_t i = 0; i < n; ++i)
      v.emplace_back(Eigen::Vector3d(rgba[4 * i], rgba[4 * i + 1], rgba[4 * i + 2]), rgba[4 * i + 3]);
    const Eigen::Vector3d c =
        isosplat::composite(std::span<const std::pair<Eigen::Vector3d, double>>(v));
    out[0] = c[0];
    out[1] = c[1];
    out[2] = c[2];
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, errlen);
  }
}

double ref_mse(int w, int h, const double* a, const double* b) {
  isosplat::ImageGrid x(w, h, 3), y(w, h, 3);
  std::memcpy(x.data.data(), a, sizeof(double) * x.data.size());
  std::memcpy(y.data.data(), b, sizeof(double) * y.data.size());
  return isosplat::mse(x, y);
}

namespace {
isosplat::ImageGrid grid_of(int w, int h, const double* d) {
  isosplat::ImageGrid g(w, h, 3);
  std::memcpy(g.data.data(), d, sizeof(double) * g.data.size());
  return g;
}
}  // namespace

// out[0] = loss(f, fhat, lambda), out[1] = l1_term, out[2] = ssim (when lambda != 0 and the
// window fits).  grad (may be null): d ssim / d fhat (ssim_gradient_wrt_second).
int ref_image_loss(int w, int h, const double* f, const double* fhat, double lambda, double* out,
                   double* grad, char* err, int errlen) {
  try {
    const auto a = grid_of(w, h, f), b = grid_of(w, h, fhat);
    out[0] = isosplat::loss(a, b, lambda);
    out[1] = isosplat::l1_term(a, b);
    if (lambda != 0.0) {
      out[2] = isosplat::ssim(a, b);
      if (grad) {
        const auto g = isosplat::ssim_gradient_wrt_second(a, b);
        std::memcpy(grad, g.data.data(), sizeof(double) * g.data.size());
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, errlen);
  }
}

// adaptive_control on IsoParticle2D (optimize.cpp:221-284).  recs: n x 6 (mu.x mu.y sigma A0 A1
// A2); params: prune_threshold, merge_distance_factor, merge_color_tol, split_sigma_max.
// Returns the new count (written to out, capacity out_cap) or -1 on error.
int64_t ref_adaptive_control_2d(int64_t n, const double* recs, const double* params,
                                int max_particles, int channels, uint64_t seed, double* out,
                                int64_t out_cap, char* err, int errlen) {
  try {
    std::vector<isosplat::IsoParticle2D> v(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      const double* r = recs + 6 * i;
      v[i].mu = Eigen::Vector2d(r[0], r[1]);
      v[i].sigma = r[2];
      v[i].amplitude = {r[3], r[4], r[5]};
    }
    isosplat::AdaptiveControlParams a;
    a.prune_threshold = params[0];
    a.merge_distance_factor = params[1];
    a.merge_color_tol = params[2];
    a.split_sigma_max = params[3];
    std::mt19937_64 rng(seed);
    const auto res = isosplat::adaptive_control(std::move(v), a, max_particles, channels, rng);
    const int64_t m = static_cast<int64_t>(res.size());
    for (int64_t i = 0; i < m && i < out_cap; ++i) {
      double* r = out + 6 * i;
      r[0] = res[i].mu[0];
      r[1] = res[i].mu[1];
      r[2] = res[i].sigma;
      r[3] = res[i].amplitude[0];
      r[4] = res[i].amplitude[1];
      r[5] = res[i].amplitude[2];
    }
    return m;
  } catch (const std::exception& e) {
    report(e, err, errlen);
    return -1;
  }
}

}  // extern "C"

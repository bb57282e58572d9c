// isosplat_b200.hpp — C++20 drop-in for the reference's isotropic 3D splat API
// (/root/reference/proj/include/isosplat/splat3d.hpp), backed by the B200 C-ABI (isg.h).
//
// Same namespace, type names, field names and function signatures as the reference:
//   isosplat::IsoSplat3D   splat3d.hpp:13-22   (mu, sigma, color, opacity, geometric_dof, validate)
//   isosplat::Camera       splat3d.hpp:37-53   (rotation, translation, focal, principal_point,
//                                               width, height, to_camera, project_point, validate)
//   isosplat::RenderOptions splat3d.hpp:87-90  (background, threads) + t_min (early termination)
//   isosplat::ImageGrid    image.hpp:11-31     (width, height, channels, data, at)
//   isosplat::render(std::span<const IsoSplat3D>, const Camera&, const RenderOptions&)
//                          splat3d.hpp:96-97
//   isosplat::project_iso / composite / kNearPlane   splat3d.hpp:55, 66-74, 84-85 (host-side)
// plus the training slots the reference lacks: isosplat::Trainer (loss_backward, adam_step).
//
// Eigen is not required: vectors/matrices are small fixed-size types with operator[] and
// (i, j) access, so caller code that indexes fields compiles unchanged.  Errors keep the
// reference's exception types: invalid splats/cameras throw std::domain_error with the
// reference's messages (validation runs in FP64 on the host, splat3d.cpp:10-37, before any
// device call), device failures throw std::runtime_error.  There is no CPU fallback.
#pragma once

#include <array>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "isg.h"

namespace isosplat {

struct Vector2d {
  double v[2] = {0.0, 0.0};
  Vector2d() = default;
  Vector2d(double x, double y) : v{x, y} {}
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
};

struct Vector3d {
  double v[3] = {0.0, 0.0, 0.0};
  Vector3d() = default;
  Vector3d(double x, double y, double z) : v{x, y, z} {}
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
  bool allFinite() const {
    return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]);
  }
};

struct Matrix3d {
  double m[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  static Matrix3d Identity() { return Matrix3d{}; }
  double& operator()(int i, int j) { return m[i][j]; }
  double operator()(int i, int j) const { return m[i][j]; }
};

inline constexpr double kNearPlane = 1e-3;  // splat3d.hpp:55

struct IsoSplat3D {
  Vector3d mu{0.0, 0.0, 0.0};  // world units
  double sigma = 1.0;          // world units, > 0
  Vector3d color{0.0, 0.0, 0.0};
  double opacity = 1.0;  // in [0,1]
  static constexpr int geometric_dof = 4;  // mu:3 + sigma:1

  // IsoSplat3D::validate, splat3d.cpp:10-17 (kernels.hpp:53-61 messages)
  void validate() const {
    if (!mu.allFinite()) throw std::domain_error("IsoSplat3D.mu: non-finite coordinates");
    if (!(sigma > 0.0) || !std::isfinite(sigma))
      throw std::domain_error("IsoSplat3D.sigma: must be positive and finite");
    if (!color.allFinite()) throw std::domain_error("IsoSplat3D.color: non-finite");
    if (!(opacity >= 0.0 && opacity <= 1.0))
      throw std::domain_error("IsoSplat3D.opacity: must be in [0,1]");
  }
};

struct Camera {
  Matrix3d rotation = Matrix3d::Identity();
  Vector3d translation{0.0, 0.0, 0.0};
  double focal = 1.0;  // pixels
  Vector2d principal_point{0.0, 0.0};
  int width = 1, height = 1;

  Vector3d to_camera(const Vector3d& w) const {  // splat3d.hpp:45-47
    Vector3d c;
    for (int i = 0; i < 3; ++i)
      c[i] = (rotation(i, 0) * w[0] + rotation(i, 1) * w[1]) + rotation(i, 2) * w[2] +
             translation[i];
    return c;
  }
  Vector2d project_point(const Vector3d& c) const {  // splat3d.hpp:48-51
    return {focal * c[0] / c[2] + principal_point[0], focal * c[1] / c[2] + principal_point[1]};
  }
  // Camera::validate, splat3d.cpp:27-37
  void validate() const {
    bool finite = translation.allFinite();
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) finite = finite && std::isfinite(rotation(i, j));
    if (!finite) throw std::domain_error("Camera: non-finite transform");
    double worst = 0.0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double d = 0.0;
        for (int k = 0; k < 3; ++k) d += rotation(i, k) * rotation(j, k);
        worst = std::fmax(worst, std::fabs(d - (i == j ? 1.0 : 0.0)));
      }
    if (worst > 1e-9) throw std::domain_error("Camera.rotation: not orthonormal within 1e-9");
    if (!(focal > 0.0)) throw std::domain_error("Camera.focal: must be > 0");
    if (width <= 0 || height <= 0) throw std::domain_error("Camera: bad image size");
  }
  isg_camera to_isg() const {
    isg_camera c{};
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) c.R[3 * i + j] = (float)rotation(i, j);
    for (int i = 0; i < 3; ++i) c.t[i] = (float)translation[i];
    c.focal = (float)focal;
    c.cx = (float)principal_point[0];
    c.cy = (float)principal_point[1];
    c.width = width;
    c.height = height;
    return c;
  }
};

struct ProjectedIso {
  Vector2d mu2d;
  double sigma2d;
  double depth;
};

// project_iso, splat3d.cpp:59-64 (host-side helper, FP64, identical arithmetic)
inline std::optional<ProjectedIso> project_iso(const IsoSplat3D& s, const Camera& cam) {
  s.validate();
  const Vector3d c = cam.to_camera(s.mu);
  if (!(c[2] > kNearPlane)) return std::nullopt;
  return ProjectedIso{cam.project_point(c), s.sigma * cam.focal / c[2], c[2]};
}

// composite, splat3d.cpp:76-87
inline Vector3d composite(std::span<const std::pair<Vector3d, double>> front_to_back) {
  Vector3d color{0.0, 0.0, 0.0};
  double T = 1.0;
  for (const auto& [c, a] : front_to_back) {
    if (!(a >= 0.0 && a <= 1.0)) throw std::domain_error("composite: alpha outside [0,1]");
    for (int i = 0; i < 3; ++i) color[i] += T * a * c[i];
    T *= 1.0 - a;
  }
  return color;
}

struct RenderOptions {
  Vector3d background{0.0, 0.0, 0.0};
  int threads = 1;       // accepted for source compatibility; the GPU ignores it
  // early termination on transmittance: the default 0 is the reference's semantics (every
  // covering splat composited, splat3d.cpp:134-141); training opts in (e.g. 1e-5)
  double t_min = 0.0;
};

// image.hpp:11-31: row-major, interleaved channels, FP64
struct ImageGrid {
  int width = 0, height = 0, channels = 1;
  std::vector<double> data;
  ImageGrid() = default;
  ImageGrid(int w, int h, int c, double fill = 0.0)
      : width(w), height(h), channels(c), data((size_t)w * h * c, fill) {}
  double& at(int x, int y, int c) { return data[((size_t)y * width + x) * channels + c]; }
  double at(int x, int y, int c) const { return data[((size_t)y * width + x) * channels + c]; }
  std::size_t value_count() const { return data.size(); }
};

namespace detail {
inline void check(isg_status s, const isg_ctx* ctx) {
  if (s == ISG_OK) return;
  std::string msg = ctx ? isg_last_error(ctx) : "";
  if (msg.empty()) msg = isg_status_string(s);
  if (s == ISG_E_DOMAIN) throw std::domain_error(msg);
  if (s == ISG_E_ARG) throw std::invalid_argument(msg);
  throw std::runtime_error(std::string("isg: ") + isg_status_string(s) + ": " + msg);
}

struct CtxDeleter {
  void operator()(isg_ctx* c) const { isg_destroy(c); }
};
using CtxPtr = std::unique_ptr<isg_ctx, CtxDeleter>;

inline CtxPtr make_ctx(int device = 0) {
  isg_ctx* c = nullptr;
  check(isg_create(device, 0, 0, 0, &c), nullptr);
  return CtxPtr(c);
}

// AoS FP64 (reference layout) -> SoA FP32 float4 pairs (device layout)
inline void to_soa(std::span<const IsoSplat3D> splats, std::vector<float>& ms,
                   std::vector<float>& co) {
  ms.resize(4 * splats.size());
  co.resize(4 * splats.size());
  for (std::size_t i = 0; i < splats.size(); ++i) {
    const IsoSplat3D& s = splats[i];
    ms[4 * i + 0] = (float)s.mu[0];
    ms[4 * i + 1] = (float)s.mu[1];
    ms[4 * i + 2] = (float)s.mu[2];
    ms[4 * i + 3] = (float)s.sigma;
    co[4 * i + 0] = (float)s.color[0];
    co[4 * i + 1] = (float)s.color[1];
    co[4 * i + 2] = (float)s.color[2];
    co[4 * i + 3] = (float)s.opacity;
  }
}
}  // namespace detail

// render(iso), splat3d.hpp:96-97 / splat3d.cpp:173-194, on the GPU.
inline ImageGrid render(std::span<const IsoSplat3D> splats, const Camera& camera,
                        const RenderOptions& options = {}) {
  camera.validate();
  for (const auto& s : splats) s.validate();
  auto ctx = detail::make_ctx();
  std::vector<float> ms, co;
  detail::to_soa(splats, ms, co);
  detail::check(isg_set_scene(ctx.get(), (int64_t)splats.size(), ms.data(), co.data()), ctx.get());
  const isg_camera cam = camera.to_isg();
  const float bg[3] = {(float)options.background[0], (float)options.background[1],
                       (float)options.background[2]};
  std::vector<float> img((size_t)camera.width * camera.height * 3);
  detail::check(isg_render(ctx.get(), &cam, bg, (float)options.t_min, img.data()), ctx.get());
  ImageGrid out(camera.width, camera.height, 3);
  for (std::size_t i = 0; i < img.size(); ++i) out.data[i] = img[i];
  return out;
}

struct AdamConfig {
  double lr_mu = 1e-3, lr_sigma = 5e-3, lr_color = 1e-2, lr_opacity = 1e-2;
  double beta1 = 0.9, beta2 = 0.999, eps = 1e-15;
};

// Training on one device: scene resident in HBM, L2 loss + backward per view, Adam step
// (the optimizer slot of update_step, optimize.cpp:78-108).
class Trainer {
 public:
  explicit Trainer(std::span<const IsoSplat3D> splats, int device = 0)
      : ctx_(detail::make_ctx(device)), n_(splats.size()) {
    for (const auto& s : splats) s.validate();
    std::vector<float> ms, co;
    detail::to_soa(splats, ms, co);
    detail::check(isg_set_scene(ctx_.get(), (int64_t)n_, ms.data(), co.data()), ctx_.get());
  }
  // weight * mse(render, target) (image.cpp:50-58); gradients accumulate until adam_step.
  double loss_backward(const Camera& camera, const ImageGrid& target,
                       const RenderOptions& options = {}, double weight = 1.0) {
    camera.validate();
    if (target.width != camera.width || target.height != camera.height || target.channels != 3)
      throw std::domain_error("loss_backward: target shape does not match the camera");
    std::vector<float> t(target.data.begin(), target.data.end());
    const isg_camera cam = camera.to_isg();
    const float bg[3] = {(float)options.background[0], (float)options.background[1],
                         (float)options.background[2]};
    double loss = 0.0;
    detail::check(isg_loss_backward(ctx_.get(), &cam, bg, (float)options.t_min, t.data(),
                                    (float)weight, &loss),
                  ctx_.get());
    return loss;
  }
  // n x 8 gradients: dmu.xyz dsigma drgb dopacity
  std::vector<float> gradients() {
    std::vector<float> g(8 * n_);
    detail::check(isg_get_grads(ctx_.get(), g.data()), ctx_.get());
    return g;
  }
  void adam_step(const AdamConfig& c = {}) {
    const float lr[4] = {(float)c.lr_mu, (float)c.lr_sigma, (float)c.lr_color,
                         (float)c.lr_opacity};
    detail::check(isg_adam_step(ctx_.get(), lr, (float)c.beta1, (float)c.beta2, (float)c.eps),
                  ctx_.get());
  }
  std::vector<IsoSplat3D> splats() {
    std::vector<float> ms(4 * n_), co(4 * n_);
    detail::check(isg_get_scene(ctx_.get(), ms.data(), co.data()), ctx_.get());
    std::vector<IsoSplat3D> out(n_);
    for (std::size_t i = 0; i < n_; ++i) {
      out[i].mu = {ms[4 * i], ms[4 * i + 1], ms[4 * i + 2]};
      out[i].sigma = ms[4 * i + 3];
      out[i].color = {co[4 * i], co[4 * i + 1], co[4 * i + 2]};
      out[i].opacity = co[4 * i + 3];
    }
    return out;
  }
  isg_ctx* handle() { return ctx_.get(); }

 private:
  detail::CtxPtr ctx_;
  std::size_t n_;
};

}  // namespace isosplat

// Exercises the C++ drop-in (paper_2403_14244_b200/csrc/isosplat_b200.hpp) exactly the way the
// reference's own caller does (tools/isosplat_main.cpp:357-398: build splats + camera, call
// isosplat::render, read ImageGrid::at), so reference caller code compiles unchanged.
//   test_dropin validate   host-only checks (no GPU needed)
//   test_dropin render     3-splat fixture on the GPU vs known answers
//   test_dropin train      Trainer: loss decreases over Adam steps
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "isosplat_b200.hpp"

using namespace isosplat;

static std::vector<IsoSplat3D> three_splats() {  // proj/tools/make_fixtures.py:73-78
  std::vector<IsoSplat3D> s(3);
  s[0].mu = {0.0, 0.0, 2.0};   s[0].sigma = 0.25; s[0].color = {1.0, 0.2, 0.1}; s[0].opacity = 0.5;
  s[1].mu = {0.35, -0.2, 3.0}; s[1].sigma = 0.45; s[1].color = {0.2, 0.9, 0.3}; s[1].opacity = 0.5;
  s[2].mu = {-0.3, 0.25, 4.0}; s[2].sigma = 0.9;  s[2].color = {0.1, 0.3, 1.0}; s[2].opacity = 1.0;
  return s;
}

static Camera camera32() {  // proj/data/camera_32.json
  Camera c;
  c.focal = 32;
  c.principal_point = {16, 16};
  c.width = c.height = 32;
  return c;
}

static int fail(const char* what) {
  std::printf("FAIL %s\n", what);
  return 1;
}

int main(int argc, char** argv) {
  const char* mode = argc > 1 ? argv[1] : "validate";
  if (!std::strcmp(mode, "validate")) {
    static_assert(IsoSplat3D::geometric_dof == 4);
    auto s = three_splats();
    s[1].sigma = -1.0;
    try {
      render(s, camera32());
      return fail("invalid sigma accepted");
    } catch (const std::domain_error& e) {
      if (std::strcmp(e.what(), "IsoSplat3D.sigma: must be positive and finite"))
        return fail(e.what());
    }
    Camera bad = camera32();
    bad.rotation(0, 0) = 1.5;
    try {
      render(three_splats(), bad);
      return fail("bad camera accepted");
    } catch (const std::domain_error& e) {
      if (std::strcmp(e.what(), "Camera.rotation: not orthonormal within 1e-9")) return fail(e.what());
    }
    const std::pair<Vector3d, double> list[3] = {
        {{1, 1, 1}, 0.5}, {{0.5, 0.5, 0.5}, 0.5}, {{0.25, 0.25, 0.25}, 1.0}};
    if (composite(list)[0] != 0.6875) return fail("composite 0.6875");
    const auto p = project_iso(three_splats()[1], camera32());
    if (!p || std::fabs(p->sigma2d - 4.8) > 1e-12) return fail("project_iso");
    std::printf("OK validate\n");
    return 0;
  }
  if (!std::strcmp(mode, "render")) {
    RenderOptions opt;
    opt.t_min = 0.0;
    const ImageGrid img = render(three_splats(), camera32(), opt);
    const struct { int x, y; double r, g, b; } known[] = {
        {15, 15, 0.539598543904, 0.293501319677, 0.419031703075},
        {16, 16, 0.540942539951, 0.302246395001, 0.405764169491},
        {19, 13, 0.255596227004, 0.451627307644, 0.287956021327},
        {13, 18, 0.308465363202, 0.292865519624, 0.770573717758}};
    for (const auto& k : known) {
      const double d = std::fmax(std::fabs(img.at(k.x, k.y, 0) - k.r),
                                 std::fmax(std::fabs(img.at(k.x, k.y, 1) - k.g),
                                           std::fabs(img.at(k.x, k.y, 2) - k.b)));
      if (d > 1e-4) return fail("pixel value");
    }
    std::printf("OK render\n");
    return 0;
  }
  if (!std::strcmp(mode, "train")) {
    auto target_scene = three_splats();
    RenderOptions opt;
    const ImageGrid target = render(target_scene, camera32(), opt);
    auto init = three_splats();
    for (auto& s : init) {
      s.mu[0] += 0.05;
      s.color[1] = 0.5;
    }
    Trainer tr(init);
    double first = 0, last = 0;
    for (int it = 0; it < 200; ++it) {
      last = tr.loss_backward(camera32(), target, opt);
      if (it == 0) first = last;
      AdamConfig c;
      c.lr_mu = 2e-3;
      tr.adam_step(c);
    }
    std::printf("loss %.6g -> %.6g\n", first, last);
    if (!(last < 0.5 * first)) return fail("loss did not decrease");
    std::printf("OK train\n");
    return 0;
  }
  return fail("unknown mode");
}

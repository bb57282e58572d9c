// Exercises the C++ drop-in (paper_2403_14244_b200/csrc/isosplat_b200.hpp) exactly the way the
// reference's own caller does (tools/isosplat_main.cpp:357-398: build splats + camera, call
// isosplat::render, read ImageGrid::at), so reference caller code compiles unchanged.
//   test_dropin validate   host-only checks (no GPU needed)
//   test_dropin render     3-splat fixture on the GPU vs known answers
//   test_dropin train      Trainer: loss decreases over Adam steps
//   test_dropin io DIR     ISPL binary/JSON + camera JSON round trips (host only)
//   test_dropin render3d SCENE CAMERA OUT.png   the reference's run_render3d flow
//                          (tools/isosplat_main.cpp:357-398) on the B200 path
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <stdexcept>
#include <vector>

#include "isosplat_b200.hpp"
#include "isosplat_io.hpp"

using namespace isosplat;

constexpr int kExitBadInput = 2;  // tools/isosplat_main.cpp:30

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
  if (!std::strcmp(mode, "io") && argc > 2) {
    const std::string dir = argv[2];
    ParticleSet set;
    set.iso3d = three_splats();
    set.metadata_json = "{\"name\":\"three_splats\"}";
    save_particles(dir + "/cpp_scene.ispl", set, false);
    save_particles(dir + "/cpp_scene.json", set, true);
    for (const char* f : {"/cpp_scene.ispl", "/cpp_scene.json"}) {
      const ParticleSet back = load_particles(dir + f);
      if (back.count() != 3) return fail("round trip count");
      for (int i = 0; i < 3; ++i)
        if (back.iso3d[i].mu[0] != set.iso3d[i].mu[0] || back.iso3d[i].sigma != set.iso3d[i].sigma ||
            back.iso3d[i].color[2] != set.iso3d[i].color[2] || back.iso3d[i].opacity != set.iso3d[i].opacity)
          return fail("round trip values");
    }
    std::ofstream(dir + "/cpp_camera.json")
        << "{\"rotation\": [[1,0,0],[0,1,0],[0,0,1]], \"translation\": [0,0,0], \"focal\": 32,"
           " \"principal_point\": [16, 16], \"image_size\": [32, 32]}\n";
    const Camera c = load_camera(dir + "/cpp_camera.json");
    if (c.focal != 32 || c.width != 32 || c.principal_point[1] != 16) return fail("camera");
    std::ofstream(dir + "/bad_quat.json")
        << "{\"quaternion\": [1, 0.1, 0, 0], \"translation\": [0,0,0], \"focal\": 1,"
           " \"principal_point\": [0, 0], \"image_size\": [4, 4]}\n";
    try {
      load_camera(dir + "/bad_quat.json");
      return fail("bad quaternion accepted");
    } catch (const std::runtime_error& e) {
      if (std::strcmp(e.what(), "camera: quaternion norm must be 1 within 1e-9")) return fail(e.what());
    }
    // files written by the Python side (tests/test_scene_io.py), if present
    for (const char* f : {"/py_scene.ispl", "/py_scene.json"}) {
      std::ifstream probe(dir + f);
      if (!probe) continue;
      const ParticleSet py = load_particles(dir + f);
      if (py.count() != 3 || py.iso3d[2].sigma != 0.9) return fail("python-written scene");
    }
    std::printf("OK io\n");
    return 0;
  }
  if (!std::strcmp(mode, "render3d") && argc > 4) {
    // run_render3d, tools/isosplat_main.cpp:357-398
    ParticleSet scene;
    Camera cam;
    try {
      scene = load_particles(argv[2]);
      cam = load_camera(argv[3]);
      if (scene.dimension != 3) throw std::runtime_error("scene file must hold 3D splats (dimension=3)");
    } catch (const std::exception& e) {
      std::cerr << "error: " << e.what() << "\n";
      return kExitBadInput;
    }
    RenderOptions options;
    ImageGrid img;
    try {
      img = render(std::span<const IsoSplat3D>(scene.iso3d), cam, options);
    } catch (const std::domain_error& e) {
      std::cerr << "error: " << e.what() << "\n";
      return kExitBadInput;
    }
    write_png(argv[4], img);
    std::cout << "rendered " << scene.count() << " splats to " << argv[4] << "\n";
    return 0;
  }
  return fail("unknown mode");
}

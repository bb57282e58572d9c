#!/usr/bin/env python3
"""Regenerate tests/golden/*.npz from the REFERENCE's own code (oracle/_ref, i.e.
/root/reference/proj/src/splat3d.cpp + image.cpp compiled by oracle/build_ref.sh).

Run in the build container (where /root/reference exists):
    bash oracle/build_ref.sh && python tests/golden/make_golden.py
The fixtures are small and committed, so the GPU box (no /root/reference) can use them.

  three_splats.npz      the shipped fixture inputs (proj/tools/make_fixtures.py:73-78,
                        proj/data/camera_32.json) and the reference render
  reference_scenes.npz  8 randomised scenes (<= 48x40 px, <= 120 splats, rotated cameras,
                        non-zero backgrounds, splats behind the camera / off screen, opacity 1)
                        and the reference renders
  reference_scenes_large.npz
                        3 larger scenes of the same kind (96x200 .. 256x144 px, 1.5K-6K splats:
                        many 16x16 tiles, long per-tile lists, opacity-1 occluders) and the
                        reference renders
  image_loss.npz        image pairs (11x11 up to 64x48, equal pixels, saturated values) with the
                        reference's loss(), l1_term(), ssim() and ssim_gradient_wrt_second()
                        (proj/src/loss.cpp:112-190) for several lambdas
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle as O  # noqa: E402
from paper_2403_14244_b200.isg import Camera  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    cam32 = Camera(np.eye(3), np.zeros(3), 32.0, (16.0, 16.0), 32, 32)
    three = np.array([[0.0, 0.0, 2.0, 0.25, 1.0, 0.2, 0.1, 0.5],
                      [0.35, -0.2, 3.0, 0.45, 0.2, 0.9, 0.3, 0.5],
                      [-0.3, 0.25, 4.0, 0.9, 0.1, 0.3, 1.0, 1.0]])
    np.savez_compressed(OUT / "three_splats.npz", splats=three, image=O.ref_render(three, cam32),
                        composite=O.ref_composite([[1, 1, 1, .5], [.5, .5, .5, .5],
                                                   [.25, .25, .25, 1.0]]))
    rng = np.random.default_rng(20240901)
    scenes = {}
    for k in range(8):
        W, H = int(rng.integers(8, 49)), int(rng.integers(8, 41))
        n = int(rng.integers(1, 121))
        sp, cam, bg = random_scene(rng, W, H, n, k)
        scenes[f"s{k}_splats"] = sp
        scenes[f"s{k}_cam"] = np.concatenate([cam.rotation.reshape(9), cam.translation,
                                              [cam.focal, *cam.principal_point, W, H]])
        scenes[f"s{k}_bg"] = bg
        scenes[f"s{k}_image"] = O.ref_render(sp, cam, bg, threads=8)
    np.savez_compressed(OUT / "reference_scenes.npz", **scenes)
    rng = np.random.default_rng(2403)
    large = {}
    for k, (W, H, n) in enumerate(LARGE_CASES):
        sp, cam, bg = random_scene(rng, W, H, n, k + 1, s2d_max=14.0)
        large[f"s{k}_splats"] = sp
        large[f"s{k}_cam"] = np.concatenate([cam.rotation.reshape(9), cam.translation,
                                             [cam.focal, *cam.principal_point, W, H]])
        large[f"s{k}_bg"] = bg
        large[f"s{k}_image"] = O.ref_render(sp, cam, bg, threads=8)
    np.savez_compressed(OUT / "reference_scenes_large.npz", **large)
    image_loss_fixture()
    print("golden fixtures written:", sorted(p.name for p in OUT.glob("*.npz")))


LARGE_CASES = [(160, 120, 3000), (256, 144, 6000), (96, 200, 1500)]


def random_scene(rng, W, H, n, k, s2d_max=10.0):
    """A randomised scene: rotated + translated camera, shifted principal point, splats in
    front of, at and behind the near plane, some off screen, ~10% opacity exactly 1, a
    non-zero background for odd k."""
    th = rng.uniform(-0.3, 0.3, 3)
    cx, sx = np.cos(th), np.sin(th)
    Rx = np.array([[1, 0, 0], [0, cx[0], -sx[0]], [0, sx[0], cx[0]]])
    Ry = np.array([[cx[1], 0, sx[1]], [0, 1, 0], [-sx[1], 0, cx[1]]])
    Rz = np.array([[cx[2], -sx[2], 0], [sx[2], cx[2], 0], [0, 0, 1]])
    R = Rz @ Ry @ Rx
    t = rng.uniform(-0.2, 0.2, 3)
    f = float(rng.uniform(0.7, 1.5) * max(W, H))
    cam = Camera(R, t, f, (W / 2 + rng.uniform(-2, 2), H / 2 + rng.uniform(-2, 2)), W, H)
    z = rng.uniform(-0.5, 6.0, n)  # some behind the camera / at the near plane
    u = rng.uniform(-0.2 * W, 1.2 * W, n)
    v = rng.uniform(-0.2 * H, 1.2 * H, n)
    s2d = np.exp(rng.uniform(np.log(0.3), np.log(s2d_max), n))
    pc = np.stack([(u - W / 2) * np.abs(z) / f, (v - H / 2) * np.abs(z) / f, z], 1)
    world = (pc - t) @ R  # R^T (p - t)
    op = rng.uniform(0.0, 1.0, n)
    op[rng.random(n) < 0.1] = 1.0
    sp = np.concatenate([world, (s2d * np.maximum(np.abs(z), 0.1) / f)[:, None],
                         rng.uniform(0, 1, (n, 3)), op[:, None]], 1)
    bg = rng.uniform(0, 1, 3) if k % 2 else np.zeros(3)
    return sp, cam, bg


IMAGE_LOSS_CASES = [(11, 11, 0.2), (17, 13, 0.2), (40, 24, 0.0), (33, 29, 1.0), (64, 48, 0.5)]


def image_loss_fixture():
    rng = np.random.default_rng(14244)
    out = {}
    for k, (W, H, lam) in enumerate(IMAGE_LOSS_CASES):
        f = rng.random((H, W, 3))
        fhat = np.clip(f + 0.15 * rng.standard_normal(f.shape), 0.0, 1.0)  # saturated values
        eq = rng.random((H, W)) < 0.1
        fhat[eq] = f[eq]  # equal pixels: L1 subgradient 0
        loss, l1, ssim, g = O.ref_image_loss(f, fhat, lam, grad=True)
        out[f"c{k}_f"], out[f"c{k}_fhat"] = f, fhat
        out[f"c{k}_meta"] = np.array([W, H, lam, loss, l1, ssim])
        out[f"c{k}_dssim"] = g if g is not None else np.zeros(0)
    np.savez_compressed(OUT / "image_loss.npz", **out)


def load_image_loss():
    g = np.load(OUT / "image_loss.npz")
    cases = []
    for k in range(len(IMAGE_LOSS_CASES)):
        W, H, lam, loss, l1, ssim = g[f"c{k}_meta"]
        cases.append(dict(f=g[f"c{k}_f"], fhat=g[f"c{k}_fhat"], lam=float(lam), loss=float(loss),
                          l1=float(l1), ssim=float(ssim), dssim=g[f"c{k}_dssim"]))
    return cases


def load_scenes(name="reference_scenes.npz"):
    """[(splats (n, 8) FP64, Camera, background, the reference's render)] of a fixture file."""
    g = np.load(OUT / name)
    out = []
    for k in range(len([f for f in g.files if f.endswith("_image")])):
        c = g[f"s{k}_cam"]
        cam = Camera(c[:9].reshape(3, 3), c[9:12], float(c[12]), (float(c[13]), float(c[14])),
                     int(c[15]), int(c[16]))
        out.append((g[f"s{k}_splats"], cam, g[f"s{k}_bg"], g[f"s{k}_image"]))
    return out


if __name__ == "__main__":
    main()

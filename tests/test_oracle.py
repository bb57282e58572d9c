"""CPU tests of the oracle itself (no GPU): pinned against the reference's known answers
(SPEC.md operation examples / acceptance criteria), the reference's brute-force renderer, finite
differences, and torch.optim.Adam.  When oracle/_ref (the reference's own splat3d.cpp compiled
here) is present, the FP64 restatement is also checked against it bit for bit."""
import hashlib

import numpy as np
import pytest

import oracle as O
from paper_2403_14244_b200.isg import Camera

CAM32 = Camera(np.eye(3), np.zeros(3), 32.0, (16.0, 16.0), 32, 32)  # proj/data/camera_32.json
THREE = np.array([  # proj/tools/make_fixtures.py:73-78
    [0.0, 0.0, 2.0, 0.25, 1.0, 0.2, 0.1, 0.5],
    [0.35, -0.2, 3.0, 0.45, 0.2, 0.9, 0.3, 0.5],
    [-0.3, 0.25, 4.0, 0.9, 0.1, 0.3, 1.0, 1.0],
])


def rand_scene(rng, n, W, H, f=None, zr=(2.0, 6.0), s2d=(0.5, 6.0)):
    f = f or float(max(W, H))
    z = rng.uniform(*zr, n)
    u = rng.uniform(-0.1 * W, 1.1 * W, n)
    v = rng.uniform(-0.1 * H, 1.1 * H, n)
    s = np.exp(rng.uniform(np.log(s2d[0]), np.log(s2d[1]), n))
    sp = np.stack([(u - W / 2) * z / f, (v - H / 2) * z / f, z, s * z / f,
                   rng.uniform(0, 1, n), rng.uniform(0, 1, n), rng.uniform(0, 1, n),
                   rng.uniform(0.05, 0.95, n)], 1)
    return sp, Camera(np.eye(3), np.zeros(3), f, (W / 2, H / 2), W, H)


# ---- known answers -----------------------------------------------------------------------
def test_composite_known_answer():
    # SPEC.md:452 / acceptance criterion 3: (1,.5),(.5,.5),(.25,1) -> 0.6875 exactly
    out = O.composite64([[1, 1, 1, .5], [.5, .5, .5, .5], [.25, .25, .25, 1.0]])
    assert np.all(out == 0.6875)
    # single splat -> c*alpha; alpha=1 in front -> c1
    assert np.allclose(O.composite64([[0.3, 0.6, 0.9, 0.5]]), [0.15, 0.3, 0.45])
    assert np.allclose(O.composite64([[0.3, 0.6, 0.9, 1.0], [1, 1, 1, 0.7]]), [0.3, 0.6, 0.9])
    with pytest.raises(ValueError):
        O.composite64([[1, 1, 1, 1.5]])


def test_project_iso_identities():
    # sigma=0.1 at z=f -> sigma_2d = 0.1; doubling z halves sigma_2d
    cam = Camera(np.eye(3), np.zeros(3), 50.0, (0, 0), 64, 64)
    p1 = O.project_iso64([0, 0, 50.0, 0.1, 0, 0, 0, 1], cam)
    p2 = O.project_iso64([0, 0, 100.0, 0.1, 0, 0, 0, 1], cam)
    assert p1[2] == pytest.approx(0.1, abs=1e-15)
    assert p2[2] == pytest.approx(0.05, abs=1e-15)
    assert O.project_iso64([0, 0, 1e-3, 0.1, 0, 0, 0, 1], cam) is None  # kNearPlane cull
    assert O.project_iso64([0, 0, -1.0, 0.1, 0, 0, 0, 1], cam) is None


def test_project_iso_roll_invariance():
    # SPEC.md:466 / criterion 4: sigma_2d invariant under camera roll about the optical axis
    rng = np.random.default_rng(3)
    for _ in range(20):
        th = rng.uniform(0, 2 * np.pi)
        R = np.array([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1]])
        s = [rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(2, 5), 0.3, 0, 0, 0, 1]
        a = O.project_iso64(s, Camera(np.eye(3), np.zeros(3), 40.0, (0, 0), 8, 8))
        b = O.project_iso64(s, Camera(R, np.zeros(3), 40.0, (0, 0), 8, 8))
        assert a[2] == pytest.approx(b[2], rel=1e-12)


def test_render_empty_is_background():
    img = O.render64(np.zeros((0, 8)), CAM32, bg=(0.1, 0.2, 0.3))
    assert np.all(img == np.array([0.1, 0.2, 0.3]))


def test_on_axis_alpha_one():
    cam = Camera(np.eye(3), np.zeros(3), 32.0, (16.5, 16.5), 33, 33)
    img = O.render64([[0, 0, 2.0, 0.2, 0.3, 0.6, 0.9, 1.0]], cam)
    assert np.allclose(img[16, 16], [0.3, 0.6, 0.9], atol=1e-15)


def test_three_splat_fixture_known_values():
    """SURVEY Appendix B (FP64 restatement of render on the shipped fixture inputs)."""
    img = O.render64(THREE, CAM32)
    assert img[15, 15] == pytest.approx([0.539598543904, 0.293501319677, 0.419031703075], abs=1e-12)
    assert img[16, 16] == pytest.approx([0.540942539951, 0.302246395001, 0.405764169491], abs=1e-12)
    assert img[13, 19] == pytest.approx([0.255596227004, 0.451627307644, 0.287956021327], abs=1e-12)
    assert img[18, 13] == pytest.approx([0.308465363202, 0.292865519624, 0.770573717758], abs=1e-12)
    assert img.sum() == pytest.approx(266.798504875079, abs=1e-9)
    assert int((img != 0).any(axis=2).sum()) == 1003
    q = np.floor(np.clip(img, 0, 1) * 255.0 + 0.5).astype(np.uint8)  # quantize8, png_io.hpp:17-21
    assert hashlib.sha256(q.tobytes()).hexdigest() == \
        "0395d81a958d41220a9beec27f43592499b76bba511589e1137b8032f75a1ae4"


def test_golden_fixture_file():
    """tests/golden/three_splats.npz (made by tests/golden/make_golden.py) still matches."""
    from pathlib import Path
    g = np.load(Path(__file__).parent / "golden" / "three_splats.npz")
    assert np.array_equal(O.render64(g["splats"], CAM32), g["image"])


def test_render_equals_brute_force():
    # SPEC.md:461,468 / criterion 3: <= 32x32, <= 100 splats, 1e-6 (here: exact)
    rng = np.random.default_rng(20240901)
    for trial in range(25):
        n = int(rng.integers(1, 101))
        sp, cam = rand_scene(rng, n, int(rng.integers(4, 33)), int(rng.integers(4, 33)))
        a = O.render64(sp, cam, threads=1 + trial % 3)
        b = O.brute_force64(sp, cam)
        assert np.abs(a - b).max() <= 1e-6


def test_render_thread_count_invariant():
    rng = np.random.default_rng(1)
    sp, cam = rand_scene(rng, 300, 64, 48)
    assert np.array_equal(O.render64(sp, cam, threads=1), O.render64(sp, cam, threads=5))


def test_mse():
    a = np.arange(12.0)
    b = a[::-1].copy()
    assert O.mse64(a, b) == pytest.approx(np.mean((a - b) ** 2), rel=1e-15)


# ---- FP32 tiled restatement vs FP64 literal ------------------------------------------------
@pytest.mark.parametrize("seed", range(5))
def test_fp32_tiled_matches_fp64(seed):
    rng = np.random.default_rng(100 + seed)
    sp, cam = rand_scene(rng, 400, 70, 45)
    ms = sp[:, :4].astype(np.float32)
    co = sp[:, 4:].astype(np.float32)
    img32 = O.render32(ms, co, cam, t_min=0.0)
    img64 = O.render64(np.concatenate([ms, co], 1).astype(np.float64), cam)
    assert np.abs(img32 - img64).max() <= 1e-4
    # early termination at t_min drops at most t_min * max(c, bg) per pixel
    img_t = O.render32(ms, co, cam, t_min=1e-5)
    assert np.abs(img_t - img64).max() <= 1e-4


def test_bins_properties():
    rng = np.random.default_rng(7)
    sp, cam = rand_scene(rng, 2000, 200, 120, s2d=(0.5, 30))
    ms = sp[:, :4].astype(np.float32)
    co = sp[:, 4:].astype(np.float32)
    keys, vals, ranges, nvis = O.bin32(ms, co, cam)
    assert np.all(np.diff(keys.astype(np.float64)) >= 0) or np.all(keys[1:] >= keys[:-1])
    tiles = (keys >> np.uint64(32)).astype(np.int64)
    for t in range(ranges.shape[0]):
        a, b = ranges[t]
        assert np.all(tiles[a:b] == t)
    # every (tile, splat) pair at most once; depth ties broken by index
    pair = tiles * (1 << 32) + vals
    assert np.unique(pair).size == pair.size
    z = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint64)
    same = (tiles[1:] == tiles[:-1]) & (z[1:] == z[:-1])
    assert np.all(vals[1:][same] > vals[:-1][same])
    # every pixel covered by a splat is in the splat's tile list (coverage completeness)
    H, W = cam.height, cam.width
    tx = (W + 15) // 16
    for i in rng.choice(ms.shape[0], 50, replace=False):
        p = O.project_iso64(np.concatenate([ms[i], co[i]]).astype(np.float64), cam)
        if p is None:
            continue
        ys, xs = np.mgrid[0:H, 0:W]
        inside = (xs + 0.5 - p[0]) ** 2 + (ys + 0.5 - p[1]) ** 2 <= 9 * p[2] ** 2 * (1 - 1e-6)
        need = set(((ys[inside] // 16) * tx + xs[inside] // 16).tolist())
        have = set(tiles[vals == i].tolist())
        assert need <= have


# ---- gradients -----------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(6))
def test_fp64_backward_matches_finite_differences(seed):
    """SPEC.md:570 convention (criterion 1): analytic vs central differences, rel <= 1e-4.
    Perturbations stay away from the 3-sigma cutoff (SPEC.md:213 precedent) by using
    h = 1e-7 and rejecting configurations whose loss is not smooth at that scale."""
    rng = np.random.default_rng(1000 + seed)
    W, H = 16, 12
    n = int(rng.integers(1, 6))
    sp, cam = rand_scene(rng, n, W, H, s2d=(1.0, 4.0))
    target = rng.uniform(0, 1, (H, W, 3))
    _, g = O.loss_grad64(sp, cam, target)
    h = 1e-7
    scale = np.abs(g).max() + 1e-12
    for i in range(n):
        for j in range(8):
            a = sp.copy()
            b = sp.copy()
            a[i, j] += h
            b[i, j] -= h
            fd = (O.loss_grad64(a, cam, target)[0] - O.loss_grad64(b, cam, target)[0]) / (2 * h)
            assert abs(fd - g[i, j]) <= 1e-4 * scale + 1e-9, (i, j, fd, g[i, j])


def test_fp32_backward_matches_fp64():
    rng = np.random.default_rng(42)
    sp, cam = rand_scene(rng, 80, 40, 30)
    target = rng.uniform(0, 1, (30, 40, 3))
    loss64, g64 = O.loss_grad64(sp, cam, target, bg=(0.2, 0.1, 0.0))
    loss32, g32 = O.loss_backward32(sp[:, :4].astype(np.float32), sp[:, 4:].astype(np.float32),
                                    cam, target.astype(np.float32), bg=(0.2, 0.1, 0.0), t_min=0.0)
    assert loss32 == pytest.approx(loss64, rel=1e-6)
    for sl in (slice(0, 3), slice(3, 4), slice(4, 7), slice(7, 8)):
        assert np.linalg.norm(g32[:, sl] - g64[:, sl]) <= 1e-4 * np.linalg.norm(g64[:, sl])


def test_fp32_backward_thread_invariant():
    rng = np.random.default_rng(5)
    sp, cam = rand_scene(rng, 300, 64, 64)
    ms, co = sp[:, :4].astype(np.float32), sp[:, 4:].astype(np.float32)
    t = rng.uniform(0, 1, (64, 64, 3)).astype(np.float32)
    _, a = O.loss_backward32(ms, co, cam, t, threads=1)
    _, b = O.loss_backward32(ms, co, cam, t, threads=7)
    assert np.array_equal(a, b)


# ---- Adam ----------------------------------------------------------------------------------
def test_adam_matches_torch():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(9)
    n = 50
    ms = np.concatenate([rng.normal(size=(n, 3)), rng.uniform(0.1, 1, (n, 1))], 1).astype(np.float32)
    co = np.concatenate([rng.uniform(0, 1, (n, 3)), rng.uniform(0.05, 0.95, (n, 1))], 1).astype(np.float32)
    lr = [1e-3, 5e-3, 1e-2, 2e-2]
    b1, b2, eps = 0.9, 0.999, 1e-8
    p_mu = torch.tensor(ms[:, :3], requires_grad=True)
    p_ls = torch.tensor(np.log(ms[:, 3]), requires_grad=True)
    p_c = torch.tensor(co[:, :3], requires_grad=True)
    p_lo = torch.tensor(np.log(co[:, 3] / (1 - co[:, 3])), requires_grad=True)
    opt = torch.optim.Adam([{"params": [p_mu], "lr": lr[0]}, {"params": [p_ls], "lr": lr[1]},
                            {"params": [p_c], "lr": lr[2]}, {"params": [p_lo], "lr": lr[3]}],
                           betas=(b1, b2), eps=eps)
    m = np.zeros((n, 8), np.float32)
    v = np.zeros((n, 8), np.float32)
    oms, oco = ms.copy(), co.copy()
    raw = O.raw_init32(oms, oco)
    for step in range(1, 6):
        g = rng.normal(size=(n, 8)).astype(np.float32)  # dL/d(mu, sigma, rgb, opacity)
        sig = torch.exp(p_ls.detach())
        op = torch.sigmoid(p_lo.detach())
        p_mu.grad = torch.tensor(g[:, :3])
        p_ls.grad = torch.tensor(g[:, 3]) * sig
        p_c.grad = torch.tensor(g[:, 4:7])
        p_lo.grad = torch.tensor(g[:, 7]) * op * (1 - op)
        opt.step()
        O.adam32(oms, oco, m, v, g, step, lr, b1, b2, eps, raw=raw)
        assert np.allclose(oms[:, :3], p_mu.detach().numpy(), atol=2e-6)
        assert np.allclose(raw[:, 0], p_ls.detach().numpy(), atol=2e-6)
        assert np.allclose(raw[:, 1], p_lo.detach().numpy(), atol=2e-6)
        assert np.allclose(np.log(oms[:, 3]), p_ls.detach().numpy(), atol=2e-6)
        assert np.allclose(oco[:, :3], p_c.detach().numpy(), atol=2e-6)
        assert np.allclose(oco[:, 3], torch.sigmoid(p_lo.detach()).numpy(), atol=2e-6)


def test_adam_skips_non_finite():
    ms = np.ones((3, 4), np.float32)
    co = np.full((3, 4), 0.5, np.float32)
    m = np.zeros((3, 8), np.float32)
    v = np.zeros((3, 8), np.float32)
    g = np.ones((3, 8), np.float32)
    g[1, 2] = np.nan
    before = ms.copy()
    assert O.adam32(ms, co, m, v, g, 1, [1e-2] * 4) == 1
    assert np.array_equal(ms[1], before[1]) and not np.array_equal(ms[0], before[0])


# ---- the reference's own code (oracle/_ref), when built ------------------------------------
ref = pytest.mark.skipif(not O.REF_LIB.exists(), reason="oracle/_ref not built (no /root/reference)")


@ref
def test_restatement_equals_reference_render():
    rng = np.random.default_rng(77)
    for trial in range(10):
        sp, cam = rand_scene(rng, int(rng.integers(1, 120)), 40, 30)
        a = O.render64(sp, cam)
        b = O.ref_render(sp, cam)
        assert np.abs(a - b).max() <= 1e-12
    assert np.array_equal(O.ref_render(THREE, CAM32), O.render64(THREE, CAM32))


@ref
def test_reference_composite_and_errors():
    assert np.all(O.ref_composite([[1, 1, 1, .5], [.5, .5, .5, .5], [.25, .25, .25, 1.0]]) == 0.6875)
    bad = THREE.copy()
    bad[1, 3] = -1.0
    with pytest.raises(ValueError, match="IsoSplat3D.sigma"):
        O.ref_render(bad, CAM32)


# ---- the synthetic workload, restated in the oracle ------------------------------------------
@pytest.mark.parametrize("n,W,H,seed", [(1000, 256, 256, 2403), (5000, 1920, 1080, 14244),
                                        (777, 3840, 2160, 5)])
def test_oracle_synth_scene_byte_equal_to_product(n, W, H, seed):
    """bench.py's CPU arms build the isg-synth v1 scene and cameras from the oracle alone (no
    libisg in that process); they must be the product's bytes (isg_synth_scene is host code,
    callable without a GPU)."""
    from paper_2403_14244_b200 import isg

    ms, co = O.synth_scene(n, W, H, seed)
    ms2, co2 = isg.synth_scene(n, W, H, seed)
    assert ms.tobytes() == ms2.tobytes() and co.tobytes() == co2.tobytes()
    for views in (1, 8):
        for k in range(views):
            a = O.synth_camera(W, H, k, views)
            b = isg.Camera.synthetic(W, H, k, views)
            assert np.array_equal(a.rotation, b.rotation)
            assert np.array_equal(a.translation, b.translation)
            assert (a.focal, a.principal_point, a.width, a.height) == \
                (b.focal, b.principal_point, b.width, b.height)


# ---- the reference's own renders, committed (tests/golden/make_golden.py) ------------------
def _golden(name):
    import sys
    sys.path.insert(0, str(O.ROOT / "tests" / "golden"))
    from make_golden import load_scenes
    return load_scenes(name)


@pytest.mark.parametrize("name", ["reference_scenes.npz", "reference_scenes_large.npz"])
def test_restatement_equals_committed_reference_renders(name):
    """The FP64 restatement reproduces the reference's own render() (oracle/_ref output
    committed as fixtures) on rotated + translated cameras, shifted principal points, splats
    behind / at the near plane and off screen, opacity exactly 1 and non-zero backgrounds; the
    FP32 tiled oracle (the GPU's bit-level model) at t_min = 0 lies within the north star's
    1e-4 image tolerance of it (FP32 accumulation over up to ~1K-entry lists: <= 3e-5 here)."""
    for sp, cam, bg, img in _golden(name):
        assert np.abs(O.render64(sp, cam, bg) - img).max() <= 1e-12
        ms, co = sp[:, :4].astype(np.float32), sp[:, 4:].astype(np.float32)
        assert np.abs(O.render32(ms, co, cam, bg=bg, t_min=0.0) - img).max() <= 1e-4
        if sp.shape[0] <= 120:
            assert np.abs(O.brute_force64(sp, cam, bg) - img).max() <= 1e-12


@ref
@pytest.mark.parametrize("seed", range(6))
def test_restatement_equals_reference_render_random_cameras(seed):
    """Live against the reference's render(): random rotations, translations, focal lengths,
    principal points, backgrounds, opacity exactly 1, splats behind the camera."""
    import sys
    sys.path.insert(0, str(O.ROOT / "tests" / "golden"))
    from make_golden import random_scene
    rng = np.random.default_rng(1000 + seed)
    W, H = int(rng.integers(8, 97)), int(rng.integers(8, 81))
    sp, cam, bg = random_scene(rng, W, H, int(rng.integers(1, 400)), seed)
    assert np.abs(O.render64(sp, cam, bg) - O.ref_render(sp, cam, bg, threads=4)).max() <= 1e-12

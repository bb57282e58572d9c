"""GPU parity tests: the CUDA path (through the C-ABI) against the CPU oracle.

Bars (BASELINE.json north_star): tile keys, sort order and per-tile ranges bit-exact; images
max|diff| <= 1e-4; gradients relative <= 1e-3 per parameter group (||dg||/||g||) and
elementwise |dg| <= 1e-3 * max|g|.
"""
import zlib

import numpy as np
import pytest

import oracle as O
from paper_2403_14244_b200 import isg

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4
T_MIN = 1e-5  # the training configs' early-termination threshold (full-size cases)
GRAD_TOL = 1e-3
GROUPS = {"mu": slice(0, 3), "sigma": slice(3, 4), "rgb": slice(4, 7), "opacity": slice(7, 8)}


@pytest.fixture(scope="module")
def rend():
    r = isg.Renderer(0)
    yield r
    r.close()


def random_scene(rng, n, W, H, sigma2d=(0.5, 8.0), depth=(2.0, 10.0), f=None):
    f = f or 1000.0 * W / 1920.0
    z = rng.uniform(*depth, n)
    u = rng.uniform(-0.1 * W, 1.1 * W, n)
    v = rng.uniform(-0.1 * H, 1.1 * H, n)
    s2d = np.exp(rng.uniform(np.log(sigma2d[0]), np.log(sigma2d[1]), n))
    ms = np.stack([(u - W / 2) * z / f, (v - H / 2) * z / f, z, s2d * np.maximum(np.abs(z), 0.05) / f], 1).astype(np.float32)
    co = np.concatenate([rng.uniform(0, 1, (n, 3)), rng.uniform(0.05, 0.95, (n, 1))], 1)
    return ms, co.astype(np.float32), isg.Camera(np.eye(3), np.zeros(3), f, (W / 2, H / 2), W, H)


def check_bins(r, ms, co, cam):
    keys, vals, ranges = r.debug_bins()
    k2, v2, r2, nvis = O.bin32(ms, co, cam)
    assert keys.shape == k2.shape, (keys.shape, k2.shape)
    assert np.array_equal(keys, k2), "tile keys differ"
    assert np.array_equal(vals, v2), "sort order differs"
    assert np.array_equal(ranges, r2), "tile ranges differ"
    assert r.stats()["n_visible"] == nvis
    return keys


CASES = [
    ("tiny", 40, 64, 48, {}),
    ("synth256", 10000, 256, 256, {}),
    ("ragged", 3000, 203, 117, {}),  # partial edge tiles
    ("large_splats", 300, 256, 192, {"sigma2d": (10.0, 60.0)}),
    ("tiny_splats", 5000, 128, 128, {"sigma2d": (0.05, 0.5)}),
    ("near_plane", 2000, 128, 96, {"depth": (-0.5, 3.0)}),
]


@pytest.mark.parametrize("name,n,W,H,kw", CASES, ids=[c[0] for c in CASES])
def test_bins_and_render(rend, name, n, W, H, kw):
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    ms, co, cam = random_scene(rng, n, W, H, **kw)
    rend.set_scene(ms, co)
    for t_min in (0.0, 1e-5, 1e-2):
        opts = isg.RenderOptions(t_min=t_min)
        img = rend.render(cam, opts)
        check_bins(rend, ms, co, cam)
        ref, tl, npr, _ = O.render32(ms, co, cam, t_min=t_min, want_state=True)
        gtl, gnp = rend.debug_pixel_state(W, H)
        same = gnp == npr
        # Where transmittance lands within one rounding of t_min, ex2.approx (GPU) and libm
        # expf (oracle) may stop one entry apart; that entry is worth at most ~t_min * max|c|.
        # Everywhere else the images agree to IMG_TOL.
        assert np.mean(same) > 0.99
        assert np.abs(img - ref)[same].max(initial=0.0) <= IMG_TOL
        assert np.abs(img - ref).max() <= IMG_TOL + 2.0 * t_min


def test_synthetic_scene_bins(rend):
    W, H = 320, 180
    ms, co = isg.synth_scene(20000, W, H, seed=2403)
    cam = isg.Camera.synthetic(W, H)
    rend.set_scene(ms, co)
    img = rend.render(cam)
    check_bins(rend, ms, co, cam)
    assert np.abs(img - O.render32(ms, co, cam)).max() <= IMG_TOL


def test_depth_ties_break_by_index(rend):
    """Equal depths keep input order (stable_sort, splat3d.cpp:164-169)."""
    W = H = 64
    n = 200
    rng = np.random.default_rng(5)
    ms, co, cam = random_scene(rng, n, W, H)
    ms[:, 2] = np.float32(4.0)  # every splat at the same depth
    ms[:, 0:2] = ms[:, 0:2] * 0.3
    rend.set_scene(ms, co)
    img = rend.render(cam, isg.RenderOptions(t_min=0.0))
    keys = check_bins(rend, ms, co, cam)
    assert len(keys) > n
    assert np.abs(img - O.render32(ms, co, cam, t_min=0.0)).max() <= IMG_TOL


def test_rotated_cameras(rend):
    W, H = 192, 128
    ms, co = isg.synth_scene(8000, W, H, seed=7)
    rend.set_scene(ms, co)
    for k in range(8):
        cam = isg.Camera.synthetic(W, H, k, 8)
        img = rend.render(cam)
        check_bins(rend, ms, co, cam)
        assert np.abs(img - O.render32(ms, co, cam)).max() <= IMG_TOL


def test_background_and_empty(rend):
    cam = isg.Camera(np.eye(3), np.zeros(3), 32.0, (16, 16), 32, 32)
    rend.set_scene(np.zeros((0, 4), np.float32), np.zeros((0, 4), np.float32))
    img = rend.render(cam, isg.RenderOptions(background=(0.25, 0.5, 1.0)))
    assert np.array_equal(img, np.broadcast_to(np.float32([0.25, 0.5, 1.0]), img.shape))


def test_three_splat_fixture(rend):
    """SURVEY Appendix B values (FP64 restatement of the reference on the shipped fixture
    inputs, proj/tools/make_fixtures.py:73-78 + proj/data/camera_32.json)."""
    sp = np.array([[0, 0, 2, .25, 1, .2, .1, .5], [.35, -.2, 3, .45, .2, .9, .3, .5],
                   [-.3, .25, 4, .9, .1, .3, 1, 1]])
    cam = isg.Camera(np.eye(3), np.zeros(3), 32.0, (16, 16), 32, 32)
    img = isg.render(sp, cam, isg.RenderOptions(t_min=0.0))
    known = {(15, 15): [0.539598543904, 0.293501319677, 0.419031703075],
             (16, 16): [0.540942539951, 0.302246395001, 0.405764169491],
             (19, 13): [0.255596227004, 0.451627307644, 0.287956021327],
             (13, 18): [0.308465363202, 0.292865519624, 0.770573717758],
             (0, 0): [0, 0, 0], (31, 31): [0, 0, 0]}
    for (x, y), val in known.items():
        assert np.abs(img[y, x] - np.array(val)).max() <= IMG_TOL
    assert abs(img.astype(np.float64).sum() - 266.798504875079) < 1e-2
    assert np.abs(img - O.render64(sp, cam)).max() <= IMG_TOL


def test_on_axis_alpha_one(rend):
    """one on-axis splat with opacity 1 -> colour c at the projection centre."""
    cam = isg.Camera(np.eye(3), np.zeros(3), 32.0, (16.5, 16.5), 33, 33)
    sp = np.array([[0, 0, 2.0, 0.2, 0.3, 0.6, 0.9, 1.0]])
    img = isg.render(sp, cam, isg.RenderOptions(t_min=0.0))
    assert np.abs(img[16, 16] - np.array([0.3, 0.6, 0.9])).max() <= 1e-6


def _grad_check(g, g_ref):
    for name, sl in GROUPS.items():
        a, b = g[:, sl], g_ref[:, sl]
        nb = np.linalg.norm(b)
        if nb == 0:
            assert np.abs(a).max() == 0
            continue
        assert np.linalg.norm(a - b) / nb <= GRAD_TOL, name
        assert np.abs(a - b).max() <= GRAD_TOL * np.abs(b).max(), name


@pytest.mark.parametrize("name,n,W,H,kw", CASES[:4], ids=[c[0] for c in CASES[:4]])
def test_loss_backward(rend, name, n, W, H, kw):
    rng = np.random.default_rng(1 + zlib.crc32(name.encode()))
    ms, co, cam = random_scene(rng, n, W, H, **kw)
    tms, tco, _ = random_scene(rng, n, W, H, **kw)
    target = O.render32(tms, tco, cam)
    rend.set_scene(ms, co)
    opts = isg.RenderOptions(t_min=1e-5)
    loss = rend.loss_backward(cam, target, opts, weight=1.0)
    g = rend.grads()
    loss_ref, g_ref = O.loss_backward32(ms, co, cam, target, t_min=1e-5)
    assert abs(loss - loss_ref) <= 1e-6 * abs(loss_ref)
    _grad_check(g, g_ref)


def test_backward_vs_fp64_reference(rend):
    """t_min=0 (exact reference forward): GPU grads vs the FP64 first-principles backward,
    which the CPU tests pin to central finite differences."""
    rng = np.random.default_rng(11)
    ms, co, cam = random_scene(rng, 60, 48, 40)
    sp = np.concatenate([ms, co], 1).astype(np.float64)
    target = rng.uniform(0, 1, (40, 48, 3))
    rend.set_scene(ms, co)
    loss = rend.loss_backward(cam, target.astype(np.float32), isg.RenderOptions(t_min=0.0))
    g = rend.grads()
    loss64, g64 = O.loss_grad64(sp, cam, target)
    assert abs(loss - loss64) <= 1e-5 * loss64
    _grad_check(g, g64)


@pytest.mark.parametrize("case", ["alpha_one", "underflow"])
def test_backward_through_zero_final_transmittance(rend, case):
    """The backward recovers every contributor's transmittance by dividing the pixel's final
    transmittance back up.  Where that is 0 or not a normal float -- an opacity-1 splat whose
    centre falls exactly on a pixel centre (alpha = 1), or t_min = 0 with a stack of opaque
    splats (T underflows) -- the forward re-walks the tile and hands over T before the last
    contributor instead (negated, debug_pixel_state); gradients must match the oracle either
    way, and ordinary tiles must keep the fast start."""
    rng = np.random.default_rng(7 if case == "alpha_one" else 8)
    W, H = 64, 48
    ms, co, cam = random_scene(rng, 400, W, H)
    if case == "alpha_one":
        # principal point on pixel centres: x = y = 0 projects exactly to (cx, cy)
        cam = isg.Camera(np.eye(3), np.zeros(3), cam.focal, (20.5, 12.5), W, H)
        extra_ms = np.array([[0.0, 0.0, 1.5, 0.004], [0.0, 0.0, 1.6, 0.01]], np.float32)
        extra_co = np.array([[0.9, 0.2, 0.1, 1.0], [0.1, 0.8, 0.3, 1.0]], np.float32)
        t_mins = (0.0, 1e-5)
    else:
        # 150 near-opaque splats over the same pixels: T falls below the smallest normal float
        k = 150
        z = np.linspace(1.2, 1.9, k, dtype=np.float32)
        extra_ms = np.stack([np.full(k, 0.01), np.full(k, -0.01), z, 0.02 * z], 1).astype(np.float32)
        extra_co = np.concatenate([rng.uniform(0, 1, (k, 3)), np.full((k, 1), 0.9)], 1).astype(np.float32)
        t_mins = (0.0,)
    ms = np.concatenate([ms, extra_ms]).astype(np.float32)
    co = np.concatenate([co, extra_co]).astype(np.float32)
    tms, tco, _ = random_scene(rng, 400, W, H)
    target = O.render32(tms, tco, cam)
    rend.set_scene(ms, co)
    for t_min in t_mins:
        opts = isg.RenderOptions(t_min=t_min)
        rend.zero_grads()
        loss = rend.loss_backward(cam, target, opts, weight=1.0)
        g = rend.grads()
        tl, _ = rend.debug_pixel_state(W, H)
        assert (tl < 0).any(), "no tile took the re-walk"
        assert (tl >= 0).any(), "every tile took the re-walk"
        loss_ref, g_ref = O.loss_backward32(ms, co, cam, target, t_min=t_min)
        assert abs(loss - loss_ref) <= 1e-6 * abs(loss_ref)
        # (the FP32 oracle, not the FP64 backward: a pixel stops where T reaches exactly 0,
        # so the splats behind an alpha-1 splat are not its "colour behind" here)
        _grad_check(g, g_ref)


@pytest.mark.parametrize("deterministic", [False, True], ids=["direct", "slot"])
def test_opacity_zero_keeps_its_gradient(rend, deterministic):
    """The blend kernels form alpha as ex2(r2 g + log2 o) and the backward accumulates
    dL/dalpha * alpha, dividing by the opacity per splat; the opacity is floored at 2^-60 for
    that, so a splat of opacity exactly 0 (valid input, IsoSplat3D::validate) still renders as
    alpha ~ 0 and still gets its opacity gradient sum(dL/dalpha * exp(...)) -- as does
    opacity 1."""
    rng = np.random.default_rng(21)
    W, H = 64, 48
    ms, co, cam = random_scene(rng, 500, W, H)
    co[::5, 3] = 0.0
    co[1::7, 3] = 1.0
    tms, tco, _ = random_scene(rng, 500, W, H)
    target = O.render32(tms, tco, cam)
    rend.set_deterministic(deterministic)
    try:
        rend.set_scene(ms, co)
        rend.zero_grads()
        img = rend.render(cam)
        assert np.abs(img - O.render32(ms, co, cam)).max() <= IMG_TOL
        loss = rend.loss_backward(cam, target, isg.RenderOptions(t_min=1e-5), weight=1.0)
        g = rend.grads()
    finally:
        rend.set_deterministic(False)
    loss_ref, g_ref = O.loss_backward32(ms, co, cam, target, t_min=1e-5)
    assert abs(loss - loss_ref) <= 1e-6 * abs(loss_ref)
    zero = co[:, 3] == 0.0
    assert np.abs(g_ref[zero, 7]).max() > 0  # the case is exercised
    _grad_check(g, g_ref)
    # the zero-opacity splats: their opacity gradient matches the oracle; the others are the
    # floor's 2^-60-scaled copies of an ordinary gradient where the oracle has exact zeros
    og, oref = g[zero, 7], g_ref[zero, 7]
    assert np.linalg.norm(og - oref) / np.linalg.norm(oref) <= GRAD_TOL
    assert np.abs(og - oref).max() <= GRAD_TOL * np.abs(oref).max()
    assert np.abs(g[zero, :7]).max() <= 1e-15 * np.abs(g_ref[:, :7]).max()


def test_target_ring_matches_device_targets():
    """Host-buffer training through the C-ABI target ring (isg_upload_target_async +
    isg_loss_backward_slot, uploads two views ahead, no host sync per step) gives the same
    trajectory as device-resident targets, bit for bit in deterministic mode."""
    import torch
    W, H, n = 96, 64, 3000
    ms, co = isg.synth_scene(n, W, H, seed=3)
    cams = [isg.Camera.synthetic(W, H, v, 4) for v in range(4)]
    targets = []
    for v, cam in enumerate(cams):
        tms, tco = isg.synth_scene(n, W, H, seed=100 + v)
        targets.append(O.render32(tms, tco, cam).astype(np.float32))
    pinned = [torch.from_numpy(t).pin_memory() for t in targets]
    host = [p.numpy() for p in pinned]
    opts = isg.RenderOptions(t_min=1e-5)
    adam = isg.AdamConfig()
    steps = 8  # graphs replayed twice; targets cycle with period 4, so slots get new data
    results = []
    for mode in ("device", "ring", "ring_graph"):
        with isg.Renderer(0) as r:
            r.set_deterministic(True)
            r.set_scene(ms, co)
            dev = [torch.from_numpy(t).cuda() for t in targets]
            torch.cuda.synchronize()
            losses = []
            if mode != "device":
                for s_ in range(min(2, steps)):  # three slots, reused: the WAR waits matter
                    r.upload_target_async(s_ % 3, host[s_ % 4])
            graphs = {}
            if mode == "ring_graph":
                r.render(cams[0], opts)  # buffers sized before any capture (captures cannot grow them)
            for s_ in range(steps):
                if mode == "device":
                    r.loss_backward_device(cams[s_ % 3], dev[s_ % 4].data_ptr(), opts)
                    r.adam_step(adam)
                else:
                    if s_ + 2 < steps:
                        r.upload_target_async((s_ + 2) % 3, host[(s_ + 2) % 4])
                    if mode == "ring":
                        r.loss_backward_slot(cams[s_ % 3], s_ % 3, opts)
                        r.adam_step(adam)
                    else:  # one graph per slot (camera s % 3), replayed on new uploads
                        key = s_ % 3
                        if key not in graphs:
                            r.graph_begin()
                            r.loss_backward_slot(cams[s_ % 3], s_ % 3, opts)
                            r.adam_step(adam)
                            graphs[key] = r.graph_end()
                        graphs[key].launch()
                losses.append(r.last_step_loss())
            results.append((np.array(losses), r.get_scene()))
    (l0, (a0, b0)) = results[0]
    for l1, (a1, b1) in results[1:]:
        assert np.array_equal(l0, l1)
        assert np.array_equal(a0, a1) and np.array_equal(b0, b1)
    with isg.Renderer(0) as r:
        r.set_scene(ms, co)
        with pytest.raises(ValueError):
            r.loss_backward_slot(cams[0], 1, opts)  # nothing uploaded
        with pytest.raises(ValueError):
            r.upload_target_async(isg.TARGET_SLOTS, host[0])


def test_image_ring_render_to_host(rend):
    """isg_render_host_async + isg_image_wait (frames rendered into the image ring while earlier
    frames travel to the host) return the same images as the synchronous render, slots reused."""
    import torch
    W, H, n = 80, 56, 2500
    ms, co = isg.synth_scene(n, W, H, seed=31)
    cams = [isg.Camera.synthetic(W, H, v, 5) for v in range(5)]
    opts = isg.RenderOptions(t_min=0.0)
    rend.set_scene(ms, co)
    ref = [rend.render(c, opts) for c in cams]
    pinned = [torch.empty((H, W, 3), dtype=torch.float32).pin_memory() for _ in range(3)]
    outs = [p.numpy() for p in pinned]
    got = []
    for i in range(9):  # 3 slots, each reused three times
        if i >= 3:
            rend.image_wait(i % 3)
            got.append(outs[i % 3].copy())
        rend.render_host_async(cams[i % 5], i % 3, outs[i % 3], opts)
    for i in range(6, 9):
        rend.image_wait(i % 3)
        got.append(outs[i % 3].copy())
    for i, img in enumerate(got):
        assert np.array_equal(img, ref[i % 5]), i
    with pytest.raises(ValueError):
        rend.render_host_async(cams[0], isg.IMAGE_SLOTS, outs[0], opts)


def _golden(name):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
    from make_golden import load_scenes
    return load_scenes(name)


@pytest.mark.parametrize("name", ["reference_scenes.npz", "reference_scenes_large.npz"])
def test_cuda_render_matches_reference_goldens(rend, name):
    """The CUDA render at t_min = 0 against the REFERENCE's own render() output (committed
    fixtures made by oracle/_ref): rotated + translated cameras, shifted principal points,
    near-plane / behind-camera / off-screen splats, opacity exactly 1, backgrounds; up to 6K
    splats over 144 tiles.  Every pixel within 1e-4 (no exceptions were needed: the FP32 depth
    order agrees with the FP64 one on these scenes), bins bit-exact vs the FP32 oracle."""
    worst = 0.0
    for sp, cam, bg, img in _golden(name):
        ms, co = sp[:, :4].astype(np.float32), sp[:, 4:].astype(np.float32)
        rend.set_scene(ms, co)
        out = rend.render(cam, isg.RenderOptions(background=tuple(bg), t_min=0.0))
        check_bins(rend, ms, co, cam)
        d = float(np.abs(out - img).max())
        worst = max(worst, d)
        assert d <= IMG_TOL, d
    print(f"{name}: max |CUDA - reference| = {worst:.3e}")


def test_gradients_on_reference_golden_scenes(rend):
    """Gradients on the reference-made large scenes (rotated cameras, opacity 1, backgrounds)
    at t_min = 0 against the FP64 first-principles backward (finite-difference pinned)."""
    for sp, cam, bg, img in _golden("reference_scenes_large.npz"):
        ms, co = sp[:, :4].astype(np.float32), sp[:, 4:].astype(np.float32)
        target = np.clip(img[::-1] * 0.9 + 0.05, 0, 1)  # a different image of the same size
        rend.set_scene(ms, co)
        loss = rend.loss_backward(cam, target.astype(np.float32),
                                  isg.RenderOptions(background=tuple(bg), t_min=0.0))
        g = rend.grads()
        loss64, g64 = O.loss_grad64(sp, cam, target, bg)
        assert abs(loss - loss64) <= 1e-5 * loss64
        _grad_check(g, g64)


def test_multi_view_accumulation(rend):
    W, H = 128, 96
    ms, co = isg.synth_scene(4000, W, H, seed=3)
    tms, tco = isg.synth_scene(4000, W, H, seed=4)
    rend.set_scene(ms, co)
    g_ref = np.zeros((4000, 8), np.float32)
    tot = 0.0
    for k in range(3):
        cam = isg.Camera.synthetic(W, H, k, 3)
        target = O.render32(tms, tco, cam)
        tot += rend.loss_backward(cam, target, weight=1 / 3)
        O.loss_backward32(ms, co, cam, target, weight=1 / 3, grads=g_ref)
    assert abs(rend.read_loss() - tot) < 1e-9 + 1e-7 * tot
    _grad_check(rend.grads(), g_ref)


def _adam_setup():
    W, H = 128, 96
    ms, co = isg.synth_scene(3000, W, H, seed=8)
    tms, tco = isg.synth_scene(3000, W, H, seed=9)
    cam = isg.Camera.synthetic(W, H)
    target = O.render32(tms, tco, cam)
    cfg = isg.AdamConfig(lr_mu=1e-3, lr_sigma=5e-3, lr_color=1e-2, lr_opacity=1e-2, eps=1e-15)
    return ms, co, cam, target, cfg


def test_adam_matches_oracle_given_grads(rend):
    """Unfused path: the GPU's own gradients fed to the oracle Adam (torch semantics, pinned
    against torch.optim.Adam in the CPU tests) reproduce the GPU update over 3 steps."""
    ms, co, cam, target, cfg = _adam_setup()
    lrs = [cfg.lr_mu, cfg.lr_sigma, cfg.lr_color, cfg.lr_opacity]
    rend.set_scene(ms, co)
    oms, oco = ms.copy(), co.copy()
    m = np.zeros((3000, 8), np.float32)
    v = np.zeros((3000, 8), np.float32)
    raw = O.raw_init32(oms, oco)  # persistent optimizer-space (log sigma, logit opacity)
    for step in range(1, 4):
        rend.loss_backward(cam, target)
        g = rend.grads()
        rend.adam_step(cfg)
        O.adam32(oms, oco, m, v, g, step, lrs, cfg.beta1, cfg.beta2, cfg.eps, raw=raw)
        gms, gco = rend.get_scene()
        assert np.abs(gms - oms).max() <= 1e-5
        assert np.abs(gco - oco).max() <= 1e-5
        oms, oco = gms.copy(), gco.copy()  # continue from the GPU state (moments already match)


def test_adam_fused_equals_unfused(rend):
    """K8 fused (projection backward + Adam) == K8a projection then K8b Adam."""
    ms, co, cam, target, cfg = _adam_setup()
    out = []
    for fused in (True, False):
        rend.set_scene(ms, co)
        rend.loss_backward(cam, target)
        g = None if fused else rend.grads()  # grads() projects first -> un-fused Adam
        rend.adam_step(cfg)
        out.append((rend.get_scene(), g))
    (ams, aco), _ = out[0]
    (bms, bco), g = out[1]
    big = np.abs(g) > 1e-2 * np.abs(g).max(axis=0, keepdims=True)
    step_tol = np.array([cfg.lr_mu] * 3 + [cfg.lr_sigma] + [cfg.lr_color] * 3 + [cfg.lr_opacity])
    pa = np.concatenate([ams[:, :3], np.log(ams[:, 3:4]), aco[:, :3],
                         np.log(aco[:, 3:4] / (1 - aco[:, 3:4]))], 1)
    pb = np.concatenate([bms[:, :3], np.log(bms[:, 3:4]), bco[:, :3],
                         np.log(bco[:, 3:4] / (1 - bco[:, 3:4]))], 1)
    d = np.abs(pa - pb)
    assert np.all(d <= 2.001 * step_tol + 1e-6)  # Adam's first step is bounded by lr
    assert np.all(d[big] <= (1e-2 * step_tol + 1e-6)[np.nonzero(big)[1]])


@pytest.mark.parametrize("n", [1, 127, 128, 129, 230_077])
def test_adam_stream_sizes(n):
    """K8's TMA stream (direct mode) updates every splat exactly once at sizes around its
    128-splat chunks and with more chunks than resident CTAs: the fused step's first Adam move
    (+-lr for any nonzero gradient) equals the un-fused one wherever the gradient is nonzero."""
    W, H = 96, 64
    ms, co = isg.synth_scene(n, W, H, seed=21)
    tms, tco = isg.synth_scene(max(n, 64), W, H, seed=22)
    cam = isg.Camera.synthetic(W, H)
    target = O.render32(tms, tco, cam)
    cfg = isg.AdamConfig(lr_mu=1e-3, lr_sigma=5e-3, lr_color=1e-2, lr_opacity=1e-2, eps=1e-15)
    out = []
    with isg.Renderer(0) as r:
        for fused in (True, False):
            r.set_scene(ms, co)
            r.loss_backward(cam, target)
            g = None if fused else r.grads()
            r.adam_step(cfg)
            out.append((r.get_scene(), g))
    (ams, aco), _ = out[0]
    (bms, bco), g = out[1]
    lr = np.array([cfg.lr_mu] * 3 + [cfg.lr_sigma] + [cfg.lr_color] * 3 + [cfg.lr_opacity])
    pa = np.concatenate([ams[:, :3], np.log(ams[:, 3:4]), aco[:, :3],
                         np.log(aco[:, 3:4] / (1 - aco[:, 3:4]))], 1)
    pb = np.concatenate([bms[:, :3], np.log(bms[:, 3:4]), bco[:, :3],
                         np.log(bco[:, 3:4] / (1 - bco[:, 3:4]))], 1)
    moved = np.abs(g) > 1e-6 * np.abs(g).max(axis=0, keepdims=True)
    d = np.abs(pa - pb)
    assert np.all(d[moved] <= (0.1 * lr + 1e-6)[np.nonzero(moved)[1]])
    assert np.all(d[~moved] <= (2.001 * lr + 1e-6)[np.nonzero(~moved)[1]])


def test_validation_errors(rend):
    cam = isg.Camera(np.eye(3), np.zeros(3), 32.0, (16, 16), 32, 32)
    good = np.array([[0, 0, 2, .25, 1, .2, .1, .5]] * 3, np.float64)
    cases = [((1, 3), 0.0, "IsoSplat3D.sigma: must be positive and finite"),
             ((2, 0), np.nan, "IsoSplat3D.mu: non-finite coordinates"),
             ((1, 7), 1.5, "IsoSplat3D.opacity: must be in [0,1]"),
             ((0, 5), np.inf, "IsoSplat3D.color: non-finite")]
    for (i, j), val, msg in cases:
        bad = good.copy()
        bad[i, j] = val
        ms, co = isg.splats_to_soa(bad)
        rend.set_scene(ms, co)
        with pytest.raises(isg.DomainError, match=msg.replace("[", r"\[").replace("]", r"\]")):
            rend.render(cam)
    rend.set_scene(*isg.splats_to_soa(good))
    bad_cam = isg.Camera(np.eye(3), np.zeros(3), -1.0, (16, 16), 32, 32)
    with pytest.raises(isg.DomainError, match="Camera.focal"):
        rend.render(bad_cam)
    with pytest.raises(ValueError):
        rend.render(cam, isg.RenderOptions(t_min=2.0))
    with pytest.raises(isg.IsgError):
        isg.Renderer(0).adam_step()


def test_key_capacity_regrow():
    """Huge splats exceed the initial key capacity: the frame is re-run, results exact."""
    W, H = 512, 512
    rng = np.random.default_rng(3)
    with isg.Renderer(0) as r:
        ms, co, cam = random_scene(rng, 2000, W, H, sigma2d=(60.0, 200.0))
        r.set_scene(ms, co)
        img = r.render(cam)
        assert r.stats()["regrow_events"] >= 1
        check_bins(r, ms, co, cam)
        assert np.abs(img - O.render32(ms, co, cam)).max() <= IMG_TOL


def test_async_overflow_of_an_earlier_view_is_reported():
    """Two asynchronous views, the FIRST overflowing the key capacity, then Adam: the step is
    skipped as a whole (no update from the partial batch), the next synchronisation reports the
    overflow once (sticky device record, not only the last frame's count), capacity has grown,
    and the re-run step matches two synchronous views + Adam."""
    import torch
    W, H = 512, 512
    rng = np.random.default_rng(3)
    ms, co, cam_near = random_scene(rng, 2000, W, H, sigma2d=(60.0, 200.0))
    cam_far = isg.Camera(np.eye(3), np.array([0.0, 0.0, 60.0]), cam_near.focal,
                         (W / 2, H / 2), W, H)  # the same splats ~10x smaller: few keys
    tms, tco, _ = random_scene(rng, 2000, W, H, sigma2d=(60.0, 200.0))
    targets = [torch.from_numpy(O.render32(tms, tco, c)).cuda() for c in (cam_near, cam_far)]
    torch.cuda.synchronize()
    cams = (cam_near, cam_far)
    with isg.Renderer(0) as r:
        r.set_deterministic(True)  # bitwise comparison below
        r.set_scene(ms, co)
        cap0 = r.stats()["key_capacity"]
        for c, t in zip(cams, targets):
            r.loss_backward_device(c, t.data_ptr(), weight=0.5)
        r.adam_step()
        with pytest.raises(isg.IsgError) as ei:
            r.synchronize()
        assert ei.value.status == 5  # ISG_E_OVERFLOW
        st = r.stats()
        assert st["overflowed_frames"] == 1 and st["key_capacity"] > cap0
        m1, c1 = r.get_scene()
        np.testing.assert_array_equal(m1, ms)  # the step did not move anything
        np.testing.assert_array_equal(c1, co)
        r.synchronize()  # reported once
        for c, t in zip(cams, targets):
            r.loss_backward_device(c, t.data_ptr(), weight=0.5)
        r.adam_step()
        r.synchronize()
        a_ms, a_co = r.get_scene()
        assert r.stats()["adam_steps"] >= 1
    with isg.Renderer(0) as r:
        r.set_deterministic(True)  # bitwise comparison below
        r.set_scene(ms, co)
        for c, t in zip(cams, targets):
            r.loss_backward(c, t.cpu().numpy(), weight=0.5)
        r.adam_step()
        b_ms, b_co = r.get_scene()
    np.testing.assert_array_equal(a_ms, b_ms)
    np.testing.assert_array_equal(a_co, b_co)


def test_render_deterministic(rend):
    W, H = 256, 256
    ms, co = isg.synth_scene(10000, W, H)
    rend.set_scene(ms, co)
    cam = isg.Camera.synthetic(W, H)
    a = rend.render(cam)
    b = rend.render(cam)
    assert np.array_equal(a, b)


def test_full_size_c2_render_parity():
    """Config C2 (1M splats, 1920x1080): bins bit-exact and image within 1e-4 of the oracle."""
    W, H, n = 1920, 1080, 1_000_000
    ms, co = isg.synth_scene(n, W, H, seed=2403)
    cam = isg.Camera.synthetic(W, H)
    with isg.Renderer(0) as r:
        r.set_scene(ms, co)
        img = r.render(cam, isg.RenderOptions(t_min=T_MIN))
        keys = check_bins(r, ms, co, cam)
        assert np.all(np.diff(keys.astype(np.int64) >> 32) >= 0)
        assert np.abs(img - O.render32(ms, co, cam, t_min=T_MIN)).max() <= IMG_TOL


def test_full_size_c3_loss_backward():
    """Config C3 (1M splats, 1920x1080, the bench's train step): L2 loss and all 8M parameter
    gradients against the oracle at full size, same tolerances as the small cases."""
    W, H, n = 1920, 1080, 1_000_000
    ms, co = isg.synth_scene(n, W, H, seed=1)
    tms, tco = isg.synth_scene(n, W, H, seed=2)
    cam = isg.Camera.synthetic(W, H)
    target = O.render32(tms, tco, cam, t_min=T_MIN)
    with isg.Renderer(0) as r:
        r.set_scene(ms, co)
        loss = r.loss_backward(cam, target, isg.RenderOptions(t_min=T_MIN))
        g = r.grads()
    loss_ref, g_ref = O.loss_backward32(ms, co, cam, target, t_min=T_MIN)
    assert abs(loss - loss_ref) <= 1e-6 * abs(loss_ref)
    _grad_check(g, g_ref)


def test_full_size_c5_bins_and_gradients():
    """Config C5 (10M splats, 3840x2160, 33 M tile keys): bins bit-exact, then the L2 loss and
    all 80 M gradients against the oracle (the target is the GPU render of a second scene: an
    input to both sides, so it need not come from the oracle)."""
    W, H, n = 3840, 2160, 10_000_000
    ms, co = isg.synth_scene(n, W, H, seed=5)
    tms, tco = isg.synth_scene(n, W, H, seed=6)
    cam = isg.Camera.synthetic(W, H)
    with isg.Renderer(0) as r:
        r.set_scene(tms, tco)
        target = r.render(cam, isg.RenderOptions(t_min=T_MIN))
        r.set_scene(ms, co)
        loss = r.loss_backward(cam, target, isg.RenderOptions(t_min=T_MIN))
        g = r.grads()
        keys = check_bins(r, ms, co, cam)
        assert len(keys) > 30_000_000
    loss_ref, g_ref = O.loss_backward32(ms, co, cam, target, t_min=T_MIN)
    assert abs(loss - loss_ref) <= 1e-6 * abs(loss_ref)
    _grad_check(g, g_ref)


def test_full_size_c4_view_batch_gradients():
    """Config C4 (3M splats, 1920x1080, the 8-view batch of one step: cameras yawed over
    +-5.25 deg and translated): the accumulated weight-1/8 loss and all 24 M gradients of the
    batch against the oracle, per group <= 1e-3, then the Adam step against the oracle's
    optimizer-space Adam fed the same gradients."""
    W, H, n, V = 1920, 1080, 3_000_000, 8
    ms, co = isg.synth_scene(n, W, H, seed=2403)
    tms, tco = isg.synth_scene(n, W, H, seed=14244)
    cams = [isg.Camera.synthetic(W, H, k, V) for k in range(V)]
    opts = isg.RenderOptions(t_min=T_MIN)
    with isg.Renderer(0) as r:
        r.set_scene(tms, tco)
        targets = [r.render(c, opts) for c in cams]
        r.set_scene(ms, co)
        loss = sum(r.loss_backward(c, t, opts, weight=1.0 / V) for c, t in zip(cams, targets))
        g = r.grads()
        r.adam_step()
        ms1, co1 = r.get_scene()
    g_ref = np.zeros((n, 8), np.float32)
    loss_ref = 0.0
    for c, t in zip(cams, targets):
        l, _ = O.loss_backward32(ms, co, c, t, t_min=T_MIN, weight=1.0 / V, grads=g_ref)
        loss_ref += l
    assert abs(loss - loss_ref) <= 1e-6 * abs(loss_ref)
    _grad_check(g, g_ref)
    oms, oco = ms.copy(), co.copy()
    m = np.zeros((n, 8), np.float32)
    v = np.zeros((n, 8), np.float32)
    cfg = isg.AdamConfig()
    O.adam32(oms, oco, m, v, g, 1, [cfg.lr_mu, cfg.lr_sigma, cfg.lr_color, cfg.lr_opacity],
             cfg.beta1, cfg.beta2, cfg.eps)
    assert np.abs(ms1 - oms).max() <= 1e-5 and np.abs(co1 - oco).max() <= 1e-5


def test_binning_modes_bit_identical(rend):
    """Tile-bucket and onesweep-radix binning give identical lists, images and gradients
    (deterministic gradient mode)."""
    W, H = 320, 200
    ms, co = isg.synth_scene(30000, W, H, seed=21)
    tms, tco = isg.synth_scene(30000, W, H, seed=22)
    cam = isg.Camera.synthetic(W, H, 2, 8)
    target = O.render32(tms, tco, cam)
    out = []
    rend.set_deterministic(True)
    for mode in (isg.Renderer.BINNING_TILE_BUCKET, isg.Renderer.BINNING_RADIX):
        rend.set_binning(mode)
        rend.set_scene(ms, co)
        img = rend.render(cam)
        bins = check_bins(rend, ms, co, cam)
        loss = rend.loss_backward(cam, target)
        out.append((img, bins, loss, rend.grads()))
    rend.set_binning(isg.Renderer.BINNING_RADIX)  # the defaults, for the tests that follow
    rend.set_deterministic(False)
    (i0, b0, l0, g0), (i1, b1, l1, g1) = out
    assert np.array_equal(i0, i1) and np.array_equal(b0, b1)
    assert l0 == l1 and np.array_equal(g0, g1)


@pytest.mark.parametrize("deterministic", [True, False], ids=["slots", "direct"])
def test_gradients_bitwise_deterministic(rend, deterministic):
    """Deterministic mode: bitwise-identical gradients run to run.  Direct mode (L2 reduction,
    order varies): identical loss, gradients equal to the deterministic ones within FP32
    summation reordering, and both within the oracle tolerance."""
    W, H = 256, 160
    ms, co = isg.synth_scene(20000, W, H, seed=31)
    tms, tco = isg.synth_scene(20000, W, H, seed=32)
    cam = isg.Camera.synthetic(W, H)
    target = O.render32(tms, tco, cam)
    rend.set_deterministic(deterministic)
    rend.set_scene(ms, co)
    runs = []
    for _ in range(3):
        rend.zero_grads()
        runs.append((rend.loss_backward(cam, target), rend.grads()))
    rend.set_deterministic(False)
    for loss, g in runs[1:]:
        assert loss == runs[0][0]
        if deterministic:
            assert np.array_equal(g, runs[0][1])
        else:
            np.testing.assert_allclose(g, runs[0][1], rtol=1e-4,
                                       atol=1e-6 * np.abs(runs[0][1]).max())
    _, g_ref = O.loss_backward32(ms, co, cam, target)
    _grad_check(runs[0][1], g_ref)


@pytest.mark.parametrize("mode", [0, 1], ids=["tile_bucket", "radix"])
def test_long_tile_lists(mode):
    """Tiles with > 2048 entries take the global-memory merge path of the tile sort."""
    W, H = 96, 80
    rng = np.random.default_rng(9)
    with isg.Renderer(0) as r:
        r.set_binning(mode)
        ms, co, cam = random_scene(rng, 5000, W, H, sigma2d=(40.0, 80.0))
        r.set_scene(ms, co)
        img = r.render(cam, isg.RenderOptions(t_min=0.0))
        keys, vals, ranges = r.debug_bins()
        assert (ranges[:, 1] - ranges[:, 0]).max() > 2048
        check_bins(r, ms, co, cam)
        assert np.abs(img - O.render32(ms, co, cam, t_min=0.0)).max() <= IMG_TOL
        tms, tco, _ = random_scene(rng, 5000, W, H, sigma2d=(40.0, 80.0))
        target = O.render32(tms, tco, cam)
        loss = r.loss_backward(cam, target, isg.RenderOptions(t_min=0.0))
        loss_ref, g_ref = O.loss_backward32(ms, co, cam, target, t_min=0.0)
        assert abs(loss - loss_ref) <= 1e-6 * abs(loss_ref)
        _grad_check(r.grads(), g_ref)


@pytest.mark.parametrize("views,loss_kind", [(1, isg.LOSS_L2), (3, isg.LOSS_L2),
                                             (2, isg.LOSS_L1_DSSIM)])
def test_cuda_graph_replay_matches_stream_execution(views, loss_kind):
    """A captured train step (loss_backward_device per view + Adam) replayed K times gives the
    bitwise-identical trajectory of K ordinary steps (device-side Adam step counter)."""
    import torch
    W, H, n, K = 128, 96, 4000, 5
    ms, co = isg.synth_scene(n, W, H, seed=31)
    tms, tco = isg.synth_scene(n, W, H, seed=32)
    cams = [isg.Camera.synthetic(W, H, k, views) for k in range(views)]
    targets = [torch.from_numpy(O.render32(tms, tco, c)).cuda() for c in cams]
    torch.cuda.synchronize()

    def step(r):
        for c, t in zip(cams, targets):
            r.loss_backward_device(c, t.data_ptr(), weight=1.0 / views)
        r.adam_step()

    results = []
    for use_graph in (False, True):
        r = isg.Renderer(0)
        r.set_deterministic(True)  # bitwise comparison below
        r.set_loss(loss_kind, 0.2)
        r.set_scene(ms, co)
        step(r)  # warm-up step sizes every buffer
        if use_graph:
            r.graph_begin()
            step(r)
            with pytest.raises(isg.IsgError):
                r.read_loss()  # synchronising call inside a capture
            g = r.graph_end()
            for _ in range(K):
                g.launch()
            g.close()
        else:
            for _ in range(K):
                step(r)
        loss = r.last_step_loss()
        results.append((r.get_scene(), loss))
        r.close()
    (a, la), (b, lb) = results
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])
    assert la == lb


def test_nccl_single_rank_path_matches_local_adam():
    """The multi-GPU step on one rank: NCCL (dlopen'd) all-reduce of the gradient buffer and the
    loss, then the un-fused Adam — identical to the fused single-GPU step."""
    W, H, n = 96, 64, 2000
    ms, co = isg.synth_scene(n, W, H, seed=41)
    tms, tco = isg.synth_scene(n, W, H, seed=42)
    cams = [isg.Camera.synthetic(W, H, k, 2) for k in range(2)]
    targets = [O.render32(tms, tco, c) for c in cams]
    out = []
    for use_nccl in (False, True):
        r = isg.Renderer(0)
        r.set_deterministic(True)  # bitwise comparison below
        r.set_scene(ms, co)
        if use_nccl:
            r.nccl_init(1, 0, isg.Renderer.nccl_unique_id())
        losses = []
        for _ in range(3):
            for c, t in zip(cams, targets):
                r.loss_backward(c, t, weight=0.5)
            r.adam_step()
            losses.append(r.last_step_loss())
        if use_nccl:
            r.nccl_detach()
        out.append((r.get_scene(), losses))
        r.close()
    (a, la), (b, lb) = out
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])
    assert la == lb


def test_cuda_graph_with_nccl_single_rank():
    """The multi-GPU step (NCCL all-reduce + un-fused Adam) captured in a CUDA graph replays
    like kernel-by-kernel execution (one rank)."""
    import torch
    W, H, n, K = 96, 64, 2000, 4
    ms, co = isg.synth_scene(n, W, H, seed=51)
    tms, tco = isg.synth_scene(n, W, H, seed=52)
    cam = isg.Camera.synthetic(W, H)
    target = torch.from_numpy(O.render32(tms, tco, cam)).cuda()
    torch.cuda.synchronize()
    out = []
    for use_graph in (False, True):
        r = isg.Renderer(0)
        r.set_deterministic(True)  # bitwise comparison below
        r.set_scene(ms, co)
        r.nccl_init(1, 0, isg.Renderer.nccl_unique_id())
        r.loss_backward_device(cam, target.data_ptr())
        r.adam_step()
        if use_graph:
            r.graph_begin()
            r.loss_backward_device(cam, target.data_ptr())
            r.adam_step()
            g = r.graph_end()
            for _ in range(K):
                g.launch()
            g.close()
        else:
            for _ in range(K):
                r.loss_backward_device(cam, target.data_ptr())
                r.adam_step()
        out.append((r.get_scene(), r.last_step_loss()))
        r.nccl_detach()
        r.close()
    np.testing.assert_array_equal(out[0][0][0], out[1][0][0])
    np.testing.assert_array_equal(out[0][0][1], out[1][0][1])
    assert out[0][1] == out[1][1]


@pytest.mark.parametrize("chunks,graph", [(1, False), (4, False), (8, True)])
def test_pipelined_exchange_matches_local_step(chunks, graph):
    """The chunked exchange (projection backward, all-reduce and Adam pipelined over splat
    ranges on two streams; loss and overflow flags in front of chunk 0) on one rank at a size
    where it really splits (600K splats, 4-8 chunks): scene bitwise equal to the fused local
    step, and the folded loss equal to the local double loss exactly."""
    import torch
    W, H, n = 320, 240, 600_000
    ms, co = isg.synth_scene(n, W, H, seed=51)
    tms, tco = isg.synth_scene(n, W, H, seed=52)
    cams = [isg.Camera.synthetic(W, H, k, 2) for k in range(2)]
    targets = [torch.from_numpy(O.render32(tms, tco, c, t_min=T_MIN)).cuda() for c in cams]
    torch.cuda.synchronize()
    opts = isg.RenderOptions(t_min=T_MIN)
    out = []
    for use_nccl in (False, True):
        r = isg.Renderer(0)
        r.set_deterministic(True)  # bitwise comparison below
        r.set_scene(ms, co)
        if use_nccl:
            r.nccl_init(1, 0, isg.Renderer.nccl_unique_id())
            r.set_exchange_chunks(chunks)
            assert r.nccl_info()["nranks"] == 1

        def step():
            for c, t in zip(cams, targets):
                r.loss_backward_device(c, t.data_ptr(), opts, weight=0.5)
            r.adam_step()
        step()
        losses = [r.last_step_loss()]
        if graph and use_nccl:
            r.graph_begin()
            step()
            g = r.graph_end()
            for _ in range(2):
                g.launch()
            g.close()
        else:
            for _ in range(2):
                step()
        losses.append(r.last_step_loss())
        out.append((r.get_scene(), losses))
        r.close()
    (a, la), (b, lb) = out
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])
    assert la == lb


def test_nccl_attach_caller_owned_communicator():
    """isg_nccl_attach uses a communicator the caller created (here ncclCommInitRank called
    directly through ctypes) and leaves it alive: the caller destroys it after the detach."""
    import ctypes as C
    import torch  # noqa: F401  (loads torch's libnccl.so.2, the copy libisg binds to)
    nccl = C.CDLL("libnccl.so.2", mode=C.RTLD_GLOBAL)
    W, H, n = 96, 64, 2000
    ms, co = isg.synth_scene(n, W, H, seed=41)
    tms, tco = isg.synth_scene(n, W, H, seed=42)
    cam = isg.Camera.synthetic(W, H)
    target = O.render32(tms, tco, cam)
    out = []
    for attach in (False, True):
        with isg.Renderer(0) as r:
            r.set_deterministic(True)  # bitwise comparison below
            r.set_scene(ms, co)
            comm = C.c_void_p()
            if attach:
                class UniqueId(C.Structure):  # ncclUniqueId is passed by value
                    _fields_ = [("internal", C.c_char * 128)]
                uid = UniqueId.from_buffer_copy(isg.Renderer.nccl_unique_id())
                assert nccl.ncclCommInitRank(C.byref(comm), 1, uid, 0) == 0
                r.nccl_attach(comm.value)
                info = r.nccl_info()
                assert info["nranks"] == 1 and info["rank"] == 0 and info["nccl_version"] > 0
            for _ in range(2):
                r.loss_backward(cam, target)
                r.adam_step()
            out.append(r.get_scene())
            if attach:
                r.nccl_detach()
                assert r.nccl_info()["nranks"] == 1
                # still alive: the caller's destroy succeeds exactly once
                assert nccl.ncclCommDestroy(comm) == 0
    np.testing.assert_array_equal(out[0][0], out[1][0])
    np.testing.assert_array_equal(out[0][1], out[1][1])


def test_step_loss_async_in_graph_matches_sync_read():
    """isg_step_loss_async captured in a step graph (the pipelined loop's D2H of each step's
    loss) delivers the same value as the synchronous isg_last_step_loss."""
    import torch
    W, H = 128, 96
    ms, co = isg.synth_scene(3000, W, H, seed=21)
    tms, tco = isg.synth_scene(3000, W, H, seed=22)
    cam = isg.Camera.synthetic(W, H)
    target = torch.from_numpy(O.render32(tms, tco, cam)).cuda()
    host = torch.zeros(1, dtype=torch.float64).pin_memory()
    with isg.Renderer(0) as r:
        r.set_scene(ms, co)
        r.loss_backward(cam, target.cpu().numpy())  # sizes the buffers
        r.zero_grads()
        r.graph_begin()
        r.loss_backward_device(cam, target.data_ptr())
        r.adam_step(isg.AdamConfig())
        r.step_loss_async(host.data_ptr())
        g = r.graph_end()
        for _ in range(3):
            g.launch()
            r.synchronize()
            assert float(host[0]) == r.last_step_loss() > 0.0
        # page-locked memory is written by a kernel through its mapped address; pageable
        # memory takes the cudaMemcpyAsync path (not capturable, so outside a graph)
        pageable = np.zeros(1, np.float64)
        r.loss_backward_device(cam, target.data_ptr())
        r.adam_step(isg.AdamConfig())
        r.step_loss_async(pageable.ctypes.data)
        r.synchronize()
        assert pageable[0] == r.last_step_loss() > 0.0


def test_three_pass_tile_sort_many_tiles():
    """> 65536 tiles (8192 x 2064 px: 17 tile-id bits) -> the tile sort runs 3 digit passes;
    its last-pass epilogue (pairs + ranges) and the empty-tile fix-up stay bit-exact."""
    W, H = 8192, 2064
    rng = np.random.default_rng(66048)
    ms, co, cam = random_scene(rng, 6000, W, H, sigma2d=(0.5, 40.0))
    with isg.Renderer(0) as r:
        r.set_scene(ms, co)
        for _ in range(3):  # later frames reuse the per-frame scratch of earlier ones
            img = r.render(cam)
            keys = check_bins(r, ms, co, cam)
        assert (keys >> 32).max() >= 65536  # tiles past the 16-bit boundary are populated
        assert np.abs(img - O.render32(ms, co, cam)).max() <= IMG_TOL


@pytest.mark.parametrize("W,H", [(1, 1), (8, 8), (16, 16), (17, 1), (1, 33)])
def test_degenerate_image_shapes(rend, W, H):
    """One-tile and one-pixel-wide images (a 1-bit tile sort): bins, image and gradients."""
    rng = np.random.default_rng(W * 100 + H)
    ms, co, cam = random_scene(rng, 50, W, H, sigma2d=(0.3, 4.0))
    rend.set_scene(ms, co)
    img = rend.render(cam)
    check_bins(rend, ms, co, cam)
    assert np.abs(img - O.render32(ms, co, cam)).max() <= IMG_TOL
    target = rng.uniform(0, 1, (H, W, 3)).astype(np.float32)
    loss = rend.loss_backward(cam, target)
    loss_ref, g_ref = O.loss_backward32(ms, co, cam, target)
    assert abs(loss - loss_ref) <= 1e-6 * abs(loss_ref) + 1e-12
    _grad_check(rend.grads(), g_ref)
    rend.zero_grads()


def test_all_splats_culled(rend):
    """Every splat behind the near plane: no keys, background image, zero gradients, and the
    Adam step leaves the (gradient-free) scene bitwise unchanged (optimizer-space state is
    persistent; a zero update rewrites nothing)."""
    W, H = 96, 64
    rng = np.random.default_rng(8)
    ms, co, cam = random_scene(rng, 500, W, H)
    ms[:, 2] = -np.abs(ms[:, 2])  # behind the camera
    rend.set_scene(ms, co)
    img = rend.render(cam, isg.RenderOptions(background=(0.1, 0.2, 0.3)))
    keys, vals, ranges = rend.debug_bins()
    assert len(keys) == 0 and np.all(ranges == 0)
    assert np.array_equal(img, np.broadcast_to(np.float32([0.1, 0.2, 0.3]), img.shape))
    target = rng.uniform(0, 1, (H, W, 3)).astype(np.float32)
    rend.loss_backward(cam, target)
    assert np.all(rend.grads() == 0)
    rend.adam_step(isg.AdamConfig(eps=0.0))  # eps 0: m == 0 must still move nothing
    m2, c2 = rend.get_scene()
    np.testing.assert_array_equal(m2, ms)
    np.testing.assert_array_equal(c2, co)


def test_adam_opacity_at_interval_ends(rend):
    """Opacity exactly 0 or 1 (IsoSplat3D::validate allows both, splat3d.cpp:14-16) enters the
    optimizer's open interval once: the splat trains (finite logit, non-zero gradient factor)
    instead of freezing, and matches the oracle's optimizer-space Adam."""
    W, H = 64, 48
    rng = np.random.default_rng(17)
    ms, co, cam = random_scene(rng, 400, W, H)
    co[::3, 3] = 1.0
    co[1::3, 3] = 0.0
    tms, tco, _ = random_scene(rng, 400, W, H)
    target = O.render32(tms, tco, cam)
    cfg = isg.AdamConfig(lr_mu=1e-3, lr_sigma=5e-3, lr_color=1e-2, lr_opacity=5e-2)
    lrs = [cfg.lr_mu, cfg.lr_sigma, cfg.lr_color, cfg.lr_opacity]
    rend.set_scene(ms, co)
    oms, oco = ms.copy(), co.copy()
    m = np.zeros((400, 8), np.float32)
    v = np.zeros((400, 8), np.float32)
    raw = O.raw_init32(oms, oco)
    assert np.all(np.isfinite(raw))
    for step in range(1, 4):
        rend.loss_backward(cam, target)
        g = rend.grads()
        rend.adam_step(cfg)
        O.adam32(oms, oco, m, v, g, step, lrs, cfg.beta1, cfg.beta2, cfg.eps, raw=raw)
    gms, gco = rend.get_scene()
    assert np.all(np.isfinite(gms)) and np.all(np.isfinite(gco))
    np.testing.assert_allclose(gco, oco, atol=1e-5)
    np.testing.assert_allclose(gms, oms, atol=1e-5)
    covered = np.abs(g[:, 7]) > 0
    moved = gco[:, 3] != co[:, 3]
    # splats that started at exactly 0 or 1 and see a gradient move
    ends = (co[:, 3] == 0.0) | (co[:, 3] == 1.0)
    assert np.all(moved[ends & covered])


def test_graph_replay_refused_after_reallocation():
    """A captured step holds device pointers: after the scene grows (buffers reallocated) or
    adaptive control swaps the scene buffers, replaying it is refused (ISG_E_STATE) instead
    of touching freed memory; a fresh capture works."""
    import torch
    W, H = 96, 64
    cam = isg.Camera.synthetic(W, H)
    with isg.Renderer(0) as r:
        ms, co = isg.synth_scene(2000, W, H, seed=41)
        r.set_scene(ms, co)
        target = torch.from_numpy(O.render32(ms, co, cam)).cuda()
        r.loss_backward(cam, target.cpu().numpy())
        r.zero_grads()

        def capture():
            r.graph_begin()
            r.loss_backward_device(cam, target.data_ptr())
            r.adam_step(isg.AdamConfig())
            return r.graph_end()
        g = capture()
        g.launch()
        r.synchronize()
        big_ms, big_co = isg.synth_scene(50000, W, H, seed=42)
        r.set_scene(big_ms, big_co)  # more splats than allocated: buffers regrow
        with pytest.raises(isg.IsgError) as e:
            g.launch()
        assert e.value.status == isg.ISG_E_STATE
        r.loss_backward(cam, target.cpu().numpy())  # sizes the key buffers for the new scene
        r.zero_grads()
        g2 = capture()
        g2.launch()
        r.synchronize()
        r.adaptive_control(isg.AdaptParams(1e-3, 0.5, 0.05, 1e9, 0))
        with pytest.raises(isg.IsgError):
            g2.launch()


def _random_rotation(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


@pytest.mark.parametrize("seed", range(32))
def test_randomized_configurations(rend, seed):
    """Seeded random image sizes, splat counts and size ranges, arbitrary camera rotations,
    translations, focal lengths, principal points, backgrounds and t_min: bins bit-exact,
    image and gradients within the stated tolerances."""
    rng = np.random.default_rng(1000 + seed)
    W, H = int(rng.integers(1, 300)), int(rng.integers(1, 200))
    n = int(rng.integers(1, 6000))
    R = _random_rotation(rng)
    f = float(rng.uniform(0.3, 2.0)) * max(W, H)
    cam = isg.Camera(R, rng.normal(size=3) * 0.2, f,
                     (float(rng.uniform(0, W)), float(rng.uniform(0, H))), W, H)
    # splats in front of the camera in camera space, mapped back to world space
    z = rng.uniform(0.5, 12.0, n)
    u, v = rng.uniform(-0.2 * W, 1.2 * W, n), rng.uniform(-0.2 * H, 1.2 * H, n)
    pc = np.stack([(u - cam.principal_point[0]) * z / f, (v - cam.principal_point[1]) * z / f,
                   z], 1)
    pc[rng.random(n) < 0.05, 2] *= -1  # some behind the camera
    mu = (pc - cam.translation) @ R  # R^T (pc - t)
    s2d = np.exp(rng.uniform(np.log(0.2), np.log(rng.uniform(1.0, 30.0)), n))
    ms = np.concatenate([mu, (s2d * np.abs(z) / f)[:, None]], 1).astype(np.float32)
    co = np.concatenate([rng.uniform(0, 1, (n, 3)), rng.uniform(0.0, 1.0, (n, 1))],
                        1).astype(np.float32)
    opts = isg.RenderOptions(background=tuple(rng.uniform(0, 1, 3)),
                             t_min=float(rng.choice([0.0, 1e-5])))
    bg = opts.background
    rend.set_scene(ms, co)
    rend.set_binning(isg.Renderer.BINNING_TILE_BUCKET)  # the alternative binning: same lists
    rend.render(cam, opts)
    check_bins(rend, ms, co, cam)
    rend.set_binning(isg.Renderer.BINNING_RADIX)
    img = rend.render(cam, opts)
    check_bins(rend, ms, co, cam)
    ref = O.render32(ms, co, cam, bg=bg, t_min=opts.t_min)
    assert np.abs(img - ref).max() <= IMG_TOL + 2.0 * opts.t_min
    target = rng.uniform(0, 1, (H, W, 3)).astype(np.float32)
    loss = rend.loss_backward(cam, target, opts)
    loss_ref, g_ref = O.loss_backward32(ms, co, cam, target, bg=bg, t_min=opts.t_min)
    assert abs(loss - loss_ref) <= 1e-5 * abs(loss_ref) + 1e-12
    _grad_check(rend.grads(), g_ref)
    rend.zero_grads()


def test_count_pairs_matches_oracle_counts(rend):
    """isg_count_pairs (the roofline's algorithmic work) against the FP32 oracle's own counts of
    evaluated and in-circle pixel-entry pairs (termination at t_min: ex2.approx vs expf may
    end a pixel's walk one entry apart, hence the small tolerance)."""
    W, H = 320, 200
    ms, co = isg.synth_scene(30000, W, H, seed=77)
    cam = isg.Camera.synthetic(W, H)
    rend.set_scene(ms, co)
    rend.render(cam)
    ev, inside = rend.count_pairs()
    _, _, _, counts = O.render32(ms, co, cam, want_state=True)
    assert ev == pytest.approx(int(counts[0]), rel=1e-3)
    assert inside == pytest.approx(int(counts[1]), rel=1e-3)

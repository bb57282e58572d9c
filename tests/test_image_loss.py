"""L1 + D-SSIM image loss: the paper's (1-l) L1 + l (1 - SSIM) and its pixel
gradient, /root/reference/proj/src/loss.cpp:16-213.

CPU: the FP64 oracle restatement (oracle/isg_oracle.c or64_image_loss) against the golden
fixtures made by the reference's own compiled loss()/ssim()/ssim_gradient_wrt_second()
(tests/golden/image_loss.npz), against oracle/_ref live when it is built, and against central
finite differences; the reference's error behaviour.
GPU: k_ssim.cu through the C-ABI against the same fixtures, and training with the loss
(render -> loss gradient -> K7 backward) against the oracle pipeline.
"""
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle as O
from paper_2403_14244_b200 import isg

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from make_golden import load_image_loss  # noqa: E402

LOSS_RTOL = 1e-5   # FP32 moments on the GPU vs the FP64 reference
PIXGRAD_TOL = 1e-3  # |dg| <= tol * max|g| elementwise, as the gradient bar of north_star


def ref_pixel_grad(case):
    """dL/dfhat from the fixture: (1-l)/N sign(fhat - f) - l dSSIM/dfhat (loss.cpp:201-213)."""
    f, fh, lam = case["f"], case["fhat"], case["lam"]
    w1 = (1.0 - lam) / f.size
    r = fh - f
    g = np.where(r > 0, w1, np.where(r < 0, -w1, 0.0))
    if lam != 0.0:
        g = g - lam * case["dssim"]
    return g


def test_oracle_matches_reference_fixture():
    for case in load_image_loss():
        loss, g = O.image_loss64(case["f"], case["fhat"], case["lam"], grad=True)
        assert loss == pytest.approx(case["loss"], rel=1e-13, abs=0)
        np.testing.assert_allclose(g, ref_pixel_grad(case), rtol=1e-11, atol=1e-17)
        if case["lam"] != 0.0:  # 1 - ssim recovered from loss and l1
            s = 1.0 - (case["loss"] - (1 - case["lam"]) * case["l1"]) / case["lam"]
            assert s == pytest.approx(case["ssim"], rel=1e-12)


def test_oracle_matches_compiled_reference():
    try:
        O.ref_lib()
    except RuntimeError:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(3)
    for (W, H, lam) in [(11, 12, 0.2), (23, 31, 0.7), (50, 20, 0.0)]:
        f = rng.random((H, W, 3))
        fh = rng.random((H, W, 3))
        loss, l1, ssim, dssim = O.ref_image_loss(f, fh, lam, grad=True)
        ol, og = O.image_loss64(f, fh, lam, grad=True)
        assert ol == loss
        case = dict(f=f, fhat=fh, lam=lam, dssim=dssim)
        np.testing.assert_allclose(og, ref_pixel_grad(case), rtol=1e-12, atol=1e-18)


def test_oracle_gradient_finite_differences():
    rng = np.random.default_rng(11)
    f = rng.random((16, 14, 3))
    fh = np.clip(f + 0.2 * rng.standard_normal(f.shape), 0.05, 0.95)
    _, g = O.image_loss64(f, fh, 0.2, weight=2.0, grad=True)
    for idx in [(7, 9, 1), (0, 0, 0), (15, 13, 2), (5, 5, 0), (3, 12, 1)]:
        if abs(fh[idx] - f[idx]) < 1e-4:
            continue
        e = 1e-6
        p, m = fh.copy(), fh.copy()
        p[idx] += e
        m[idx] -= e
        fd = (O.image_loss64(f, p, 0.2, 2.0) - O.image_loss64(f, m, 0.2, 2.0)) / (2 * e)
        assert fd == pytest.approx(g[idx], rel=1e-5, abs=1e-10)


def test_oracle_errors():
    f = np.zeros((12, 12, 3))
    with pytest.raises(ValueError, match="lambda must be in"):
        O.image_loss64(f, f, 1.5)
    small = np.zeros((10, 12, 3))
    with pytest.raises(ValueError, match="smaller than the 11x11"):
        O.image_loss64(small, small, 0.2)
    assert O.image_loss64(small, small + 0.5, 0.0) == pytest.approx(0.5)  # lambda 0: L1 only
    assert O.image_loss64(f, f, 0.2) == 0.0  # identical images: ssim 1, l1 0


# ---- GPU ------------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def rend():
    r = isg.Renderer(0)
    yield r
    r.close()


@pytest.mark.gpu
def test_gpu_image_loss_matches_reference_fixture(rend):
    import torch
    for case in load_image_loss():
        f = torch.from_numpy(case["f"].astype(np.float32)).cuda()
        fh = torch.from_numpy(case["fhat"].astype(np.float32)).cuda()
        H, W = f.shape[:2]
        # the FP32 images are the inputs: the FP64 expectation is recomputed on them
        exp_loss, exp_g = O.image_loss64(f.cpu().numpy(), fh.cpu().numpy(), case["lam"], 0.5,
                                         grad=True)
        rend.set_loss(isg.LOSS_L1_DSSIM, case["lam"])
        g = torch.empty_like(f)
        loss = rend.image_loss_device(W, H, fh.data_ptr(), f.data_ptr(), 0.5, g.data_ptr())
        assert loss == pytest.approx(exp_loss, rel=LOSS_RTOL)
        assert rend.image_loss_device(W, H, fh.data_ptr(), f.data_ptr(), 0.5) == loss
        g = g.cpu().numpy()
        assert np.abs(g - exp_g).max() <= PIXGRAD_TOL * np.abs(exp_g).max()
        # and against the reference's own numbers directly
        assert loss == pytest.approx(0.5 * case["loss"], rel=1e-4)
    rend.set_loss(isg.LOSS_L2)


@pytest.mark.gpu
def test_gpu_l2_image_loss(rend):
    import torch
    rng = np.random.default_rng(1)
    f = rng.random((37, 29, 3)).astype(np.float32)
    fh = rng.random((37, 29, 3)).astype(np.float32)
    tf, tfh = torch.from_numpy(f).cuda(), torch.from_numpy(fh).cuda()
    g = torch.empty_like(tf)
    rend.set_loss(isg.LOSS_L2)
    loss = rend.image_loss_device(29, 37, tfh.data_ptr(), tf.data_ptr(), 2.0, g.data_ptr())
    assert loss == pytest.approx(2.0 * O.mse64(fh, f), rel=1e-6)
    np.testing.assert_allclose(g.cpu().numpy(), 2.0 * 2.0 * (fh - f) / f.size, rtol=1e-5,
                               atol=1e-9)


@pytest.mark.gpu
def test_gpu_loss_validation(rend):
    import torch
    with pytest.raises(isg.DomainError, match="lambda must be in"):
        rend.set_loss(isg.LOSS_L1_DSSIM, 1.5)
    with pytest.raises(ValueError):
        rend.set_loss(7, 0.2)
    rend.set_loss(isg.LOSS_L1_DSSIM, 0.2)
    x = torch.zeros((10, 40, 3), device="cuda")
    with pytest.raises(isg.DomainError, match="smaller than the 11x11"):
        rend.image_loss_device(40, 10, x.data_ptr(), x.data_ptr())
    ms, co = isg.synth_scene(50, 40, 10, seed=1)
    rend.set_scene(ms, co)
    cam = isg.Camera.synthetic(40, 10)
    with pytest.raises(isg.DomainError, match="smaller than the 11x11"):
        rend.loss_backward(cam, np.zeros((10, 40, 3), np.float32))
    rend.set_loss(isg.LOSS_L1_DSSIM, 0.0)  # L1 alone has no window
    rend.loss_backward(cam, np.zeros((10, 40, 3), np.float32))
    rend.zero_grads()
    rend.set_loss(isg.LOSS_L2)


def _grad_check(g, g_ref, tol=1e-3):
    for sl in (slice(0, 3), slice(3, 4), slice(4, 7), slice(7, 8)):
        a, b = g[:, sl], g_ref[:, sl]
        nb = np.linalg.norm(b)
        assert np.linalg.norm(a - b) <= tol * nb + 1e-12
        assert np.abs(a - b).max() <= tol * np.abs(b).max() + 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("lam", [0.2, 0.0, 1.0])
def test_gpu_train_with_l1_dssim_matches_oracle(rend, lam):
    W, H = 96, 72
    ms, co = isg.synth_scene(2000, W, H, seed=2403)
    tms, tco = isg.synth_scene(2000, W, H, seed=14244)
    cam = isg.Camera.synthetic(W, H, 1, 3)
    target = O.render32(tms, tco, cam)
    rend.set_scene(ms, co)
    rend.set_loss(isg.LOSS_L1_DSSIM, lam)
    loss = rend.loss_backward(cam, target, weight=0.7)
    g = rend.grads()
    # oracle pipeline: FP32 tiled render -> FP64 loss gradient -> FP32 tiled backward
    img = O.render32(ms, co, cam)
    loss_ref, dldc = O.image_loss64(target, img, lam, 0.7, grad=True)
    g_ref = O.backward_dldc32(ms, co, cam, dldc.astype(np.float32))
    assert loss == pytest.approx(loss_ref, rel=LOSS_RTOL)
    _grad_check(g, g_ref)
    # eval_loss agrees with the training loss
    import torch
    t = torch.from_numpy(target).cuda()
    assert rend.eval_loss_device(cam, t.data_ptr(), weight=0.7) == pytest.approx(loss, rel=1e-12)
    rend.zero_grads()
    rend.set_loss(isg.LOSS_L2)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(12))
def test_gpu_image_loss_randomized(rend, seed):
    """Seeded random image sizes (from the 11-pixel window minimum to several ragged 32-pixel
    tiles), lambdas, weights and image statistics: loss and dL/dfhat against the FP64 oracle."""
    import torch
    rng = np.random.default_rng(700 + seed)
    H, W = int(rng.integers(11, 140)), int(rng.integers(11, 140))
    lam = float(rng.choice([0.0, 0.2, float(rng.uniform(0, 1)), 1.0]))
    weight = float(rng.uniform(0.1, 3.0))
    f = rng.uniform(0, 1, (H, W, 3))
    if seed % 3 == 0:  # smooth images: the SSIM terms dominate
        f = np.cumsum(np.cumsum(rng.normal(0, 0.02, (H, W, 3)), 0), 1)
        f = (f - f.min()) / max(f.max() - f.min(), 1e-6)
    fh = np.clip(f + rng.normal(0, float(rng.uniform(0.01, 0.3)), f.shape), 0, 1)
    f32, fh32 = f.astype(np.float32), fh.astype(np.float32)
    exp_loss, exp_g = O.image_loss64(f32, fh32, lam, weight, grad=True)
    tf, tfh = torch.from_numpy(f32).cuda(), torch.from_numpy(fh32).cuda()
    g = torch.empty_like(tf)
    rend.set_loss(isg.LOSS_L1_DSSIM, lam)
    loss = rend.image_loss_device(W, H, tfh.data_ptr(), tf.data_ptr(), weight, g.data_ptr())
    rend.set_loss(isg.LOSS_L2)
    assert loss == pytest.approx(exp_loss, rel=LOSS_RTOL, abs=1e-9)
    g = g.cpu().numpy()
    assert np.abs(g - exp_g).max() <= PIXGRAD_TOL * np.abs(exp_g).max()

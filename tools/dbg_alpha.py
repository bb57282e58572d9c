"""GPU vs FP32-oracle gradients on scenes whose final transmittance is 0 or underflows (an
opacity-1 splat centred on a pixel; a stack of opaque splats at t_min = 0): the K6 re-walk /
K7 select-based start.  Run on the GPU box: python tools/dbg_alpha.py"""
import numpy as np, sys, os
sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import oracle as O
from paper_2403_14244_b200 import isg
from test_gpu_parity import random_scene
for case in ["alpha_one","underflow"]:
    rng = np.random.default_rng(7 if case == "alpha_one" else 8)
    W, H = 64, 48
    ms, co, cam = random_scene(rng, 400, W, H)
    if case == "alpha_one":
        cam = isg.Camera(np.eye(3), np.zeros(3), cam.focal, (20.5, 12.5), W, H)
        extra_ms = np.array([[0.0, 0.0, 1.5, 0.004], [0.0, 0.0, 1.6, 0.01]], np.float32)
        extra_co = np.array([[0.9, 0.2, 0.1, 1.0], [0.1, 0.8, 0.3, 1.0]], np.float32)
    else:
        k = 150
        z = np.linspace(1.2, 1.9, k, dtype=np.float32)
        extra_ms = np.stack([np.full(k, 0.01), np.full(k, -0.01), z, 0.02 * z], 1).astype(np.float32)
        extra_co = np.concatenate([rng.uniform(0, 1, (k, 3)), np.full((k, 1), 0.9)], 1).astype(np.float32)
    ms = np.concatenate([ms, extra_ms]).astype(np.float32)
    co = np.concatenate([co, extra_co]).astype(np.float32)
    tms, tco, _ = random_scene(rng, 400, W, H)
    target = O.render32(tms, tco, cam)
    r = isg.Renderer(0)
    r.set_scene(ms, co)
    for t_min in (0.0, 1e-5):
        opts = isg.RenderOptions(t_min=t_min)
        r.zero_grads()
        loss = r.loss_backward(cam, target, opts, weight=1.0)
        g = r.grads()
        tl, npr = r.debug_pixel_state(W, H)
        loss_ref, g_ref = O.loss_backward32(ms, co, cam, target, t_min=t_min)
        d = np.abs(g - g_ref).max(1)
        bad = np.argsort(-d)[:5]
        print(case, t_min, 'loss', loss, loss_ref, 'neg tl', (tl<0).sum(), 'rel', np.linalg.norm(g-g_ref)/np.linalg.norm(g_ref))
        for i in bad: print('  ', i, g[i], g_ref[i])
        print('  nan', np.isnan(g).sum(), 'tl zero', (tl==0).sum(), 'min |tl|', np.abs(tl[npr>0]).min())
    r.close()

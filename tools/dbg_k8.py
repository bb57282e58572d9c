"""Train C3-like steps and report when parameters go non-finite (K8 stream debugging)."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2403_14244_b200 import isg
import torch
n, W, H = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, 1920, 1080
ms, co = isg.synth_scene(n, W, H, seed=2403)
tms, tco = isg.synth_scene(n, W, H, seed=14244)
cam = isg.Camera.synthetic(W, H)
opts = isg.RenderOptions(t_min=1e-5)
r = isg.Renderer(0, n, W, H)
r.set_scene(tms, tco)
target = r.render(cam, opts)
r.set_scene(ms, co)
for step in range(60):
    loss = r.loss_backward(cam, target, opts)
    r.adam_step(isg.AdamConfig())
    a, b = r.get_scene()
    bad = ~np.isfinite(a).all(1) | (a[:, 3] <= 0) | ~np.isfinite(b).all(1)
    if step % 10 == 0 or bad.any():
        print(step, loss, 'bad', bad.sum(), np.nonzero(bad)[0][:10])
    if bad.any():
        i = np.nonzero(bad)[0][0]; print(a[i], b[i]); break

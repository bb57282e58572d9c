"""Render FPS of the C2 workload at t_min = 1e-5 and at t_min = 0 (one-frame graphs replayed).
Run on the GPU box: python tools/render_tmin.py"""
import sys
sys.path.insert(0, '.')
import torch
from paper_2403_14244_b200 import isg
n, W, H = 1_000_000, 1920, 1080
ms, co = isg.synth_scene(n, W, H, seed=2403)
cam = isg.Camera.synthetic(W, H)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
r = isg.Renderer(0, n, W, H); r.set_stream(s.cuda_stream); r.set_scene(ms, co)
out = torch.empty((H, W, 3), device='cuda')
for tmin in (1e-5, 0.0, 1e-5, 0.0):
    opts = isg.RenderOptions(t_min=tmin)
    r.render_device(cam, opts, out.data_ptr()); r.synchronize()
    r.graph_begin(); r.render_device(cam, opts, out.data_ptr()); g = r.graph_end()
    for _ in range(5): g.launch()
    r.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(200): g.launch()
    e1.record(s); r.synchronize()
    print(f"t_min {tmin}: {200 / e0.elapsed_time(e1) * 1e3:.1f} FPS", flush=True)
    g.close()

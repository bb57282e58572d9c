"""Probe: C4-style 8-view loss_backward passes on one context vs split over two contexts on two
streams (views alternating), each context replaying its own captured graph of its views.
Measures only the view passes (no gradient merge / Adam): the overlap available to lanes."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2403_14244_b200 import isg  # noqa: E402

n, W, H, V = 3_000_000, 1920, 1080, 8
ms, co = isg.synth_scene(n, W, H, seed=2403)
cams = [isg.Camera.synthetic(W, H, v, V) for v in range(V)]
opts = isg.RenderOptions(t_min=1e-5)
tgt = torch.full((H, W, 3), 0.5, device="cuda")


def build(k):
    rs, ss, gs = [], [], []
    for j in range(k):
        s = torch.cuda.Stream()
        r = isg.Renderer(0, n, W, H)
        r.set_stream(s.cuda_stream)
        r.set_scene(ms, co)
        r.loss_backward_device(cams[0], tgt.data_ptr(), opts, 1.0 / V)
        r.synchronize()
        r.zero_grads()
        r.graph_begin()
        for v in range(j, V, k):
            r.loss_backward_device(cams[v], tgt.data_ptr(), opts, 1.0 / V)
        gs.append(r.graph_end())
        rs.append(r); ss.append(s)
    return rs, ss, gs


for k in (1, 2):
    rs, ss, gs = build(k)
    for _ in range(2):
        for g in gs:
            g.launch()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    steps = 10
    e0.record()
    for s in ss:
        s.wait_event(e0)
    for _ in range(steps):
        for g in gs:
            g.launch()
    cur = torch.cuda.current_stream()
    for s in ss:
        ev = torch.cuda.Event(); ev.record(s); cur.wait_event(ev)
    e1.record()
    torch.cuda.synchronize()
    print(f"lanes {k}: {e0.elapsed_time(e1) / steps:.3f} ms per 8 view passes", flush=True)
    for r in rs:
        r.zero_grads()
        r.synchronize()
    del gs

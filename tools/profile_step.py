#!/usr/bin/env python3
"""Minimal driver for ncu captures: C3 (1M splats, 1080p) train steps through the C-ABI with
device-resident inputs, no timing and no CPU work, so `ncu -k regex:...` sees only our
kernels.  Usage: python tools/profile_step.py [--steps 3] [--config c3|c2|c4|c5] [--render]
[--loss l2|l1_dssim]"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2403_14244_b200 import isg  # noqa: E402

SIZES = {"c2": (1_000_000, 1920, 1080), "c3": (1_000_000, 1920, 1080),
         "c4": (3_000_000, 1920, 1080), "c5": (10_000_000, 3840, 2160),
         "small": (10_000, 256, 256)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(SIZES))
    ap.add_argument("--render", action="store_true", help="forward only")
    ap.add_argument("--loss", default="l2", choices=["l2", "l1_dssim"])
    ap.add_argument("--const-target", action="store_true",
                    help="a constant target image (no target render frame: the capture then "
                         "holds only train-step kernels)")
    ap.add_argument("--deterministic", action="store_true")
    a = ap.parse_args()
    n, W, H = SIZES[a.config]
    ms, co = isg.synth_scene(n, W, H, seed=2403)
    tms, tco = isg.synth_scene(n, W, H, seed=14244)
    # c4: the first view of the 8-view batch (one view pass; the batch repeats it 8 times)
    cam = isg.Camera.synthetic(W, H, 0, 8) if a.config == "c4" else isg.Camera.synthetic(W, H)
    opts = isg.RenderOptions(t_min=1e-5)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    r = isg.Renderer(0, n, W, H)
    r.set_stream(stream.cuda_stream)
    if a.loss == "l1_dssim":
        r.set_loss(isg.LOSS_L1_DSSIM, 0.2)
    if a.deterministic:
        r.set_deterministic(True)
    target = torch.empty((H, W, 3), dtype=torch.float32, device="cuda")
    if a.const_target:
        target.fill_(0.5)
    else:
        r.set_scene(tms, tco)
        r.render_device(cam, opts, target.data_ptr())
    r.set_scene(ms, co)
    out = torch.empty_like(target)
    for _ in range(a.steps):
        if a.render:
            r.render_device(cam, opts, out.data_ptr())
        else:
            r.loss_backward_device(cam, target.data_ptr(), opts)
            r.adam_step(isg.AdamConfig())
    r.synchronize()
    print("steps done", a.steps, r.stats())


if __name__ == "__main__":
    main()

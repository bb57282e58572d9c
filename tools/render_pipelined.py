"""Render throughput with frames in flight: k contexts (same scene, own frame buffers and
streams), frames issued round-robin, each context replaying its own one-frame CUDA graph.
Usage: python tools/render_pipelined.py [--ctx 1 2 3] [--frames 200]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2403_14244_b200 import isg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, nargs="+", default=[1, 2, 3])
    ap.add_argument("--frames", type=int, default=200)
    a = ap.parse_args()
    n, W, H = 1_000_000, 1920, 1080
    ms, co = isg.synth_scene(n, W, H, seed=2403)
    cam = isg.Camera.synthetic(W, H)
    opts = isg.RenderOptions(t_min=1e-5)
    for k in a.ctx:
        rs, streams, outs, graphs = [], [], [], []
        for _ in range(k):
            s = torch.cuda.Stream()
            r = isg.Renderer(0, n, W, H)
            r.set_stream(s.cuda_stream)
            r.set_scene(ms, co)
            out = torch.empty((H, W, 3), device="cuda")
            r.render_device(cam, opts, out.data_ptr())  # size buffers before capture
            r.synchronize()
            r.graph_begin()
            r.render_device(cam, opts, out.data_ptr())
            graphs.append(r.graph_end())
            rs.append(r); streams.append(s); outs.append(out)
        for i in range(10):
            graphs[i % k].launch()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(torch.cuda.current_stream())
        for s in streams:
            s.wait_event(e0)
        for i in range(a.frames):
            graphs[i % k].launch()
        for s in streams:
            ev = torch.cuda.Event(); ev.record(s); torch.cuda.current_stream().wait_event(ev)
        e1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        ms_ = e0.elapsed_time(e1)
        print(f"contexts {k}: {a.frames / ms_ * 1e3:.1f} frames/s ({ms_ / a.frames:.3f} ms/frame)",
              flush=True)
        for r in rs:
            r.synchronize()
        del graphs


if __name__ == "__main__":
    main()

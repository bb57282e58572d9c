"""H2D bandwidth of one 1080p RGB float target (25 MB) from pinned memory: one copy on one
stream, and the same bytes split over 2 / 4 streams (several DMA engines at once)."""
import torch

n = 1920 * 1080 * 3
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    parts = [(i * n // k, (i + 1) * n // k) for i in range(k)]
    for _ in range(3):
        for s, (a, b) in zip(streams, parts):
            with torch.cuda.stream(s):
                d[a:b].copy_(h[a:b], non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(40):
        for s in streams:
            s.wait_event(e0) if False else None
        evs = []
        for s, (a, b) in zip(streams, parts):
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                d[a:b].copy_(h[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s)
            evs.append(ev)
        for ev in evs:
            torch.cuda.current_stream().wait_event(ev)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 40
    print(f"H2D {n * 4 / 1e6:.1f} MB over {k} stream(s): {ms:.3f} ms, {n * 4 / ms / 1e6:.1f} GB/s")

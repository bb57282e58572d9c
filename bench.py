#!/usr/bin/env python3
"""Benchmark of the B200 isotropic-splat train step (BASELINE.json metric).

Default workload (config C3, BASELINE.json configs[2]): 1M isotropic Gaussians
(isg-synth v1, seed 2403), one 1920x1080 view per GPU per step, forward + L2 loss + backward
+ Adam, target = render of the seed-14244 scene.  One "step" = one view per GPU + one Adam
step on every replica (gradients all-reduced over NCCL when N > 1): weak scaling.  The same
line carries a `render` object: C2 render FPS (BASELINE metric's second half) of the same
scene and camera, with its own e2e and the reference's own render() beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1|c2|c3|c4|c5]
  python bench.py --impl reference ...   # CPU reference arm (oracle only, all host cores)
  python bench.py --loss l1_dssim        # train with the paper's 0.8 L1 + 0.2 D-SSIM loss

--gpus N > 1 without torchrun's environment re-launches itself under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU, NCCL); under torchrun
WORLD_SIZE must equal --gpus.

`value` is device-resident throughput (inputs in HBM before the timed region); `e2e` is the
same metric through the C-ABI with host buffers (target H2D + loss D2H inside the timed
region).  The roofline object reports the dominant kernel; cpu_baseline times the CPU oracle
(the FP32 tiled restatement) on the box's host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (n_gaussians, W, H, views_per_step_total, train, description)
    "c1": (10_000, 256, 256, 1, True, "synthetic 10K isotropic Gaussians, 256x256, fwd+L2+bwd+Adam"),
    "c2": (1_000_000, 1920, 1080, 1, False, "synthetic 1M isotropic Gaussians, 1920x1080 render"),
    "c3": (1_000_000, 1920, 1080, 1, True,
           "synthetic 1M isotropic Gaussians, 1920x1080, fwd+L2+bwd+Adam, 1 view/GPU/step"),
    "c4": (3_000_000, 1920, 1080, 8, True,
           "synthetic 3M isotropic Gaussians, 1080p, 8-view batch per step sharded over GPUs"),
    "c5": (10_000_000, 3840, 2160, 1, True, "synthetic 10M isotropic Gaussians, 4K fwd+bwd+Adam"),
}
T_MIN = 1e-5        # training configs' early-termination threshold (an opt-in)
RENDER_T_MIN = 0.0  # render FPS (C2, and the render sub-object): the reference's exact
                    # semantics, every covering splat composited (splat3d.cpp:134-141)


def t_min_of(config: str) -> float:
    return RENDER_T_MIN if config == "c2" else T_MIN
METRICS = {  # BASELINE.json's metric, named per workload
    "c1": ("fwd+bwd train iters/sec (10K isotropic Gaussians, 256x256)", "iters/s"),
    "c2": ("render FPS (1M isotropic Gaussians, 1080p)", "frames/s"),
    "c3": ("fwd+bwd train iters/sec (1M isotropic Gaussians, 1080p)", "iters/s"),
    "c4": ("fwd+bwd train iters/sec (3M isotropic Gaussians, 1080p, 8-view batch per iter)",
           "iters/s"),
    "c5": ("fwd+bwd train iters/sec (10M isotropic Gaussians, 4K)", "iters/s"),
}
RENDER_METRIC = METRICS["c2"][0]
LR = [1e-3, 5e-3, 1e-2, 1e-2]  # AdamConfig defaults (lr_mu, lr_sigma, lr_color, lr_opacity)


def workload(config: str, world: int):
    """Per-step work of `config` on `world` GPUs: (views of one step in camera order, the
    number of views each rank renders, iterations one step counts).  C4 is one 8-view batch
    per step split over the ranks (strong scaling, 1 iteration per step); the other configs
    give every rank one view per step (weak scaling, `world` iterations per step)."""
    n, W, H, views_total, train, _ = CONFIGS[config]
    if config == "c4":
        per_rank = max(1, views_total // world)
        return [(v, per_rank * world) for v in range(per_rank * world)], per_rank, 1
    return [(r, world) for r in range(world)], 1, world


def config_dict(args, world: int) -> dict:
    """The `config` object of both arms' JSON lines (identical for the same arguments)."""
    n, W, H, views_total, train, desc = CONFIGS[args.config]
    views, per_rank, _ = workload(args.config, world)
    flush = args.config == "c1"
    return {"workload": desc, "config": args.config, "n_gaussians": n, "width": W, "height": H,
            "views_per_step": len(views), "t_min": t_min_of(args.config),
            "loss": "L2 (mse)" if args.loss == "l2" else "0.8 L1 + 0.2 D-SSIM",
            "binning": args.binning,
            "gradients": ("deterministic (per-pair slots, fixed-order sums)" if
                          getattr(args, "deterministic", False) else
                          "direct (warp pre-reduced, red.global.add into per-splat sums)"),
            "launch": "eager" if args.no_graph else "cuda_graph (one graph launch per step)",
            "parallelism": f"dp{world} (views sharded, scene replicated)",
            "l2": ("L2 flushed between steps (256 MB memset outside the timed intervals)" if flush
                   else "no flush: the per-step working set exceeds the 126 MB L2")}

# Algorithmic FP32 work per (pixel, list entry) pair, FLOPs (FMA = 2), see DESIGN.md §Roofline:
FWD_FLOP_EVAL, FWD_FLOP_IN = 6, 12      # 3-sigma test; exp+alpha+composite+transmittance
BWD_FLOP_EVAL, BWD_FLOP_IN = 6, 36      # same test; transmittance recovery + 7 gradients
FP32_LANES = 148 * 128
NCU_SUMMARY = "profiles/r2/ncu_full_step.json"  # dram traffic per launch, --set full capture


def stage_bytes(n, keys, tiles):
    """Algorithmic DRAM bytes per step of the memory-bound stages:
    K1 32 B read + 56 B written per splat (plus the depth histograms, negligible); depth sort:
    per pass 8 B read + 8 B written per splat (4 passes; K1 built the histograms); scan/emit:
    order + tile count + tile box + slot offset (20 B) per splat, tile key + splat (8 B) per
    key, range init 8 B per tile; tile sort: pass 1 reads the key and writes key + index
    (12 B), the last pass reads key + index, gathers the splat and writes the (splat, slot)
    pair (20 B) per key; K8: 96 B read + 96 B written per splat + 32 B per gradient slot."""
    return {"preprocess": 88 * n, "depth_sort": 4 * 16 * n,
            "scan_emit": 20 * n + 8 * keys + 8 * tiles, "tile_sort": 32 * keys,
            "project_adam": 192 * n + 32 * keys}


def ncu_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of `kernel` from the committed capture."""
    try:
        d = json.loads((ROOT / NCU_SUMMARY).read_text())["kernels"]["k_" + kernel]
        mb = lambda s: float(s.split()[0]) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3}[s.split()[1]]
        return {"bytes": mb(d["dram__bytes_read.sum"]) + mb(d["dram__bytes_write.sum"]),
                "source": NCU_SUMMARY}
    except Exception:
        return None


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled DURING the timed region.

    NVML polled from a thread every ~1 ms (a C3 timed region is ~140 ms, a C1 one ~12 ms), on
    the device found by PCI bus id; falls back to `nvidia-smi -lms 20` when NVML is absent."""

    REASONS = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4)]

    def __init__(self, index: int):
        self.index = index
        self.rows = []          # (sm_mhz, max_mhz, reasons bitmask)
        self.p = None
        self.thread = None
        self.stop = False
        self.source = "unavailable"
        self.out = ROOT / "gpurun_out" / f"clocks_{os.getpid()}.csv"

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _poll(self, pynvml, h):
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while not self.stop:
            sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.rows.append((float(sm), float(mx), int(rs)))
            time.sleep(0.001)

    def __enter__(self):
        try:
            pynvml, h = self._nvml_handle()
            self.rows.append((float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                              float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)),
                              int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))))
            self.rows.clear()
            self.thread = threading.Thread(target=self._poll, args=(pynvml, h), daemon=True)
            self.thread.start()
            self.source = "nvml 1 ms"
            return self
        except Exception:
            self.thread = None
        try:
            self.out.parent.mkdir(exist_ok=True)
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.out, "w"), stderr=subprocess.DEVNULL)
            self.source = "nvidia-smi 20 ms"
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.thread is not None:
            self.stop = True
            self.thread.join(timeout=5)
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
            try:
                for r in self.out.read_text().strip().splitlines():
                    f = [x.strip() for x in r.split(",")]
                    if len(f) >= 3 and f[0].replace(".", "").isdigit():
                        self.rows.append((float(f[0]), float(f[1]), int(f[2], 16)))
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"],
                    "source": self.source}
        reasons = sorted({n for _, _, m in self.rows for n, bit in self.REASONS if m & bit})
        return {"sm_mhz": float(np.median([r[0] for r in self.rows])),
                "sm_max_mhz": max(r[1] for r in self.rows), "reasons": reasons,
                "samples": len(self.rows), "source": self.source}


class CpuTrainer:
    """CPU oracle (FP32 tiled restatement, oracle/isg_oracle.c) train steps: every view of the
    step forward + L2 + backward (weight 1/V), then Adam on (mu, log sigma, rgb, logit o) with
    its persistent optimizer state -- the GPU step's algorithm, on the host's threads."""

    def __init__(self, ms, co, cams, targets, threads=0):
        import oracle as O
        self.O = O
        self.ms, self.co = ms.copy(), co.copy()
        self.m = np.zeros((ms.shape[0], 8), np.float32)
        self.v = np.zeros_like(self.m)
        self.raw = O.raw_init32(self.ms, self.co)
        self.cams, self.targets, self.threads, self.t = cams, targets, threads, 0

    def step(self) -> float:
        """One step; returns its seconds."""
        t0 = time.perf_counter()
        g = np.zeros((self.ms.shape[0], 8), np.float32)
        w = 1.0 / len(self.cams)
        for c, tg in zip(self.cams, self.targets):
            self.O.loss_backward32(self.ms, self.co, c, tg, t_min=T_MIN, weight=w,
                                   threads=self.threads, grads=g)
        self.t += 1
        self.O.adam32(self.ms, self.co, self.m, self.v, g, self.t, LR, 0.9, 0.999, 1e-15,
                      raw=self.raw)
        return time.perf_counter() - t0


def reference_render_fps(ms, co, cam, cores):
    """The reference's OWN render() (oracle/_ref: src/splat3d.cpp:173-194 compiled unmodified;
    rows split into `threads` bands, :148-160) timed on a bounded sample and extrapolated to the
    full frame.  A sub-image is the same camera with the principal point shifted, so its pixels
    are exactly the frame's.  F = a 1x1 image (projection + sort of every splat, the per-call
    fixed cost); B = a band of `cores` rows (every thread composites one full row); the full
    frame is F + (B - F) * H / cores (each thread then composites H / cores rows).
    Returns (frames/s, sample description) or None when oracle/_ref is not built."""
    import oracle as O
    try:
        O.ref_lib()
    except Exception:
        return None
    sp = np.concatenate([ms, co], 1).astype(np.float64)
    W, H = cam.width, cam.height
    cx, cy = cam.principal_point
    rows = max(1, min(cores, H))

    def sub(w, h, x0, y0):
        c = O.Camera(np.asarray(cam.rotation), np.asarray(cam.translation), cam.focal,
                     (cx - x0, cy - y0), w, h)
        t0 = time.perf_counter()
        O.ref_render(sp, c, threads=cores)
        return time.perf_counter() - t0

    fixed = sub(1, 1, W // 2, H // 2)
    band = sub(W, rows, 0, H // 2 - rows // 2)
    full = fixed + max(band - fixed, 0.0) * H / rows
    return 1.0 / full, (f"the reference's own render() (oracle/_ref, src/splat3d.cpp:173-194, "
                        f"FP64, every pixel tests every splat) with threads={cores}: a 1x1 image "
                        f"({fixed:.2f} s, projection + sort) and a {rows}-row band "
                        f"({band:.2f} s, one row per thread); full {W}x{H} frame extrapolated "
                        f"to {full:.1f} s")


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1




def reference_train_line(args, world):
    """The CPU oracle's train steps on this run's workload (all of a step's views + Adam),
    bounded to ~60 s of timed steps.  Returns (iters/s, sample, steps timed, s/step)."""
    import oracle as O
    n, W, H, _, _, _ = CONFIGS[args.config]
    views, _, iters = workload(args.config, world)
    ms, co = O.synth_scene(n, W, H, seed=2403)
    tms, tco = O.synth_scene(n, W, H, seed=14244)
    cams = [O.synth_camera(W, H, v, nv) for v, nv in views]
    cores = host_threads()
    targets = [O.render32(tms, tco, c, t_min=T_MIN, threads=cores) for c in cams]
    tr = CpuTrainer(ms, co, cams, targets, threads=cores)
    first = tr.step()  # warm-up step
    steps = max(1, min(args.steps, int(60.0 / max(first, 1e-3))))
    sec = float(np.median([tr.step() for _ in range(steps)]))
    sample = (f"{steps} full {args.config.upper()} train steps ({len(views)} view(s) of "
              f"fwd+L2+bwd, then Adam) of the FP32 tiled CPU oracle, median; the reference "
              f"itself has no 3D backward (SPEC.md:484)")
    return iters / sec, sample, steps, sec


def run_reference(args):
    """--impl reference: the CPU path on the host cores, rank 0 only, from the oracle alone
    (oracle/ restates the synthetic workload; the product library is not loaded)."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    import oracle as O
    n, W, H, _, train, _ = CONFIGS[args.config]
    metric, unit = METRICS[args.config]
    cores = host_threads()
    base = {"impl": "reference", "metric": metric, "unit": unit, "n_gpus": world,
            "warmup": 1, "higher_is_better": True,
            "scaling": "strong" if args.config == "c4" else "weak", "vs_baseline": None,
            "data": "synthetic (isg-synth v1: scene seed 2403, target seed 14244; oracle restatement)",
            "config": config_dict(args, world), "gpu_launches": 0}
    ref_render = None
    if n <= 1_000_000 and W * H <= 1920 * 1080:
        # the reference's own render() (FP64, every pixel tests every splat), extrapolated
        ms, co = O.synth_scene(n, W, H, seed=2403)
        ref_render = reference_render_fps(ms, co, O.synth_camera(W, H), cores)
    if not train:
        if ref_render is None:
            print(json.dumps({"impl": "reference", "unavailable":
                              "oracle/_ref (the reference's render) was not built"}), flush=True)
            return
        fps, sample = ref_render
        line = dict(base, value=fps * world, steps=1, ms_per_step=1e3 / fps, dtype="f64",
                    cpu_baseline={"value": fps * world, "unit": unit, "cores": cores,
                                  "kind": "reference", "sample": sample},
                    e2e={"value": fps * world, "unit": unit, "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0})
        print(json.dumps(line), flush=True)
        return
    val, sample, steps, sec = reference_train_line(args, world)
    line = dict(base, value=val, steps=steps, steps_requested=args.steps, ms_per_step=sec * 1e3,
                dtype="f32",
                cpu_baseline={"value": val, "unit": unit, "cores": cores, "kind": "port",
                              "sample": sample},
                e2e={"value": val, "unit": unit, "h2d_bytes_per_step": 0,
                     "d2h_bytes_per_step": 0})
    if ref_render is not None and args.config == "c3":
        line["render"] = {"metric": RENDER_METRIC, "value": ref_render[0], "unit": "frames/s",
                          "cpu_baseline": {"value": ref_render[0], "unit": "frames/s",
                                           "cores": cores, "kind": "reference",
                                           "sample": ref_render[1]}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
def time_render(r, cam, opts, steps, warmup, stream, barrier, world):
    """C2-style render timing on the resident scene: device-resident FPS (one graph launch
    per frame, CUDA events) and end-to-end FPS (each frame's image copied to pinned host
    memory on a copy stream while the next frames render; NB images in flight).  Returns a
    dict."""
    import torch
    import torch.distributed as dist

    from paper_2403_14244_b200 import isg
    W, H = cam.width, cam.height
    NB = 3
    bufs = [torch.empty((H, W, 3), dtype=torch.float32, device="cuda") for _ in range(NB)]
    host = [torch.empty((H, W, 3), dtype=torch.float32).pin_memory() for _ in range(NB)]
    r.render(cam, opts)  # sizes the buffers (untimed)
    graphs = []
    for b in range(NB):
        r.graph_begin()
        r.render_device(cam, opts, bufs[b].data_ptr())
        graphs.append(r.graph_end())
    for _ in range(max(warmup, 3)):
        graphs[0].launch()
    r.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    l0 = r.stats()["kernel_launches"]
    barrier()
    ev[0].record(stream)
    for i in range(steps):
        graphs[i % NB].launch()
    ev[1].record(stream)
    barrier()
    r.synchronize()
    launches = r.stats()["kernel_launches"] - l0
    dev_ms = ev[0].elapsed_time(ev[1]) / steps
    # end to end through the C-ABI alone: frame i rendered into the library's image ring slot
    # i % NB and copied to pinned host image i % NB on the library's copy stream
    # (isg_render_host_async) while the next frames render; isg_image_wait before a host
    # buffer is reused (kernel by kernel: the ring call is not captured)
    outs = [h.numpy() for h in host]
    for b in range(NB):  # size the ring slots (untimed)
        r.render_host_async(cam, b, outs[b], opts)
    for b in range(NB):
        r.image_wait(b)
    barrier()
    t0 = time.perf_counter()
    for i in range(steps):
        b = i % NB
        if i >= NB:
            r.image_wait(b)  # frame i - NB is on the host: its buffer is free
        r.render_host_async(cam, b, outs[b], opts)
    for b in range(NB):
        r.image_wait(b)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / steps
    # frames in flight: a second context on the same scene with its own frame buffers and
    # stream; one-frame graphs of the two contexts launched alternately, so one frame's
    # latency-bound binning overlaps the other's blending (throughput, not latency)
    ms_, co_ = r.get_scene()
    r2 = isg.Renderer(0, len(ms_), W, H)
    s2 = torch.cuda.Stream()
    r2.set_stream(s2.cuda_stream)
    r2.set_scene(ms_, co_)
    out2 = torch.empty((H, W, 3), dtype=torch.float32, device="cuda")
    r2.render_device(cam, opts, out2.data_ptr())
    r2.synchronize()
    r2.graph_begin()
    r2.render_device(cam, opts, out2.data_ptr())
    g2 = r2.graph_end()
    pair = [graphs[0], g2]
    for i in range(4):
        pair[i % 2].launch()
    r.synchronize()
    r2.synchronize()
    evp = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    barrier()
    evp[0].record(stream)
    s2.wait_event(evp[0])
    for i in range(steps):
        pair[i % 2].launch()
    join = torch.cuda.Event()
    join.record(s2)
    stream.wait_event(join)
    evp[1].record(stream)
    r.synchronize()
    r2.synchronize()
    pipe_ms = evp[0].elapsed_time(evp[1]) / steps
    g2.close()
    r2.close()
    for g in graphs:
        g.close()
    r.synchronize()
    if world > 1:
        tt = torch.tensor([pipe_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        pipe_ms = float(tt.item())
    if world > 1:
        tt = torch.tensor([dev_ms, e2e_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dev_ms, e2e_ms = (float(x) for x in tt.tolist())
    return {"metric": RENDER_METRIC, "value": world * 1e3 / dev_ms, "unit": "frames/s",
            "ms_per_frame": dev_ms, "frames": steps, "gpu_launches": int(launches),
            "t_min": opts.t_min,
            "two_frames_in_flight": {
                "value": world * 1e3 / pipe_ms, "unit": "frames/s", "ms_per_frame": pipe_ms,
                "mode": "two contexts on the same scene (own frame buffers and streams), "
                        "one-frame graphs launched alternately: throughput with one frame's "
                        "binning overlapping the other's blend; `value` above is one frame "
                        "at a time"},
            "e2e": {"value": world * 1e3 / e2e_ms, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": W * H * 3 * 4,
                    "mode": f"C-ABI only: isg_render_host_async into one of {NB} slots of the "
                            "library's image ring, each image copied to pinned host memory on "
                            "the library's copy stream while the next frames render, "
                            "isg_image_wait before a host buffer is reused (every copy complete "
                            "inside the timed region); kernel by kernel"}}


def run_isg(args):
    import torch
    import torch.distributed as dist

    from paper_2403_14244_b200 import isg

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL's communicator lines (rank count, transport) on stdout for the driver to check
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, W, H, views_total, train, desc = CONFIGS[args.config]
    metric, unit = METRICS[args.config]
    views, per_rank, iters_per_step = workload(args.config, world)
    step_views = len(views)
    # a real (non-legacy) stream: the context launches on it and the events below time it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    ms, co = isg.synth_scene(n, W, H, seed=2403)
    tms, tco = isg.synth_scene(n, W, H, seed=14244)
    r = isg.Renderer(local, n, W, H)
    r.set_stream(stream.cuda_stream)
    if args.loss == "l1_dssim":
        r.set_loss(isg.LOSS_L1_DSSIM, 0.2)
    if args.binning == "bucket":
        r.set_binning(r.BINNING_TILE_BUCKET)
    if args.deterministic:
        r.set_deterministic(True)
    opts = isg.RenderOptions(t_min=t_min_of(args.config))
    cfg = isg.AdamConfig()
    my_views = views[rank * per_rank:(rank + 1) * per_rank]
    cams = [isg.Camera.synthetic(W, H, v, nv) for v, nv in my_views]
    # targets: renders of the target scene, resident in HBM
    targets = []
    r.set_scene(tms, tco)
    for c in cams:
        t = torch.empty((H, W, 3), dtype=torch.float32, device="cuda")
        r.render_device(c, opts, t.data_ptr())
        targets.append(t)
    r.synchronize()
    r.set_scene(ms, co)
    nccl = None
    p = torch.cuda.get_device_properties(local)
    devices = [f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}"]
    if world > 1:
        uid = r.nccl_unique_id() if rank == 0 else b"\0" * 128
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        r.nccl_init(world, rank, obj[0])
        info = r.nccl_info()
        gathered = [None] * world
        dist.all_gather_object(gathered, (info, devices[0]))
        nccl = {"comm_nranks": [g[0]["nranks"] for g in gathered],
                "comm_ranks": [g[0]["rank"] for g in gathered],
                "nccl_version": info["nccl_version"],
                "exchange": "pipelined chunked all-reduce (isg_adam_step)"}
        devices = [g[1] for g in gathered]
        if any(c != world for c in nccl["comm_nranks"]):
            raise SystemExit(f"bench: NCCL communicator size {nccl['comm_nranks']} != {world}")

    def step():
        if train:
            for c, t in zip(cams, targets):
                r.loss_backward_device(c, t.data_ptr(), opts, weight=1.0 / step_views)
            r.adam_step(cfg)
        else:
            r.render_device(cams[0], opts, targets[0].data_ptr())

    # one synchronous frame sizes the key buffers (capacity growth happens here, untimed)
    if train:
        r.loss_backward(cams[0], targets[0].cpu().numpy(), opts, weight=1.0 / step_views)
        r.zero_grads()
    else:
        r.render(cams[0], opts)
    for _ in range(max(args.warmup, 3)):
        step()
    r.synchronize()
    step_eager = step
    graph = None
    if not args.no_graph:
        # the whole step (every view's frame + backward, the exchange, Adam) as one CUDA graph
        # launch; a replay re-runs every kernel on the live buffers
        r.graph_begin()
        step_eager()
        graph = r.graph_end()

        def step():
            graph.launch()
        for _ in range(2):
            step()
        r.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timed region ----------------------------------------------------
    # A step whose working set (scene + Adam state, keys and their (splat, slot) pairs, the
    # per-pixel images) exceeds the 126 MB L2 runs back to back.  A smaller one (C1) gets an
    # L2 flush (a 256 MB memset) between steps, outside the per-step event pairs.
    n_keys = r.stats()["n_keys"]
    working_set = n * 104 + n_keys * 24 + W * H * (3 * 4 * 2 + 8)
    flush = args.config == "c1"
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if flush else None
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)] if flush else None
    if train:
        # the stage-timing pass and the end-to-end region below restart from this state, so
        # all three measure the same training trajectory (the scene evolves under Adam)
        r.snapshot()
    barrier()
    launches_t0 = r.stats()["kernel_launches"]
    with ClockSampler(local) as clocks:
        ev[0].record(stream)
        for i in range(args.steps):
            if flush:
                flush_buf.zero_()
                ev_s[i].record(stream)
            step()
            ev[i + 1].record(stream)
        barrier()
    r.synchronize()  # surfaces overflow / validation errors of the async frames
    if flush:
        step_ms = [ev_s[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
        total_ms = float(sum(step_ms))
    else:
        step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
        total_ms = ev[0].elapsed_time(ev[-1])
    if world > 1:
        tt = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_per_step = total_ms / args.steps
    value = (iters_per_step if train else world) / (ms_per_step / 1e3)
    launches_timed = r.stats()["kernel_launches"] - launches_t0

    # ---- stage timing (separate pass, events per kernel, kernel by kernel) ----------------
    if train:
        r.restore()
    r.profile(True)
    r.profile_read()
    prof_steps = args.steps  # the same trajectory as the timed region (the scene trains)
    for _ in range(prof_steps):
        step_eager()
    prof = r.profile_read()
    r.profile(False)

    # ---- end to end through the public API with host buffers ------------------------------
    # --e2e ring (default): the C-ABI target ring, no torch copies; --e2e graph: one CUDA
    # graph per step with torch copies of the targets on a side stream (round-2 first session).
    if args.e2e == "graph":
        # Train: every step uploads its targets from pinned host memory and reads its loss back;
        # step i+2's upload runs on a copy stream into the third of three target buffers while
        # step i computes (the prefetch a training loop does), and the host reads step i-1's loss
        # (copied D2H inside step i-1's graph) while step i runs.  Render: time_render().
        # --no-graph: isg_loss_backward with the host target per view + Adam + sync.
        host_targets = [t.cpu().numpy() for t in targets]
        pinned = [torch.from_numpy(h).pin_memory() for h in host_targets]
        host_views = [p.numpy() for p in pinned]
        use_pipe = train and graph is not None
        NB = 3  # target buffers: step i+2's upload may start once step i-1 is done
        step_losses = []
        if use_pipe:
            bufs = [[torch.empty_like(t) for t in targets] for _ in range(NB)]
            loss_host = torch.zeros(NB, dtype=torch.float64).pin_memory()
            graphs = []
            for b in range(NB):
                def step_b(bb=bufs[b], slot=loss_host[b:b + 1]):
                    for c, t in zip(cams, bb):
                        r.loss_backward_device(c, t.data_ptr(), opts, weight=1.0 / step_views)
                    r.adam_step(cfg)
                    r.step_loss_async(slot.data_ptr())  # the step's loss D2H, inside the graph
                for t, h in zip(bufs[b], pinned):
                    t.copy_(h)
                r.graph_begin()
                step_b()
                graphs.append(r.graph_end())
            copy_stream = torch.cuda.Stream()
            ev_copy = [torch.cuda.Event() for _ in range(NB)]
            ev_done = [torch.cuda.Event() for _ in range(NB)]
            r.synchronize()
        e2e = None
        if train:
            r.restore()
            barrier()
            l0 = r.stats()["kernel_launches"]
            t_start = time.perf_counter()
            if use_pipe:
                with torch.cuda.stream(copy_stream):
                    for k in range(min(NB - 1, args.steps)):
                        for t, h in zip(bufs[k], pinned):
                            t.copy_(h, non_blocking=True)
                        ev_copy[k].record(copy_stream)
            for i in range(args.steps):
                if use_pipe:
                    b = i % NB
                    stream.wait_event(ev_copy[b])
                    graphs[b].launch()
                    ev_done[b].record(stream)
                    if i + NB - 1 < args.steps:  # prefetch step i+2's inputs once step i-1 is done
                        nb = (i + NB - 1) % NB
                        with torch.cuda.stream(copy_stream):
                            copy_stream.wait_event(ev_done[nb])
                            for t, h in zip(bufs[nb], pinned):
                                t.copy_(h, non_blocking=True)
                            ev_copy[nb].record(copy_stream)
                    if i >= 1:  # step i-1's loss is on the host once its graph is done
                        pb = (i - 1) % NB
                        ev_done[pb].synchronize()
                        step_losses.append(float(loss_host[pb]))
                else:
                    for c, h in zip(cams, host_views):
                        r.loss_backward(c, h, opts, weight=1.0 / step_views)  # H2D target, D2H loss
                    r.adam_step(cfg)
                    r.synchronize()
            if use_pipe:
                ev_done[(args.steps - 1) % NB].synchronize()
                step_losses.append(float(loss_host[(args.steps - 1) % NB]))
            e2e_step = (time.perf_counter() - t_start) * 1e3 / args.steps
            launches_per_step = (r.stats()["kernel_launches"] - l0) / args.steps
            if world > 1:
                tt = torch.tensor([e2e_step], device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                e2e_step = float(tt.item())
            e2e = {"value": iters_per_step / (e2e_step / 1e3), "unit": unit,
                   "h2d_bytes_per_step": sum(h.nbytes for h in host_views),
                   "d2h_bytes_per_step": 8 if use_pipe else 8 * len(host_views),
                   "ms_per_step": e2e_step, "gpu_launches_per_step": launches_per_step,
                   **({"loss_first_last": [step_losses[0], step_losses[-1]],
                       "losses_read": len(step_losses)} if use_pipe else {}),
                   "mode": ("cuda graph per step, targets prefetched two steps ahead from pinned "
                            "host memory on a copy stream (3 buffers); every step's loss copied "
                            "D2H into pinned memory inside its graph and read by the host while "
                            "the next step runs (all reads inside the timed region)") if use_pipe
                   else "isg_loss_backward with host targets per view + adam_step + sync"}

    else:
        # Train: every step uploads its targets from pinned host memory through the C-ABI's target
        # ring (isg_upload_target_async: step i+2's views on the library's copy stream while step i
        # computes; isg_loss_backward_slot: only the backward waits for its upload) and reads its
        # loss back (isg_step_loss_async into pinned memory; the host reads step i-1's loss while
        # step i runs).  No torch copy is involved (torch events only tell the host when a loss
        # landed).  Render: time_render().  --no-graph: isg_loss_backward (synchronous) per view.
        host_targets = [t.cpu().numpy() for t in targets]
        pinned = [torch.from_numpy(h).pin_memory() for h in host_targets]
        host_views = [p.numpy() for p in pinned]
        use_pipe = train and graph is not None
        NB = 3  # ring slots per view: step i+2's upload may start once step i-1 has read its slot
        step_losses = []
        if use_pipe:
            loss_host = torch.zeros(NB, dtype=torch.float64).pin_memory()
            ev_done = [torch.cuda.Event() for _ in range(NB)]

            def upload(i):  # step i's views into ring slots (i % NB) * views + v
                for v, h in enumerate(host_views):
                    r.upload_target_async((i % NB) * len(host_views) + v, h)

            def ring_step(i):
                for v, c in enumerate(cams):
                    r.loss_backward_slot(c, (i % NB) * len(cams) + v, opts, weight=1.0 / step_views)
                r.adam_step(cfg)
                r.step_loss_async(loss_host[i % NB:i % NB + 1].data_ptr())
            if len(host_views) * NB > isg.TARGET_SLOTS:
                raise SystemExit(f"bench: {len(host_views)} views need {len(host_views) * NB} target "
                                 f"ring slots (ISG_TARGET_SLOTS = {isg.TARGET_SLOTS})")
            for i in range(NB):  # allocate the slots outside the timed region
                upload(i)
            r.synchronize()
            ring_graphs = []  # step b of the ring, captured once per slot set (slot fixed)
            for b in range(NB):
                r.graph_begin()
                ring_step(b)
                ring_graphs.append(r.graph_end())
        e2e = None
        if train:
            r.restore()
            barrier()
            l0 = r.stats()["kernel_launches"]
            t_start = time.perf_counter()
            if use_pipe:
                for k in range(min(NB - 1, args.steps)):
                    upload(k)
            for i in range(args.steps):
                if use_pipe:
                    if i + NB - 1 < args.steps:  # step i+2's upload waits for step i-1's reads
                        upload(i + NB - 1)
                    ring_graphs[i % NB].launch()
                    ev_done[i % NB].record(stream)
                    if i >= 1:  # step i-1's loss is on the host once its work is done
                        pb = (i - 1) % NB
                        ev_done[pb].synchronize()
                        step_losses.append(float(loss_host[pb]))
                else:
                    for c, h in zip(cams, host_views):
                        r.loss_backward(c, h, opts, weight=1.0 / step_views)  # H2D target, D2H loss
                    r.adam_step(cfg)
                    r.synchronize()
            if use_pipe:
                ev_done[(args.steps - 1) % NB].synchronize()
                step_losses.append(float(loss_host[(args.steps - 1) % NB]))
            e2e_step = (time.perf_counter() - t_start) * 1e3 / args.steps
            launches_per_step = (r.stats()["kernel_launches"] - l0) / args.steps
            if world > 1:
                tt = torch.tensor([e2e_step], device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                e2e_step = float(tt.item())
            e2e = {"value": iters_per_step / (e2e_step / 1e3), "unit": unit,
                   "h2d_bytes_per_step": sum(h.nbytes for h in host_views),
                   "d2h_bytes_per_step": 8 if use_pipe else 8 * len(host_views),
                   "ms_per_step": e2e_step, "gpu_launches_per_step": launches_per_step,
                   **({"loss_first_last": [step_losses[0], step_losses[-1]],
                       "losses_read": len(step_losses)} if use_pipe else {}),
                   "mode": ("C-ABI only: targets uploaded from pinned host memory two steps ahead "
                            "into the library's target ring (isg_upload_target_async on its copy "
                            "stream, isg_loss_backward_slot), every step's loss copied D2H into "
                            "pinned memory (isg_step_loss_async) and read by the host while the "
                            "next step runs (all reads inside the timed region); one CUDA graph "
                            "launch per step, captured once per ring slot set") if use_pipe
                   else "isg_loss_backward with host targets per view + adam_step + sync"}

    # ---- render FPS (C2): BASELINE's second metric on the same scene and camera ------------
    render = None
    if not train or args.config == "c3":
        if train:
            r.restore()  # the untrained seed-2403 scene: exactly C2's workload
        render = time_render(r, cams[0], isg.RenderOptions(t_min=RENDER_T_MIN),
                             max(args.steps, 50), args.warmup, stream,
                             barrier, world)
        if not train:  # C2 itself: `value` is the timed region above, e2e the pipelined frames
            e2e = dict(render["e2e"], ms_per_step=1e3 * world / render["e2e"]["value"])
    st = r.stats()
    if rank != 0:
        r.close()
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel ----------------------------------------------------
    peaks, peak_kind = load_peaks()
    top = max(prof.items(), key=lambda kv: kv[1][0])
    top_name, (top_ms_total, top_calls) = top
    top_ms = top_ms_total / max(top_calls, 1)
    roof = {"kernel": top_name, "stage_ms_per_step": {k: v[0] / prof_steps for k, v in prof.items()}}
    # algorithmic work of the blend kernels (roofline): view 0 of the current scene, every
    # pixel walking its list until termination, counted on the GPU (isg_count_pairs), outside
    # every timed region
    count_img = torch.empty((H, W, 3), dtype=torch.float32, device="cuda")
    r.render_device(cams[0], opts, count_img.data_ptr())
    pairs = r.count_pairs()
    del count_img
    cpu = None
    cores = host_threads()
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle as O
        cam0 = cams[0]
        ms_now, co_now = r.get_scene()
        if train:
            tr = CpuTrainer(ms_now, co_now, [cam0], [host_targets[0]], threads=cores)
            sec = tr.step()
            cpu = {"value": 1.0 / sec, "unit": unit, "cores": cores, "kind": "port",
                   "sample": f"1 full {args.config.upper()} train step (fwd+L2+bwd+Adam, one "
                             "view) of the FP32 tiled CPU oracle"}
        if render is not None and n <= 1_000_000:
            # the reference's own renderer is the render baseline
            res = reference_render_fps(ms, co, cam0, cores)
            if res is not None:
                render["cpu_baseline"] = {"value": res[0], "unit": "frames/s", "cores": cores,
                                          "kind": "reference", "sample": res[1]}
                if not train:
                    cpu = render["cpu_baseline"]
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    if top_name in ("blend_fwd", "blend_bwd") and pairs:
        ev_p, in_p = pairs
        flops = (FWD_FLOP_EVAL * ev_p + FWD_FLOP_IN * in_p) if top_name == "blend_fwd" else \
            (BWD_FLOP_EVAL * ev_p + BWD_FLOP_IN * in_p)
        achieved = flops / (top_ms / 1e3) / 1e12
        peak = 2 * FP32_LANES * sm_mhz * 1e6 / 1e12
        roof.update({"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(top_name),
                     "work": f"{flops:.3e} algorithmic FP32 FLOP/launch ({ev_p} evaluated + "
                             f"{in_p} in-circle pixel-splat pairs)",
                     "peak_kind": f"spec FP32 FMA rate at the measured sm_max_mhz {sm_mhz:.0f}"})
    else:
        gb = stage_bytes(n, st["n_keys"], st["n_tiles"]).get(top_name)
        if gb:
            achieved = gb / (top_ms / 1e3) / 1e9
            roof.update({"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                         "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                         "peak_kind": peak_kind})
    # every memory-bound stage against HBM: algorithmic bytes of one frame (the last frame's
    # key count) / CUDA-event time per call (a multi-view step calls the frame stages per view)
    call_ms = {k: v[0] / max(v[1], 1) for k, v in prof.items()}
    roof["hbm_stages"] = {
        k: {"ms_per_call": call_ms[k], "bytes": b, "GB/s": b / (call_ms[k] / 1e3) / 1e9,
            "frac": b / (call_ms[k] / 1e3) / 1e9 / peaks["hbm_gbs"]}
        for k, b in stage_bytes(n, st["n_keys"], st["n_tiles"]).items()
        if call_ms.get(k, 0) > 0}
    roof["ms_per_launch"] = top_ms

    clk = clocks.summary()
    line = {
        "metric": metric, "value": value, "unit": unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "ms_per_step_median": float(np.median(step_ms)),
        "higher_is_better": True, "scaling": "strong" if args.config == "c4" else "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (isg-synth v1: scene seed 2403, target seed 14244)",
        "config": config_dict(args, world),
        "l2_working_set_mb": working_set / 1e6,
        "iters_per_step": iters_per_step, "views_per_step": step_views,
        "e2e": e2e,
        "gpu_launches": int(launches_timed),
        "gpu_launches_per_step": launches_timed / args.steps,
        "gpus_active": world, "devices": devices,
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clk,
        "stats": {"n_visible": st["n_visible"], "n_keys": st["n_keys"],
                  "pairs_evaluated": pairs[0] if pairs else None,
                  "pairs_in_circle": pairs[1] if pairs else None},
    }
    if args.config == "c4":
        line["views_per_s"] = step_views / (ms_per_step / 1e3)
    if train and render is not None:
        line["render"] = render
    if not train and render is not None:  # C2: the frames-in-flight throughput beside `value`
        line["two_frames_in_flight"] = render["two_frames_in_flight"]
    if nccl is not None:
        line["nccl"] = nccl
    print(json.dumps(line), flush=True)
    r.close()
    if world > 1:
        dist.destroy_process_group()


def free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_command(argv, gpus: int, port: int):
    """The torchrun command a `--gpus N` run without torchrun's environment re-launches."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={gpus}", "--master-addr", "127.0.0.1", f"--master-port={port}",
            str(Path(__file__).resolve()), *argv]


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="isg", choices=["isg", "reference"])
    ap.add_argument("--e2e", default="ring", choices=["ring", "graph"],
                    help="end-to-end path: the C-ABI target ring (default) or CUDA graphs with "
                         "torch-side target copies")
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the device-resident step kernel by kernel (no CUDA graph)")
    ap.add_argument("--binning", default="radix", choices=["radix", "bucket"],
                    help="binning strategy (identical tile lists)")
    ap.add_argument("--deterministic", action="store_true",
                    help="slot-mode gradient accumulation (bitwise deterministic, slower)")
    ap.add_argument("--loss", default="l2", choices=["l2", "l1_dssim"],
                    help="training loss (BASELINE configs use L2; l1_dssim = the paper's loss)")
    argv = sys.argv[1:] if argv is None else argv
    args = ap.parse_args(argv)
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
                  f"(torchrun --nproc-per-node {args.gpus}) or drop --gpus", file=sys.stderr)
            return 2
    elif args.gpus > 1:
        # one process per GPU: re-launch under torchrun (rank 0 prints the line)
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        return subprocess.call(spawn_command(argv, args.gpus, free_port()), env=env)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_isg(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())

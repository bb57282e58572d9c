#!/usr/bin/env python3
"""Time one adaptive-control pass (prune / merge / split, k_adapt.cu) on the C3 scene
(1M isg-synth splats) with parameters that trigger all three rules.  Wall clock around the
synchronous C-ABI call (it synchronises internally), after one warm-up pass on a copy."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

from paper_2403_14244_b200 import isg  # noqa: E402


def main():
    n, W, H = 1_000_000, 1920, 1080
    ms, co = isg.synth_scene(n, W, H, seed=2403)
    prm = isg.AdaptParams(prune_threshold=0.1, merge_distance_factor=2.0, merge_color_tol=0.3,
                          split_sigma_max=0.05, max_particles=1_100_000)
    r = isg.Renderer(0, n, W, H)
    for rep in range(3):
        r.set_scene(ms, co)
        t0 = time.perf_counter()
        res = r.adaptive_control(prm, seed=1, round_=rep)
        dt = time.perf_counter() - t0
        print(f"rep {rep}: {dt * 1e3:.1f} ms  {res}", flush=True)


if __name__ == "__main__":
    main()

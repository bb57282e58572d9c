"""The multi-rank view-batch step with the real library on the GPU (world_size 2, one process
per rank, both on cuda:0).  The per-view gradients come from libisg's kernels; the reduction
between the ranks runs on the host through gloo (isg_get_grads -> all_reduce -> isg_set_grads)
instead of NCCL, so no kernel of one rank waits for the other's.  Checks, as the CPU test does
for the oracle backend (tests/test_multi_rank.py):
  * every view is processed by exactly one rank per step,
  * the replicas stay bitwise identical (same reduced gradients, same Adam),
  * 2 ranks reproduce one process training on the whole batch (up to the summation order of
    the view gradients),
  * the reported step loss is the global batch loss.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2403_14244_b200 import isg
from paper_2403_14244_b200.view_batch import ViewBatchDriver

pytestmark = pytest.mark.gpu

W, H, N, VIEWS, STEPS = 96, 64, 4000, 4, 3


class GlooRendererBackend:
    """libisg per-view gradients; host all-reduce through gloo; libisg Adam."""

    def __init__(self, r, cams, targets, opts, adam, world):
        self.r, self.cams, self.targets = r, cams, targets
        self.opts, self.adam, self.world = opts, adam, world
        self.seen = []

    def loss_backward(self, view, weight):
        self.seen.append(view)
        self.r.loss_backward_device(self.cams[view], self.targets[view].data_ptr(), self.opts,
                                    weight)

    def step(self):
        loss = self.r.read_loss()
        if self.world > 1:
            g = torch.from_numpy(self.r.grads())
            dist.all_reduce(g)
            self.r.set_grads(g.numpy())
            lt = torch.tensor([loss], dtype=torch.float64)
            dist.all_reduce(lt)
            loss = float(lt.item())
        self.r.adam_step(self.adam)
        return loss


def problem():
    ms, co = isg.synth_scene(N, W, H, seed=2403)
    tms, tco = isg.synth_scene(N, W, H, seed=14244)
    cams = [isg.Camera.synthetic(W, H, k, VIEWS) for k in range(VIEWS)]
    targets = [O.render32(tms, tco, c) for c in cams]
    return ms, co, cams, targets


def run(world, rank):
    ms, co, cams, targets = problem()
    dev = [torch.from_numpy(t).cuda() for t in targets]
    opts = isg.RenderOptions(t_min=1e-5)
    adam = isg.AdamConfig(lr_mu=2e-3, lr_sigma=5e-3, lr_color=1e-2, lr_opacity=1e-2, eps=1e-15)
    with isg.Renderer(0) as r:
        r.set_deterministic(True)  # per-rank gradients reproducible run to run
        r.set_scene(ms, co)
        be = GlooRendererBackend(r, cams, dev, opts, adam, world)
        drv = ViewBatchDriver(be, VIEWS, world, rank)
        losses = [drv.train_step() for _ in range(STEPS)]
        ms2, co2 = r.get_scene()
    return ms2, co2, be.seen, losses


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ms, co, seen, losses = run(world, rank)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), ms=ms, co=co, seen=np.array(seen),
             losses=np.array(losses))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_ranks_on_the_library_match_one_rank(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, free_port(), str(tmp_path)), nprocs=world, join=True)
    r = [np.load(tmp_path / f"rank{k}.npz") for k in range(world)]
    seen = np.concatenate([x["seen"] for x in r])
    assert sorted(seen.tolist()) == sorted(list(range(VIEWS)) * STEPS)
    assert np.array_equal(r[0]["ms"], r[1]["ms"]) and np.array_equal(r[0]["co"], r[1]["co"])
    assert np.array_equal(r[0]["losses"], r[1]["losses"])
    ms1, co1, _, losses1 = run(1, 0)
    assert np.allclose(r[0]["losses"], losses1, rtol=1e-5)
    assert np.abs(r[0]["ms"] - ms1).max() < 1e-4
    assert np.abs(r[0]["co"] - co1).max() < 1e-4
    assert losses1[-1] < losses1[0]

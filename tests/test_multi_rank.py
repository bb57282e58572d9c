"""Multi-process view-batch training on CPU (gloo, world_size 2): the host logic of the
multi-GPU path (paper_2403_14244_b200/view_batch.py) driven with the CPU oracle as the per-view
gradient, the same all-reduce-then-Adam step, and checks that
  * every view is processed by exactly one rank,
  * replicas stay bitwise identical after every step,
  * 2 ranks reproduce the 1-rank full-batch trajectory (up to float summation order),
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
from paper_2403_14244_b200.view_batch import ViewBatchDriver, shard_views

W, H, N, VIEWS, STEPS = 64, 48, 600, 4, 3
LR = [2e-3, 5e-3, 1e-2, 1e-2]


class OracleBackend:
    """CPU stand-in for RendererBackend: same semantics, gloo all-reduce instead of NCCL."""

    def __init__(self, ms, co, cams, targets, world):
        self.ms, self.co = ms.copy(), co.copy()
        self.raw = O.raw_init32(self.ms, self.co)
        self.m = np.zeros((ms.shape[0], 8), np.float32)
        self.v = np.zeros_like(self.m)
        self.g = np.zeros_like(self.m)
        self.cams, self.targets, self.world = cams, targets, world
        self.loss, self.t, self.seen = 0.0, 0, []

    def loss_backward(self, view, weight):
        self.seen.append(view)
        loss, _ = O.loss_backward32(self.ms, self.co, self.cams[view], self.targets[view],
                                    weight=weight, grads=self.g, threads=1)
        self.loss += loss

    def step(self):
        if self.world > 1:
            g = torch.from_numpy(self.g)
            dist.all_reduce(g)
            lt = torch.tensor([self.loss], dtype=torch.float64)
            dist.all_reduce(lt)
            self.loss = float(lt.item())
        self.t += 1
        O.adam32(self.ms, self.co, self.m, self.v, self.g, self.t, LR, 0.9, 0.999, 1e-15,
                 raw=self.raw)
        self.g[:] = 0
        loss, self.loss = self.loss, 0.0
        return loss


def problem():
    ms, co = isg.synth_scene(N, W, H, seed=2403)
    tms, tco = isg.synth_scene(N, W, H, seed=14244)
    cams = [isg.Camera.synthetic(W, H, k, VIEWS) for k in range(VIEWS)]
    targets = [O.render32(tms, tco, c) for c in cams]
    return ms, co, cams, targets


def run(world, rank):
    ms, co, cams, targets = problem()
    be = OracleBackend(ms, co, cams, targets, world)
    drv = ViewBatchDriver(be, VIEWS, world, rank)
    losses = [drv.train_step() for _ in range(STEPS)]
    return be, losses


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    be, losses = run(world, rank)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), ms=be.ms, co=be.co, seen=np.array(be.seen),
             losses=np.array(losses))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_views_partition():
    for world in (1, 2, 3, 4, 8):
        owned = [v for r in range(world) for v in shard_views(8, world, r)]
        assert sorted(owned) == list(range(8))
    with pytest.raises(ValueError):
        shard_views(8, 2, 2)


def test_two_rank_gloo_matches_single_rank(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, free_port(), str(tmp_path)), nprocs=world, join=True)
    r = [np.load(tmp_path / f"rank{k}.npz") for k in range(world)]
    # every view exactly once per step, split across ranks
    seen = np.concatenate([x["seen"] for x in r])
    assert sorted(seen.tolist()) == sorted(list(range(VIEWS)) * STEPS)
    # replicas bitwise identical
    assert np.array_equal(r[0]["ms"], r[1]["ms"]) and np.array_equal(r[0]["co"], r[1]["co"])
    assert np.array_equal(r[0]["losses"], r[1]["losses"])
    # same trajectory as one rank doing the whole batch
    be1, losses1 = run(1, 0)
    assert np.allclose(r[0]["losses"], losses1, rtol=1e-6)
    assert np.abs(r[0]["ms"] - be1.ms).max() < 1e-5
    assert np.abs(r[0]["co"] - be1.co).max() < 1e-5
    assert losses1[-1] < losses1[0]

"""View-batch data parallelism: one process per GPU, Gaussians replicated, views sharded.

A training step over a batch of V views:

  rank r owns views r, r + N, r + 2N, ...         (round-robin, `shard_views`)
  for each owned view:  loss_backward(weight = 1/V)  -> gradients accumulate on the device
  adam_step():  NCCL all-reduce (sum) of the n x 8 gradient buffer and the loss inside the
                C-ABI (isg_nccl_*), then the identical Adam update on every replica

Because NCCL's all-reduce returns bitwise-identical sums on every rank and Adam is
deterministic, replicas stay bitwise identical without ever broadcasting parameters.  The
weights make the all-reduced gradient exactly the gradient of the batch-mean loss, so N ranks
reproduce the single-GPU full-batch step (up to float summation order).

The driver is backend-agnostic (`ViewBackend`): the product backend is `RendererBackend`
(libisg.so on the GPU, NCCL rendezvous through torch.distributed); the CPU tests drive the
same code with a gloo process group and the CPU oracle as the per-view gradient.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Protocol, Sequence


def shard_views(n_views: int, world: int, rank: int) -> List[int]:
    """Round-robin view assignment; every view is owned by exactly one rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_views: bad world/rank")
    if n_views < 0:
        raise ValueError("shard_views: negative view count")
    return list(range(rank, n_views, world))


class ViewBackend(Protocol):
    def loss_backward(self, view: int, weight: float) -> None: ...
    def step(self) -> float: ...  # reduce over ranks + optimizer update; returns batch loss


@dataclass
class ViewBatchDriver:
    backend: ViewBackend
    n_views: int
    world: int = 1
    rank: int = 0

    def __post_init__(self):
        self.views = shard_views(self.n_views, self.world, self.rank)
        self.weight = 1.0 / self.n_views

    def train_step(self) -> float:
        for v in self.views:
            self.backend.loss_backward(v, self.weight)
        return self.backend.step()


def nccl_rendezvous(renderer, world: int, rank: int) -> None:
    """Create the library's NCCL communicator: rank 0 draws the unique id, torch.distributed
    (any backend) broadcasts it, every rank attaches it to its context."""
    import torch.distributed as dist

    uid = renderer.nccl_unique_id() if rank == 0 else b"\0" * 128
    obj = [uid]
    dist.broadcast_object_list(obj, src=0)
    renderer.nccl_init(world, rank, obj[0])


class RendererBackend:
    """Product backend: device-resident targets, gradients and the all-reduce inside libisg."""

    def __init__(self, renderer, cameras: Sequence, target_ptrs: Sequence[int], options, adam):
        self.r = renderer
        self.cameras = cameras
        self.targets = target_ptrs
        self.options = options
        self.adam = adam

    def loss_backward(self, view: int, weight: float) -> None:
        self.r.loss_backward_device(self.cameras[view], self.targets[view], self.options, weight)

    def step(self) -> float:
        self.r.adam_step(self.adam)  # all-reduces gradients and the weighted loss first
        return self.r.last_step_loss()

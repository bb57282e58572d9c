"""3D training driver with the semantics of the reference's fit loop.

Follows fit_impl (/root/reference/proj/src/optimize.cpp:298-358) for isotropic 3D splats:

  initial loss over all views; non-finite -> DivergenceError(0, offending particle)
  per epoch: gradients of every view (weight 1/V, so the loss is the view-batch mean), one
    optimizer step (Adam here; the reference's update_step slot, optimize.cpp:78-108);
    backoff=True: the stepped loss is evaluated and the step is rejected (state restored from a
    snapshot, rate_scale halved) when it would increase the loss (:327-340) — the recorded loss
    then never increases;
    non-finite loss -> DivergenceError(epoch, offending particle) (:319, :330-332)
  adapt=True: adaptive control (prune / merge / split, k_adapt.cu) every adapt_every epochs,
    then the loss is re-evaluated (:341-351); the particle cap is max(max_particles, n0), or
    2 n0 when max_particles is 0 (:309-312)
  history: loss_history, particle_count_history, epoch, rate_scale, skipped_updates

Outputs like run_fit_typed (tools/isosplat_main.cpp:116-137): particles.ispl|.json (metadata
epoch, final_loss), loss.csv (write_loss_csv format), state.json sidecar.

The driver is backend-agnostic: `RendererBackend` runs it on the GPU (libisg); the CPU tests
drive the same loop with the CPU oracle.
"""
from __future__ import annotations

import json
import math
from dataclasses import asdict, dataclass, field
from pathlib import Path
from typing import List, Optional, Protocol, Sequence

import numpy as np

from . import scene_io
from .isg import LOSS_L1_DSSIM, LOSS_L2, AdamConfig, AdaptParams, DomainError, RenderOptions


class DivergenceError(RuntimeError):
    """optimize.hpp:30-36 / optimize.cpp:13-17."""

    def __init__(self, epoch: int, particle_index: int):
        super().__init__(f"fit diverged at epoch {epoch} (particle {particle_index})")
        self.epoch = epoch
        self.particle_index = particle_index


@dataclass
class FitConfig3D:
    epochs: int = 100
    adam: AdamConfig = field(default_factory=AdamConfig)
    t_min: float = 1e-5
    background: tuple = (0.0, 0.0, 0.0)
    backoff: bool = False  # reject-and-halve steps that increase the loss
    loss: str = "l2"       # "l2" (mse) or "l1_dssim" ((1-lam) L1 + lam (1 - SSIM), loss.cpp:184)
    lam: float = 0.2       # FitConfig::lambda (the paper's 0.2)
    adapt: bool = False    # adaptive control every adapt_every epochs (optimize.cpp:341-351)
    adapt_every: int = 100
    adapt_params: AdaptParams = field(default_factory=AdaptParams)
    rng_seed: int = 0

    def validate(self):  # particles.hpp:73-83 style
        if self.epochs < 0:
            raise ValueError("epochs: must be >= 0")
        if self.loss not in ("l2", "l1_dssim"):
            raise ValueError("loss: must be 'l2' or 'l1_dssim'")
        if not 0.0 <= self.lam <= 1.0:
            raise ValueError("lambda: must be in [0,1]")
        if self.adapt_every < 1:
            raise ValueError("adapt_every: must be >= 1")
        a = self.adapt_params  # AdaptiveControlParams::validate (optimize.hpp:21-27)
        if not a.prune_threshold >= 0:
            raise ValueError("prune_threshold: must be >= 0")
        if not a.merge_distance_factor > 0:
            raise ValueError("merge_distance_factor: must be > 0")
        if not a.merge_color_tol >= 0:
            raise ValueError("merge_color_tol: must be >= 0")
        if not a.split_sigma_max > 0:
            raise ValueError("split_sigma_max: must be > 0")
        if a.max_particles < 0:
            raise ValueError("max_particles: must be >= 0")
        for name in ("lr_mu", "lr_sigma", "lr_color", "lr_opacity"):
            if not getattr(self.adam, name) > 0:
                raise ValueError(f"{name}: must be > 0")
        if not 0.0 <= self.t_min < 1.0:
            raise ValueError("t_min: must be in [0,1)")


@dataclass
class FitState3D:
    epoch: int = 0
    loss_history: List[float] = field(default_factory=list)
    particle_count_history: List[int] = field(default_factory=list)
    rate_scale: float = 1.0
    skipped_updates: int = 0
    initial_loss: float = 0.0
    final_loss: float = 0.0


class FitBackend(Protocol):
    n_views: int

    def count(self) -> int: ...
    def params(self) -> np.ndarray: ...            # (n, 8) mu.xyz sigma rgb opacity
    def eval_loss(self, view: int, weight: float) -> float: ...
    def loss_backward(self, view: int, weight: float) -> None: ...
    def step(self, rate_scale: float) -> float: ...  # returns the batch loss of the step
    def snapshot(self) -> None: ...
    def restore(self) -> None: ...
    def skipped_updates(self) -> int: ...
    def adaptive_control(self, params: AdaptParams, seed: int, round_: int) -> dict: ...


def offending_particle(params: np.ndarray) -> int:
    """First splat with a non-finite or invalid parameter (optimize.cpp offending_particle)."""
    p = np.asarray(params)
    bad = ~np.all(np.isfinite(p), axis=1) | ~(p[:, 3] > 0) | ~((p[:, 7] >= 0) & (p[:, 7] <= 1))
    idx = np.flatnonzero(bad)
    return int(idx[0]) if idx.size else -1


def _batch_loss(be: FitBackend, w: float, epoch: int) -> float:
    try:
        loss = sum(be.eval_loss(v, w) for v in range(be.n_views))
    except DomainError:
        raise DivergenceError(epoch, offending_particle(be.params())) from None
    if not math.isfinite(loss):
        raise DivergenceError(epoch, offending_particle(be.params()))
    return loss


def fit(be: FitBackend, config: FitConfig3D) -> FitState3D:
    config.validate()
    if be.count() == 0:
        raise ValueError("init_particles: must be nonempty")
    st = FitState3D()
    w = 1.0 / be.n_views
    n0 = be.count()
    a = config.adapt_params  # particle cap, optimize.cpp:309-312
    cap = max(a.max_particles, n0) if a.max_particles > 0 else 2 * n0
    adapt_round = 0
    current = _batch_loss(be, w, 0)
    st.initial_loss = current
    for e in range(config.epochs):
        try:
            for v in range(be.n_views):
                be.loss_backward(v, w)
            if config.backoff:
                be.snapshot()
                be.step(st.rate_scale)
                stepped = _batch_loss(be, w, e)
                if stepped <= current:
                    current = stepped
                else:
                    be.restore()  # reject the step, try smaller (optimize.cpp:337-339)
                    st.rate_scale *= 0.5
            else:
                loss = be.step(st.rate_scale)
                if not math.isfinite(loss):
                    raise DivergenceError(e, offending_particle(be.params()))
                current = loss
        except DomainError:
            raise DivergenceError(e, offending_particle(be.params())) from None
        if config.adapt and (e + 1) % config.adapt_every == 0:
            be.adaptive_control(AdaptParams(a.prune_threshold, a.merge_distance_factor,
                                            a.merge_color_tol, a.split_sigma_max, cap),
                                config.rng_seed, adapt_round)
            adapt_round += 1
            current = _batch_loss(be, w, e)
        st.loss_history.append(current)
        st.particle_count_history.append(be.count())
        st.epoch = e + 1
    st.final_loss = current
    st.skipped_updates = be.skipped_updates()
    return st


def save_fit_outputs(out_dir, st: FitState3D, config: FitConfig3D, params: np.ndarray,
                     as_json: bool = False) -> None:
    """particles + loss.csv + state.json, as run_fit_typed (isosplat_main.cpp:116-137)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    ps = scene_io.ParticleSet(np.asarray(params, np.float64),
                              metadata={"epoch": st.epoch, "final_loss": st.final_loss})
    scene_io.save_particles(out / ("particles.json" if as_json else "particles.ispl"), ps, as_json)
    first = st.particle_count_history[0] if st.particle_count_history else ps.count()
    scene_io.write_loss_csv(out / "loss.csv", st.initial_loss, first, st.loss_history,
                            st.particle_count_history)
    cfg = asdict(config)
    sidecar = {"epoch": st.epoch, "initial_loss": st.initial_loss, "final_loss": st.final_loss,
               "rate_scale": st.rate_scale, "skipped_updates": st.skipped_updates,
               "particles": ps.count(), "config": cfg, "loss_history": st.loss_history,
               "particle_count_history": st.particle_count_history}
    (out / "state.json").write_text(json.dumps(sidecar, indent=2) + "\n")


class RendererBackend:
    """GPU backend: scene, Adam state and (device) targets resident in HBM."""

    def __init__(self, renderer, cameras: Sequence, target_ptrs: Sequence[int],
                 config: FitConfig3D):
        self.r = renderer
        self.cameras = list(cameras)
        self.targets = list(target_ptrs)
        self.n_views = len(self.cameras)
        self.opts = RenderOptions(background=config.background, t_min=config.t_min)
        self.adam = config.adam
        renderer.set_loss(LOSS_L1_DSSIM if config.loss == "l1_dssim" else LOSS_L2, config.lam)

    def count(self) -> int:
        return self.r.n

    def params(self) -> np.ndarray:
        ms, co = self.r.get_scene()
        return np.concatenate([ms, co], 1).astype(np.float64)

    def eval_loss(self, view: int, weight: float) -> float:
        return self.r.eval_loss_device(self.cameras[view], self.targets[view], self.opts, weight)

    def loss_backward(self, view: int, weight: float) -> None:
        self.r.loss_backward_device(self.cameras[view], self.targets[view], self.opts, weight)

    def step(self, rate_scale: float) -> float:
        a = self.adam
        self.r.adam_step(AdamConfig(a.lr_mu * rate_scale, a.lr_sigma * rate_scale,
                                    a.lr_color * rate_scale, a.lr_opacity * rate_scale,
                                    a.beta1, a.beta2, a.eps))
        return self.r.last_step_loss()

    def snapshot(self) -> None:
        self.r.snapshot()

    def restore(self) -> None:
        self.r.restore()

    def skipped_updates(self) -> int:
        return int(self.r.stats()["skipped_updates"])

    def adaptive_control(self, params: AdaptParams, seed: int, round_: int) -> dict:
        return self.r.adaptive_control(params, seed, round_)

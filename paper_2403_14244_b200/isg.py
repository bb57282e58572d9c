"""ctypes binding of the C-ABI (include/isg.h) — the Python face of the B200 hot path.

Mirrors the reference's render/train API (/root/reference/proj/include/isosplat/splat3d.hpp:
IsoSplat3D :13-22, Camera :37-53, RenderOptions :87-90, render :96-97) over libisg.so.
There is no CPU fallback: if libisg.so is missing or no CUDA device is present the calls
raise.  Errors keep the reference's exception types: invalid splats / cameras raise
``DomainError`` (std::domain_error), bad arguments ``ValueError`` (std::invalid_argument).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("ISG_LIB_PATH", _PKG / "libisg.so"))  # override: A/B builds

ISG_OK, ISG_E_DOMAIN, ISG_E_ARG, ISG_E_CUDA, ISG_E_OOM, ISG_E_OVERFLOW, ISG_E_NCCL, ISG_E_STATE = range(8)
LOSS_L2, LOSS_L1_DSSIM = 0, 1  # ISG_LOSS_* (include/isg.h)


class IsgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class DomainError(IsgError, ValueError):
    """std::domain_error of the reference (invalid splat / camera)."""


class CameraT(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3), ("focal", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32), ("height", C.c_int32)]


class AdaptParamsT(C.Structure):
    """isg_adapt_params: AdaptiveControlParams (optimize.hpp:14-28) for 3D splats."""
    _fields_ = [("prune_threshold", C.c_double), ("merge_distance_factor", C.c_double),
                ("merge_color_tol", C.c_double), ("split_sigma_max", C.c_double),
                ("max_particles", C.c_int64)]


class AdaptResultT(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("n_before", "n_pruned", "n_merged", "n_split",
                                         "n_after")]


class StatsT(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("n_gaussians", "n_visible", "n_keys", "key_capacity",
                                         "n_tiles", "adam_steps", "skipped_updates",
                                         "regrow_events", "kernel_launches", "overflowed_frames")]


_lib = None


def lib() -> C.CDLL:
    """Load libisg.so (built by __graft_entry__.build()).  Raises if absent — no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
    L = C.CDLL(str(LIB_PATH))
    P, I64, I32, F = C.c_void_p, C.c_int64, C.c_int32, C.c_float
    fp = C.POINTER(C.c_float)
    sigs = {
        "isg_abi_version": ([], C.c_int),
        "isg_status_string": ([C.c_int], C.c_char_p),
        "isg_last_error": ([P], C.c_char_p),
        "isg_create": ([C.c_int, I64, I32, I32, C.POINTER(P)], C.c_int),
        "isg_destroy": ([P], None),
        "isg_set_stream": ([P, P], C.c_int),
        "isg_synchronize": ([P], C.c_int),
        "isg_get_stats": ([P, C.POINTER(StatsT)], C.c_int),
        "isg_set_scene": ([P, I64, P, P], C.c_int),
        "isg_set_scene_device": ([P, I64, P, P], C.c_int),
        "isg_get_scene": ([P, P, P], C.c_int),
        "isg_render": ([P, C.POINTER(CameraT), fp, F, P], C.c_int),
        "isg_render_device": ([P, C.POINTER(CameraT), fp, F, P], C.c_int),
        "isg_loss_backward": ([P, C.POINTER(CameraT), fp, F, P, F, C.POINTER(C.c_double)], C.c_int),
        "isg_loss_backward_device": ([P, C.POINTER(CameraT), fp, F, P, F], C.c_int),
        "isg_upload_target_async": ([P, C.c_int32, P, C.c_int32, C.c_int32], C.c_int),
        "isg_render_host_async": ([P, C.POINTER(CameraT), fp, F, C.c_int32, P], C.c_int),
        "isg_image_wait": ([P, C.c_int32], C.c_int),
        "isg_loss_backward_slot": ([P, C.POINTER(CameraT), fp, F, C.c_int32, F], C.c_int),
        "isg_read_loss": ([P, C.POINTER(C.c_double)], C.c_int),
        "isg_zero_grads": ([P], C.c_int),
        "isg_get_grads": ([P, P], C.c_int),
        "isg_set_grads": ([P, P], C.c_int),
        "isg_grads_device": ([P, C.POINTER(P)], C.c_int),
        "isg_adam_step": ([P, fp, F, F, F], C.c_int),
        "isg_last_step_loss": ([P, C.POINTER(C.c_double)], C.c_int),
        "isg_step_loss_async": ([P, C.c_void_p], C.c_int),
        "isg_eval_loss": ([P, C.POINTER(CameraT), fp, F, P, F, C.POINTER(C.c_double)], C.c_int),
        "isg_snapshot": ([P], C.c_int),
        "isg_restore": ([P], C.c_int),
        "isg_set_loss": ([P, C.c_int, F], C.c_int),
        "isg_graph_begin": ([P], C.c_int),
        "isg_graph_end": ([P, C.POINTER(P)], C.c_int),
        "isg_graph_launch": ([P, P], C.c_int),
        "isg_graph_destroy": ([P], None),
        "isg_adaptive_control": ([P, C.POINTER(AdaptParamsT), C.c_uint64, C.c_uint64,
                                  C.POINTER(AdaptResultT)], C.c_int),
        "isg_image_loss_device": ([P, I32, I32, P, P, F, C.POINTER(C.c_double), P], C.c_int),
        "isg_nccl_get_unique_id": ([P], C.c_int),
        "isg_nccl_init": ([P, C.c_int, C.c_int, P], C.c_int),
        "isg_nccl_detach": ([P], C.c_int),
        "isg_nccl_attach": ([P, P], C.c_int),
        "isg_nccl_info": ([P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
        "isg_set_exchange_chunks": ([P, C.c_int], C.c_int),
        "isg_debug_bins": ([P, P, P, C.POINTER(I64), P], C.c_int),
        "isg_debug_pixel_state": ([P, P, P], C.c_int),
        "isg_count_pairs": ([P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
        "isg_set_binning": ([P, C.c_int], C.c_int),
        "isg_set_deterministic": ([P, C.c_int], C.c_int),
        "isg_profile_enable": ([P, C.c_int], C.c_int),
        "isg_profile_num_stages": ([], C.c_int),
        "isg_profile_stage_name": ([C.c_int], C.c_char_p),
        "isg_profile_read": ([P, P, P], C.c_int),
        "isg_synth_scene": ([C.c_uint64, I64, I32, I32, P, P], C.c_int),
        "isg_synth_camera": ([I32, I32, I32, I32, C.POINTER(CameraT)], C.c_int),
    }
    for name, (args, res) in sigs.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


# exported symbol list (tests check that the library exports every declaration of isg.h)
C_ABI_SYMBOLS = (
    "isg_abi_version", "isg_status_string", "isg_last_error", "isg_create", "isg_destroy",
    "isg_set_stream", "isg_synchronize", "isg_get_stats", "isg_set_scene", "isg_set_scene_device",
    "isg_get_scene", "isg_render", "isg_render_device", "isg_loss_backward",
    "isg_render_host_async", "isg_image_wait",
    "isg_loss_backward_device", "isg_upload_target_async", "isg_loss_backward_slot", "isg_read_loss", "isg_zero_grads", "isg_get_grads", "isg_set_grads",
    "isg_grads_device", "isg_adam_step", "isg_last_step_loss", "isg_step_loss_async", "isg_eval_loss", "isg_snapshot",
    "isg_restore", "isg_set_loss", "isg_image_loss_device", "isg_adaptive_control",
    "isg_graph_begin", "isg_graph_end", "isg_graph_launch", "isg_graph_destroy", "isg_nccl_get_unique_id",
    "isg_nccl_init", "isg_nccl_attach", "isg_nccl_info", "isg_set_exchange_chunks",
    "isg_nccl_detach", "isg_debug_bins", "isg_debug_pixel_state", "isg_count_pairs", "isg_set_binning",
    "isg_set_deterministic",
    "isg_profile_enable",
    "isg_profile_num_stages", "isg_profile_stage_name", "isg_profile_read", "isg_synth_scene",
    "isg_synth_camera",
)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------------------------
# Reference-shaped value types (splat3d.hpp:13-53, 87-90)
# ---------------------------------------------------------------------------------------------
@dataclass
class Camera:
    """Rigid world->camera transform + pinhole intrinsics (splat3d.hpp:37-53)."""
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))
    focal: float = 1.0
    principal_point: tuple = (0.0, 0.0)
    width: int = 1
    height: int = 1

    def validate(self) -> None:
        """Camera::validate (splat3d.cpp:27-37), FP64, 1e-9 orthonormality."""
        R = np.asarray(self.rotation, dtype=np.float64)
        t = np.asarray(self.translation, dtype=np.float64)
        if not (np.all(np.isfinite(R)) and np.all(np.isfinite(t))):
            raise DomainError(ISG_E_DOMAIN, "Camera: non-finite transform")
        if np.max(np.abs(R @ R.T - np.eye(3))) > 1e-9:
            raise DomainError(ISG_E_DOMAIN, "Camera.rotation: not orthonormal within 1e-9")
        if not self.focal > 0.0:
            raise DomainError(ISG_E_DOMAIN, "Camera.focal: must be > 0")
        if self.width <= 0 or self.height <= 0:
            raise DomainError(ISG_E_DOMAIN, "Camera: bad image size")

    def to_c(self) -> CameraT:
        c = CameraT()
        R = np.asarray(self.rotation, dtype=np.float64).reshape(9)
        for i in range(9):
            c.R[i] = float(R[i])
        for i in range(3):
            c.t[i] = float(self.translation[i])
        c.focal = float(self.focal)
        c.cx, c.cy = float(self.principal_point[0]), float(self.principal_point[1])
        c.width, c.height = int(self.width), int(self.height)
        return c

    @staticmethod
    def from_c(c: CameraT) -> "Camera":
        return Camera(np.array(list(c.R), dtype=np.float64).reshape(3, 3),
                      np.array(list(c.t), dtype=np.float64), float(c.focal),
                      (float(c.cx), float(c.cy)), int(c.width), int(c.height))

    @staticmethod
    def synthetic(width: int, height: int, view: int = 0, n_views: int = 1) -> "Camera":
        c = CameraT()
        _check(None, lib().isg_synth_camera(width, height, view, n_views, C.byref(c)))
        return Camera.from_c(c)


TARGET_SLOTS = 32  # ISG_TARGET_SLOTS (include/isg.h)
IMAGE_SLOTS = 8  # ISG_IMAGE_SLOTS


@dataclass
class RenderOptions:
    """RenderOptions (splat3d.hpp:87-90) + t_min, the early-termination threshold.  The default
    0 is the reference's exact semantics (every covering splat composited, splat3d.cpp:134-141);
    training configs opt in to early termination (e.g. 1e-5).  `threads` is accepted for API
    parity and ignored."""
    background: tuple = (0.0, 0.0, 0.0)
    threads: int = 1
    t_min: float = 0.0


@dataclass
class AdaptParams:
    """AdaptiveControlParams (optimize.hpp:14-28); split_sigma_max in world units (the
    reference's 15 px is a 2D pixel scale).  max_particles: effective cap (0: twice the
    current count)."""
    prune_threshold: float = 1e-3
    merge_distance_factor: float = 0.5
    merge_color_tol: float = 0.05
    split_sigma_max: float = float("inf")
    max_particles: int = 0


@dataclass
class AdamConfig:
    lr_mu: float = 1e-3
    lr_sigma: float = 5e-3
    lr_color: float = 1e-2
    lr_opacity: float = 1e-2
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-15

    def lrs(self):
        return (C.c_float * 4)(self.lr_mu, self.lr_sigma, self.lr_color, self.lr_opacity)


def _process_nccl() -> None:
    """libisg resolves NCCL at run time and prefers one already loaded in the process.  Load
    torch's bundled NCCL first (importing torch does) so that the process holds one NCCL —
    otherwise an older system libnccl.so.2 loaded here would later shadow torch's (same
    SONAME) and break `import torch`."""
    try:
        import torch  # noqa: F401
    except Exception:
        pass


def _check(ctx, status: int) -> None:
    if status == ISG_OK:
        return
    L = lib()
    msg = (L.isg_last_error(ctx) or b"").decode() if ctx else ""
    msg = msg or L.isg_status_string(status).decode()
    if status == ISG_E_DOMAIN:
        raise DomainError(status, msg)
    if status == ISG_E_ARG:
        raise ValueError(msg)
    raise IsgError(status, f"{L.isg_status_string(status).decode()}: {msg}")


class Graph:
    """A captured sequence of asynchronous calls (isg_graph), replayed with launch()."""

    def __init__(self, renderer, handle):
        self._r, self._h = renderer, handle

    def launch(self):
        _check(self._r._h, lib().isg_graph_launch(self._r._h, self._h))

    def close(self):
        if self._h:
            lib().isg_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def splats_to_soa(splats: np.ndarray):
    """(n, 8) [mu.xyz, sigma, rgb, opacity] (the ISPL record, particle_io.hpp:36-46) ->
    two contiguous float32 (n, 4) arrays."""
    s = np.asarray(splats, dtype=np.float64).reshape(-1, 8)
    return (np.ascontiguousarray(s[:, 0:4], dtype=np.float32),
            np.ascontiguousarray(s[:, 4:8], dtype=np.float32))


def synth_scene(n: int, width: int, height: int, seed: int = 2403):
    """isg-synth v1 scene as (mu_sigma (n,4) f32, rgb_opacity (n,4) f32)."""
    ms = np.empty((n, 4), np.float32)
    co = np.empty((n, 4), np.float32)
    _check(None, lib().isg_synth_scene(seed, n, width, height, _ptr(ms), _ptr(co)))
    return ms, co


class Renderer:
    """One device context (isg_ctx): scene, Adam state, buffers, one CUDA stream."""

    def __init__(self, device: int = 0, max_gaussians: int = 0, max_width: int = 0,
                 max_height: int = 0):
        L = lib()
        h = C.c_void_p()
        st = L.isg_create(device, max_gaussians, max_width, max_height, C.byref(h))
        if st != ISG_OK:
            raise IsgError(st, f"isg_create failed: {L.isg_status_string(st).decode()}")
        self._h = h
        self.n = 0

    def close(self):
        if getattr(self, "_h", None):
            lib().isg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- plumbing ---------------------------------------------------------------------------
    @property
    def handle(self):
        return self._h

    def set_stream(self, stream_ptr: int | None):
        _check(self._h, lib().isg_set_stream(self._h, C.c_void_p(stream_ptr or 0)))

    def synchronize(self):
        _check(self._h, lib().isg_synchronize(self._h))

    def stats(self) -> dict:
        s = StatsT()
        _check(self._h, lib().isg_get_stats(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in StatsT._fields_}

    # -- scene ------------------------------------------------------------------------------
    def set_scene(self, mu_sigma: np.ndarray, rgb_opacity: np.ndarray):
        ms = np.ascontiguousarray(mu_sigma, dtype=np.float32).reshape(-1, 4)
        co = np.ascontiguousarray(rgb_opacity, dtype=np.float32).reshape(-1, 4)
        if ms.shape != co.shape:
            raise ValueError("set_scene: mu_sigma and rgb_opacity differ in length")
        _check(self._h, lib().isg_set_scene(self._h, ms.shape[0], _ptr(ms), _ptr(co)))
        self.n = ms.shape[0]

    def set_scene_device(self, n: int, mu_sigma_ptr: int, rgb_opacity_ptr: int):
        _check(self._h, lib().isg_set_scene_device(self._h, n, C.c_void_p(mu_sigma_ptr),
                                                   C.c_void_p(rgb_opacity_ptr)))
        self.n = n

    def get_scene(self):
        ms = np.empty((self.n, 4), np.float32)
        co = np.empty((self.n, 4), np.float32)
        _check(self._h, lib().isg_get_scene(self._h, _ptr(ms), _ptr(co)))
        return ms, co

    # -- forward ----------------------------------------------------------------------------
    @staticmethod
    def _cam(camera):
        if isinstance(camera, CameraT):
            return camera
        return camera.to_c()

    @staticmethod
    def _bg(options: RenderOptions):
        return (C.c_float * 3)(*[float(b) for b in options.background])

    def render(self, camera, options: RenderOptions = RenderOptions(),
               out: Optional[np.ndarray] = None) -> np.ndarray:
        """render(iso) (splat3d.cpp:173-194): (H, W, 3) float32 image (into `out` if given,
        e.g. a pinned buffer)."""
        c = self._cam(camera)
        if out is None:
            out = np.empty((c.height, c.width, 3), np.float32)
        elif out.dtype != np.float32 or out.size != c.height * c.width * 3 or not out.flags.c_contiguous:
            raise ValueError("render: out must be a C-contiguous float32 (H, W, 3) array")
        _check(self._h, lib().isg_render(self._h, C.byref(c), self._bg(options),
                                         float(options.t_min), _ptr(out)))
        return out

    def render_device(self, camera, options: RenderOptions, out_ptr: int):
        c = self._cam(camera)
        _check(self._h, lib().isg_render_device(self._h, C.byref(c), self._bg(options),
                                                float(options.t_min), C.c_void_p(out_ptr)))

    # -- training ---------------------------------------------------------------------------
    def loss_backward(self, camera, target: np.ndarray, options: RenderOptions = RenderOptions(),
                      weight: float = 1.0) -> float:
        c = self._cam(camera)
        t = np.ascontiguousarray(target, dtype=np.float32)
        if t.size != c.width * c.height * 3:
            raise ValueError("loss_backward: target shape does not match the camera")
        loss = C.c_double()
        _check(self._h, lib().isg_loss_backward(self._h, C.byref(c), self._bg(options),
                                                float(options.t_min), _ptr(t), float(weight),
                                                C.byref(loss)))
        return loss.value

    def loss_backward_device(self, camera, target_ptr: int,
                             options: RenderOptions = RenderOptions(), weight: float = 1.0):
        c = self._cam(camera)
        _check(self._h, lib().isg_loss_backward_device(self._h, C.byref(c), self._bg(options),
                                                       float(options.t_min),
                                                       C.c_void_p(target_ptr), float(weight)))

    def render_host_async(self, camera, slot: int, out: np.ndarray,
                          options: RenderOptions = RenderOptions()):
        """isg_render_host_async: render into image ring slot `slot` and enqueue the copy into
        `out` (a C-contiguous H x W x 3 float32 array that stays alive; page-locked memory makes
        the copy truly asynchronous).  image_wait(slot) before reading `out`."""
        if not (out.flags.c_contiguous and out.dtype == np.float32):
            raise ValueError("render_host_async: out must be a C-contiguous float32 array")
        c = self._cam(camera)
        _check(self._h, lib().isg_render_host_async(self._h, C.byref(c), self._bg(options),
                                                    float(options.t_min), int(slot), _ptr(out)))

    def image_wait(self, slot: int):
        _check(self._h, lib().isg_image_wait(self._h, int(slot)))

    def upload_target_async(self, slot: int, target: np.ndarray):
        """isg_upload_target_async: enqueue the H2D copy of an H x W x 3 float32 target into ring
        slot `slot` (< TARGET_SLOTS) on the context's copy stream.  The array must stay alive and
        unchanged until the copy has run (page-locked memory makes it truly asynchronous)."""
        t = np.ascontiguousarray(target, dtype=np.float32)
        if t is not target:
            raise ValueError("upload_target_async: target must be a C-contiguous float32 array "
                             "(a temporary copy would be freed before the asynchronous upload)")
        H, W = t.shape[:2]
        _check(self._h, lib().isg_upload_target_async(self._h, int(slot), _ptr(t), W, H))

    def loss_backward_slot(self, camera, slot: int, options: RenderOptions = RenderOptions(),
                           weight: float = 1.0):
        """isg_loss_backward_slot: loss_backward_device on target ring slot `slot`."""
        c = self._cam(camera)
        _check(self._h, lib().isg_loss_backward_slot(self._h, C.byref(c), self._bg(options),
                                                     float(options.t_min), int(slot),
                                                     float(weight)))

    def read_loss(self) -> float:
        v = C.c_double()
        _check(self._h, lib().isg_read_loss(self._h, C.byref(v)))
        return v.value

    def zero_grads(self):
        _check(self._h, lib().isg_zero_grads(self._h))

    def grads(self) -> np.ndarray:
        g = np.empty((self.n, 8), np.float32)
        _check(self._h, lib().isg_get_grads(self._h, _ptr(g)))
        return g

    def set_grads(self, grads: np.ndarray):
        """isg_set_grads: replace the accumulated gradients (n x 8, host)."""
        g = np.ascontiguousarray(grads, dtype=np.float32)
        _check(self._h, lib().isg_set_grads(self._h, _ptr(g)))

    def grads_device_ptr(self) -> int:
        p = C.c_void_p()
        _check(self._h, lib().isg_grads_device(self._h, C.byref(p)))
        return p.value or 0

    def adam_step(self, cfg: AdamConfig = AdamConfig()):
        _check(self._h, lib().isg_adam_step(self._h, cfg.lrs(), cfg.beta1, cfg.beta2, cfg.eps))

    def eval_loss_device(self, camera, target_ptr: int, options: RenderOptions = RenderOptions(),
                         weight: float = 1.0) -> float:
        """weight * mse of one view, no gradients (pending gradients are kept)."""
        c = self._cam(camera)
        v = C.c_double()
        _check(self._h, lib().isg_eval_loss(self._h, C.byref(c), self._bg(options),
                                            float(options.t_min), C.c_void_p(target_ptr),
                                            float(weight), C.byref(v)))
        return v.value

    def snapshot(self):
        _check(self._h, lib().isg_snapshot(self._h))

    def restore(self):
        _check(self._h, lib().isg_restore(self._h))

    def set_loss(self, kind: int = LOSS_L2, lam: float = 0.2):
        """Training/eval loss: LOSS_L2 (mse) or LOSS_L1_DSSIM ((1-lam) L1 + lam (1 - SSIM),
        loss.cpp:184-190)."""
        _check(self._h, lib().isg_set_loss(self._h, int(kind), float(lam)))

    def image_loss_device(self, width: int, height: int, fhat_ptr: int, target_ptr: int,
                          weight: float = 1.0, dldc_ptr: Optional[int] = None) -> float:
        """The configured loss of a device image against a device target (+ dL/dfhat)."""
        v = C.c_double()
        _check(self._h, lib().isg_image_loss_device(
            self._h, int(width), int(height), C.c_void_p(fhat_ptr), C.c_void_p(target_ptr),
            float(weight), C.byref(v), C.c_void_p(dldc_ptr) if dldc_ptr else None))
        return v.value

    def adaptive_control(self, params: "AdaptParams", seed: int = 0, round_: int = 0) -> dict:
        """Prune / merge / split the resident splat set (optimize.cpp:221-284); returns the
        counts.  Adam state restarts."""
        p = AdaptParamsT(params.prune_threshold, params.merge_distance_factor,
                         params.merge_color_tol, params.split_sigma_max,
                         int(params.max_particles))
        res = AdaptResultT()
        _check(self._h, lib().isg_adaptive_control(self._h, C.byref(p), int(seed), int(round_),
                                                   C.byref(res)))
        self.n = int(res.n_after)
        return {k: int(getattr(res, k)) for k, _ in AdaptResultT._fields_}

    # -- CUDA graphs -------------------------------------------------------------------------
    def graph_begin(self):
        """Start capturing the asynchronous calls on the context stream."""
        _check(self._h, lib().isg_graph_begin(self._h))

    def graph_end(self) -> "Graph":
        g = C.c_void_p()
        _check(self._h, lib().isg_graph_end(self._h, C.byref(g)))
        return Graph(self, g)

    def last_step_loss(self) -> float:
        v = C.c_double()
        _check(self._h, lib().isg_last_step_loss(self._h, C.byref(v)))
        return v.value

    def step_loss_async(self, host_ptr: int) -> None:
        """Enqueue the last step's loss D2H into page-locked host memory at host_ptr (no sync;
        capturable into a graph)."""
        _check(self._h, lib().isg_step_loss_async(self._h, C.c_void_p(host_ptr)))

    # -- multi-GPU --------------------------------------------------------------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        _process_nccl()
        buf = (C.c_char * 128)()
        _check(None, lib().isg_nccl_get_unique_id(buf))
        return bytes(buf)

    def nccl_init(self, nranks: int, rank: int, uid: bytes):
        _process_nccl()
        buf = (C.c_char * 128).from_buffer_copy(uid)
        _check(self._h, lib().isg_nccl_init(self._h, nranks, rank, buf))

    def nccl_attach(self, comm_ptr: int):
        """Use a caller-owned ncclComm_t (its address as an int); the caller keeps ownership."""
        _process_nccl()
        _check(self._h, lib().isg_nccl_attach(self._h, C.c_void_p(comm_ptr)))

    def nccl_info(self) -> dict:
        """{'nranks', 'rank'} as the attached communicator reports them, and the NCCL version."""
        n, r, v = C.c_int(), C.c_int(), C.c_int()
        _check(self._h, lib().isg_nccl_info(self._h, C.byref(n), C.byref(r), C.byref(v)))
        return {"nranks": n.value, "rank": r.value, "nccl_version": v.value}

    def set_exchange_chunks(self, chunks: int):
        _check(self._h, lib().isg_set_exchange_chunks(self._h, int(chunks)))

    def nccl_detach(self):
        _check(self._h, lib().isg_nccl_detach(self._h))

    BINNING_TILE_BUCKET, BINNING_RADIX = 0, 1

    def set_deterministic(self, on: bool = True):
        """Slot-mode gradient accumulation (bitwise deterministic) instead of the default
        direct L2 reduction (isg_set_deterministic)."""
        _check(self._h, lib().isg_set_deterministic(self._h, int(bool(on))))

    def set_binning(self, mode: int):
        """0 = tile-bucket, 1 = onesweep radix (default); bit-identical tile lists."""
        _check(self._h, lib().isg_set_binning(self._h, int(mode)))

    # -- stage timing -----------------------------------------------------------------------
    def profile(self, on: bool = True):
        _check(self._h, lib().isg_profile_enable(self._h, int(on)))

    def profile_read(self) -> dict:
        L = lib()
        k = L.isg_profile_num_stages()
        ms = np.zeros(k, np.float64)
        calls = np.zeros(k, np.int64)
        _check(self._h, L.isg_profile_read(self._h, _ptr(ms), _ptr(calls)))
        return {L.isg_profile_stage_name(i).decode(): (float(ms[i]), int(calls[i]))
                for i in range(k) if calls[i]}

    # -- parity hooks -----------------------------------------------------------------------
    def debug_bins(self):
        n = C.c_int64()
        _check(self._h, lib().isg_debug_bins(self._h, None, None, C.byref(n), None))
        keys = np.empty(n.value, np.uint64)
        vals = np.empty(n.value, np.uint32)
        st = self.stats()
        ranges = np.empty((st["n_tiles"], 2), np.uint32)
        _check(self._h, lib().isg_debug_bins(self._h, _ptr(keys), _ptr(vals), C.byref(n),
                                             _ptr(ranges)))
        return keys, vals, ranges

    def count_pairs(self):
        """(evaluated, inside) pixel-entry pairs of the last frame (isg_count_pairs)."""
        a, b = C.c_int64(), C.c_int64()
        _check(self._h, lib().isg_count_pairs(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def debug_pixel_state(self, width: int, height: int):
        tl = np.empty((height, width), np.float32)
        npr = np.empty((height, width), np.uint32)
        _check(self._h, lib().isg_debug_pixel_state(self._h, _ptr(tl), _ptr(npr)))
        return tl, npr


def render(splats: np.ndarray, camera: Camera, options: RenderOptions = RenderOptions(),
           device: int = 0) -> np.ndarray:
    """Drop-in for isosplat::render(std::span<const IsoSplat3D>, const Camera&,
    const RenderOptions&) (splat3d.hpp:96-97): splats as an (n, 8) array of ISPL records.
    Validates in FP64 first (splat3d.cpp:10-37), then renders on the GPU."""
    camera.validate()
    s = np.asarray(splats, dtype=np.float64).reshape(-1, 8)
    validate_splats(s)
    ms, co = splats_to_soa(s)
    with Renderer(device) as r:
        r.set_scene(ms, co)
        return r.render(camera, options)


def validate_splats(s: np.ndarray) -> None:
    """IsoSplat3D::validate (splat3d.cpp:10-17) over (n, 8) FP64 records; raises at the first
    invalid splat, with the reference's message."""
    s = np.asarray(s, dtype=np.float64).reshape(-1, 8)
    mu_ok = np.all(np.isfinite(s[:, 0:3]), axis=1)
    sg_ok = (s[:, 3] > 0) & np.isfinite(s[:, 3])
    c_ok = np.all(np.isfinite(s[:, 4:7]), axis=1)
    o_ok = (s[:, 7] >= 0) & (s[:, 7] <= 1)
    ok = mu_ok & sg_ok & c_ok & o_ok
    if ok.all():
        return
    i = int(np.argmin(ok))
    if not mu_ok[i]:
        raise DomainError(ISG_E_DOMAIN, "IsoSplat3D.mu: non-finite coordinates")
    if not sg_ok[i]:
        raise DomainError(ISG_E_DOMAIN, "IsoSplat3D.sigma: must be positive and finite")
    if not c_ok[i]:
        raise DomainError(ISG_E_DOMAIN, "IsoSplat3D.color: non-finite")
    raise DomainError(ISG_E_DOMAIN, "IsoSplat3D.opacity: must be in [0,1]")

"""ctypes loader for the CPU oracle (oracle/isg_oracle.c, oracle/_ref) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs use
this module, always as the checker or the timed CPU baseline, never as the product path.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]  # repo root
ORACLE_LIB = ROOT / "oracle" / "_build" / "libisg_oracle.so"
REF_LIB = ROOT / "oracle" / "_ref" / "libisosplat_ref.so"


class Cam32(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3), ("focal", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32), ("height", C.c_int32)]


class Cam64(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3), ("focal", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("width", C.c_int32), ("height", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not ORACLE_LIB.exists():
            import sys
            sys.path.insert(0, str(ROOT))
            from paper_2403_14244_b200 import build
            build.build_oracle()
        L = C.CDLL(str(ORACLE_LIB))
        P, I64 = C.c_void_p, C.c_int64
        L.or_version.restype = C.c_int
        L.or64_project_iso.argtypes = [P, C.POINTER(Cam64), P]
        L.or64_project_iso.restype = C.c_int
        L.or64_composite.argtypes = [I64, P, P]
        L.or64_composite.restype = C.c_int
        L.or64_render.argtypes = [I64, P, C.POINTER(Cam64), P, C.c_int, P]
        L.or64_render.restype = C.c_int
        L.or64_brute_force.argtypes = [I64, P, C.POINTER(Cam64), P, P]
        L.or64_brute_force.restype = C.c_int
        L.or64_mse.argtypes = [I64, P, P]
        L.or64_mse.restype = C.c_double
        L.or64_loss_grad.argtypes = [I64, P, C.POINTER(Cam64), P, P, C.c_double, P, P]
        L.or64_loss_grad.restype = C.c_int
        L.or32_bin.argtypes = [I64, P, P, C.POINTER(Cam32), P, P, I64, P, C.POINTER(I64)]
        L.or32_bin.restype = I64
        L.or32_render.argtypes = [I64, P, P, C.POINTER(Cam32), P, C.c_float, C.c_int, P, P, P, P]
        L.or32_render.restype = C.c_int
        L.or32_loss_backward.argtypes = [I64, P, P, C.POINTER(Cam32), P, C.c_float, P, C.c_float,
                                         C.c_int, C.POINTER(C.c_double), P, P]
        L.or32_loss_backward.restype = C.c_int
        L.or32_adam.argtypes = [I64, P, P, P, P, P, P, I64, P, C.c_float, C.c_float, C.c_float,
                                C.POINTER(I64)]
        L.or32_adam.restype = None
        L.or32_raw_init.argtypes = [I64, P, P, P]
        L.or32_raw_init.restype = None
        L.or_synth_scene.argtypes = [C.c_uint64, I64, C.c_int, C.c_int, P, P]
        L.or_synth_scene.restype = None
        L.or_synth_camera.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, P]
        L.or_synth_camera.restype = None
        L.or32_backward_dldc.argtypes = [I64, P, P, C.POINTER(Cam32), P, C.c_float, P, C.c_int, P]
        L.or32_backward_dldc.restype = C.c_int
        L.or64_image_loss.argtypes = [C.c_int, C.c_int, P, P, C.c_double, C.c_double,
                                      C.POINTER(C.c_double), P]
        L.or64_image_loss.restype = C.c_int
        L.or_adaptive_control.argtypes = [C.c_int, I64, P, P, C.c_int, C.c_uint64, C.c_uint64, P,
                                          I64, P]
        L.or_adaptive_control.restype = I64
        L.or_split_direction.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, P]
        L.or_split_direction.restype = None
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def cam64(camera) -> Cam64:
    c = Cam64()
    R = np.asarray(camera.rotation, np.float64).reshape(9)
    for i in range(9):
        c.R[i] = R[i]
    for i in range(3):
        c.t[i] = float(camera.translation[i])
    c.focal = float(camera.focal)
    c.cx, c.cy = map(float, camera.principal_point)
    c.width, c.height = int(camera.width), int(camera.height)
    return c


class Camera:
    """Plain camera record the oracle functions accept (any object with these attributes
    does): rotation (3x3 world->camera), translation, focal, principal_point, width, height."""

    def __init__(self, rotation, translation, focal, principal_point, width, height):
        self.rotation = np.asarray(rotation, np.float64).reshape(3, 3)
        self.translation = np.asarray(translation, np.float64).reshape(3)
        self.focal = float(focal)
        self.principal_point = (float(principal_point[0]), float(principal_point[1]))
        self.width, self.height = int(width), int(height)


def synth_scene(n, width, height, seed=2403):
    """isg-synth v1 scene restated in the oracle: (mu_sigma, rgb_opacity), both
    (n, 4) float32, byte-equal to the product's isg_synth_scene."""
    ms = np.empty((n, 4), np.float32)
    co = np.empty((n, 4), np.float32)
    lib().or_synth_scene(seed, n, width, height, _p(ms), _p(co))
    return ms, co


def synth_camera(width, height, view=0, n_views=1) -> Camera:
    """Camera `view` of an n-view isg-synth batch (the FP32 values of isg_synth_camera)."""
    v = np.zeros(15, np.float32)
    lib().or_synth_camera(width, height, view, n_views, _p(v))
    return Camera(v[:9].astype(np.float64).reshape(3, 3), v[9:12].astype(np.float64),
                  float(v[12]), (float(v[13]), float(v[14])), width, height)


def cam32(camera) -> Cam32:
    c = Cam32()
    R = np.asarray(camera.rotation, np.float64).reshape(9)
    for i in range(9):
        c.R[i] = float(np.float32(R[i]))
    for i in range(3):
        c.t[i] = float(np.float32(camera.translation[i]))
    c.focal = float(np.float32(camera.focal))
    c.cx, c.cy = (float(np.float32(v)) for v in camera.principal_point)
    c.width, c.height = int(camera.width), int(camera.height)
    return c


# ---- FP64 literal -------------------------------------------------------------------------
def project_iso64(splat8, camera):
    s = np.ascontiguousarray(splat8, np.float64)
    out = np.zeros(4)
    ok = lib().or64_project_iso(_p(s), C.byref(cam64(camera)), _p(out))
    return out if ok else None


def composite64(rgba):
    a = np.ascontiguousarray(rgba, np.float64).reshape(-1, 4)
    out = np.zeros(3)
    if lib().or64_composite(a.shape[0], _p(a), _p(out)):
        raise ValueError("composite: alpha outside [0,1]")
    return out


def render64(splats, camera, bg=(0, 0, 0), threads=0):
    s = np.ascontiguousarray(splats, np.float64).reshape(-1, 8)
    out = np.zeros((camera.height, camera.width, 3))
    b = np.asarray(bg, np.float64)
    lib().or64_render(s.shape[0], _p(s), C.byref(cam64(camera)), _p(b), threads, _p(out))
    return out


def brute_force64(splats, camera, bg=(0, 0, 0)):
    s = np.ascontiguousarray(splats, np.float64).reshape(-1, 8)
    out = np.zeros((camera.height, camera.width, 3))
    b = np.asarray(bg, np.float64)
    lib().or64_brute_force(s.shape[0], _p(s), C.byref(cam64(camera)), _p(b), _p(out))
    return out


def mse64(a, b):
    a = np.ascontiguousarray(a, np.float64).ravel()
    b = np.ascontiguousarray(b, np.float64).ravel()
    return lib().or64_mse(a.size, _p(a), _p(b))


def loss_grad64(splats, camera, target, bg=(0, 0, 0), weight=1.0):
    s = np.ascontiguousarray(splats, np.float64).reshape(-1, 8)
    t = np.ascontiguousarray(target, np.float64)
    b = np.asarray(bg, np.float64)
    g = np.zeros((s.shape[0], 8))
    loss = np.zeros(1)
    lib().or64_loss_grad(s.shape[0], _p(s), C.byref(cam64(camera)), _p(b), _p(t), weight,
                         _p(loss), _p(g))
    return float(loss[0]), g


# ---- FP32 tiled ---------------------------------------------------------------------------
def bin32(ms, co, camera):
    ms = np.ascontiguousarray(ms, np.float32)
    co = np.ascontiguousarray(co, np.float32)
    c = cam32(camera)
    nvis = C.c_int64()
    k = lib().or32_bin(ms.shape[0], _p(ms), _p(co), C.byref(c), None, None, 0, None,
                       C.byref(nvis))
    tiles = ((camera.width + 15) // 16) * ((camera.height + 15) // 16)
    keys = np.empty(k, np.uint64)
    vals = np.empty(k, np.uint32)
    ranges = np.empty((tiles, 2), np.uint32)
    lib().or32_bin(ms.shape[0], _p(ms), _p(co), C.byref(c), _p(keys), _p(vals), k, _p(ranges),
                   C.byref(nvis))
    return keys, vals, ranges, nvis.value


def render32(ms, co, camera, bg=(0, 0, 0), t_min=0.0, threads=0, want_state=False):
    ms = np.ascontiguousarray(ms, np.float32)
    co = np.ascontiguousarray(co, np.float32)
    H, W = camera.height, camera.width
    out = np.empty((H, W, 3), np.float32)
    tl = np.empty((H, W), np.float32)
    npr = np.empty((H, W), np.uint32)
    counts = np.zeros(2, np.int64)
    b = np.asarray(bg, np.float32)
    lib().or32_render(ms.shape[0], _p(ms), _p(co), C.byref(cam32(camera)), _p(b), t_min, threads,
                      _p(out), _p(tl), _p(npr), _p(counts))
    if want_state:
        return out, tl, npr, counts
    return out


def loss_backward32(ms, co, camera, target, bg=(0, 0, 0), t_min=0.0, weight=1.0, threads=0,
                    grads=None, want_image=False):
    ms = np.ascontiguousarray(ms, np.float32)
    co = np.ascontiguousarray(co, np.float32)
    t = np.ascontiguousarray(target, np.float32)
    b = np.asarray(bg, np.float32)
    if grads is None:
        grads = np.zeros((ms.shape[0], 8), np.float32)
    img = np.empty((camera.height, camera.width, 3), np.float32) if want_image else None
    loss = C.c_double()
    lib().or32_loss_backward(ms.shape[0], _p(ms), _p(co), C.byref(cam32(camera)), _p(b), t_min,
                             _p(t), weight, threads, C.byref(loss), _p(grads),
                             _p(img) if img is not None else None)
    if want_image:
        return loss.value, grads, img
    return loss.value, grads


def raw_init32(ms, co):
    """Optimizer-space state (log sigma, logit clamp(opacity, 1e-6, 1 - 1e-6)), n x 2 float32."""
    ms = np.ascontiguousarray(ms, np.float32)
    co = np.ascontiguousarray(co, np.float32)
    raw = np.zeros((ms.shape[0], 2), np.float32)
    lib().or32_raw_init(ms.shape[0], _p(ms), _p(co), _p(raw))
    return raw


def adam32(ms, co, m, v, grads, step, lr, b1=0.9, b2=0.999, eps=1e-15, raw=None):
    """In place on ms, co, m, v (all float32, C-contiguous) and raw, the persistent
    (log sigma, logit opacity) optimizer state (n x 2; None = raw_init32(ms, co), i.e. the
    first step after the splats were set).  Returns the number of skipped updates."""
    skipped = C.c_int64()
    lrs = np.asarray(lr, np.float32)
    g = np.ascontiguousarray(grads, np.float32)
    if raw is None:
        raw = raw_init32(ms, co)
    lib().or32_adam(ms.shape[0], _p(ms), _p(co), _p(raw), _p(m), _p(v), _p(g), step, _p(lrs), b1,
                    b2, eps, C.byref(skipped))
    return skipped.value


def backward_dldc32(ms, co, camera, dldc, bg=(0, 0, 0), t_min=0.0, threads=0, grads=None):
    """FP32 tiled backward for a given pixel gradient dL/dC (HWC3); accumulates into grads."""
    ms = np.ascontiguousarray(ms, np.float32)
    co = np.ascontiguousarray(co, np.float32)
    g = np.ascontiguousarray(dldc, np.float32)
    b = np.asarray(bg, np.float32)
    if grads is None:
        grads = np.zeros((ms.shape[0], 8), np.float32)
    lib().or32_backward_dldc(ms.shape[0], _p(ms), _p(co), C.byref(cam32(camera)), _p(b), t_min,
                             _p(g), threads, _p(grads))
    return grads


def image_loss64(target, fhat, lam=0.2, weight=1.0, grad=False):
    """weight * loss(target, fhat, lam) (loss.cpp:184-190) and optionally weight * dL/dfhat."""
    f = np.ascontiguousarray(target, np.float64)
    fh = np.ascontiguousarray(fhat, np.float64)
    H, W = f.shape[:2]
    g = np.zeros_like(f) if grad else None
    v = C.c_double()
    st = lib().or64_image_loss(W, H, _p(f), _p(fh), lam, weight, C.byref(v),
                               _p(g) if grad else None)
    if st == -1:
        raise ValueError("loss: lambda must be in [0,1]")
    if st == -2:
        raise ValueError("ssim: image smaller than the 11x11 window")
    return (v.value, g) if grad else v.value


class AdaptParams(C.Structure):
    """AdaptiveControlParams (optimize.hpp:14-28) with the effective particle cap."""
    _fields_ = [("prune_threshold", C.c_double), ("merge_distance_factor", C.c_double),
                ("merge_color_tol", C.c_double), ("split_sigma_max", C.c_double),
                ("max_particles", C.c_int64)]


def adaptive_control(records, params: AdaptParams, dims=3, channels=3, seed=0, round_=0):
    """Oracle prune -> merge -> split (optimize.cpp:150-284); dims 2 = the reference's 2D
    rules, dims 3 = the 3D splat rules.  Returns (records, (pruned, merged, split))."""
    R = 8 if dims == 3 else 6
    a = np.ascontiguousarray(records, np.float64).reshape(-1, R)
    cap = max(int(params.max_particles), a.shape[0]) + 1
    out = np.zeros((cap, R))
    counts = np.zeros(3, np.int64)
    m = lib().or_adaptive_control(dims, a.shape[0], _p(a), C.byref(params), channels, seed,
                                  round_, _p(out), cap, _p(counts))
    return out[:m].copy(), tuple(int(c) for c in counts)


def split_direction(seed, round_, index):
    d = np.zeros(3)
    lib().or_split_direction(seed, round_, index, _p(d))
    return d


# ---- the reference's own code (oracle/_ref, built by oracle/build_ref.sh) -----------------
_ref = None


def ref_lib():
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            raise RuntimeError("oracle/_ref/libisosplat_ref.so not built (needs /root/reference)")
        L = C.CDLL(str(REF_LIB))
        P, I64 = C.c_void_p, C.c_int64
        L.ref_render.argtypes = [I64, P, P, C.c_int, C.c_int, P, C.c_int, P, C.c_char_p, C.c_int]
        L.ref_render.restype = C.c_int
        L.ref_project_iso.argtypes = [P, P, P, C.c_char_p, C.c_int]
        L.ref_project_iso.restype = C.c_int
        L.ref_composite.argtypes = [I64, P, P, C.c_char_p, C.c_int]
        L.ref_composite.restype = C.c_int
        L.ref_mse.argtypes = [C.c_int, C.c_int, P, P]
        L.ref_mse.restype = C.c_double
        L.ref_image_loss.argtypes = [C.c_int, C.c_int, P, P, C.c_double, P, P, C.c_char_p,
                                     C.c_int]
        L.ref_image_loss.restype = C.c_int
        L.ref_adaptive_control_2d.argtypes = [I64, P, P, C.c_int, C.c_int, C.c_uint64, P, I64,
                                              C.c_char_p, C.c_int]
        L.ref_adaptive_control_2d.restype = I64
        _ref = L
    return _ref


def _ref_cam(camera):
    return np.concatenate([np.asarray(camera.rotation, np.float64).reshape(9),
                           np.asarray(camera.translation, np.float64).reshape(3),
                           [float(camera.focal)], np.asarray(camera.principal_point, np.float64)])


def ref_render(splats, camera, bg=(0, 0, 0), threads=1):
    """The reference's isosplat::render (splat3d.cpp:173-194) on (n, 8) FP64 records."""
    s = np.ascontiguousarray(splats, np.float64).reshape(-1, 8)
    c = _ref_cam(camera)
    b = np.asarray(bg, np.float64)
    out = np.zeros((camera.height, camera.width, 3))
    err = C.create_string_buffer(512)
    st = ref_lib().ref_render(s.shape[0], _p(s), _p(c), camera.width, camera.height, _p(b),
                              threads, _p(out), err, 512)
    if st:
        raise ValueError(err.value.decode())
    return out


def ref_project_iso(splat8, camera):
    s = np.ascontiguousarray(splat8, np.float64)
    c = _ref_cam(camera)
    out = np.zeros(4)
    err = C.create_string_buffer(512)
    st = ref_lib().ref_project_iso(_p(s), _p(c), _p(out), err, 512)
    if st < 0:
        raise ValueError(err.value.decode())
    return out if st else None


def ref_composite(rgba):
    a = np.ascontiguousarray(rgba, np.float64).reshape(-1, 4)
    out = np.zeros(3)
    err = C.create_string_buffer(512)
    if ref_lib().ref_composite(a.shape[0], _p(a), _p(out), err, 512):
        raise ValueError(err.value.decode())
    return out


def ref_image_loss(target, fhat, lam=0.2, grad=False):
    """The reference's loss(), l1_term(), ssim() and ssim_gradient_wrt_second()
    (loss.cpp:112-190) -> (loss, l1, ssim[, dssim/dfhat])."""
    f = np.ascontiguousarray(target, np.float64)
    fh = np.ascontiguousarray(fhat, np.float64)
    H, W = f.shape[:2]
    out = np.full(3, np.nan)
    g = np.zeros_like(f) if grad else None
    err = C.create_string_buffer(512)
    if ref_lib().ref_image_loss(W, H, _p(f), _p(fh), lam, _p(out), _p(g) if grad else None,
                                err, 512):
        raise ValueError(err.value.decode())
    return (out[0], out[1], out[2], g) if grad else (out[0], out[1], out[2])


def ref_adaptive_control_2d(records, prune_threshold=1e-3, merge_distance_factor=0.5,
                            merge_color_tol=0.05, split_sigma_max=15.0, max_particles=0,
                            channels=3, seed=0):
    """The reference's adaptive_control on IsoParticle2D records (n, 6)."""
    a = np.ascontiguousarray(records, np.float64).reshape(-1, 6)
    prm = np.array([prune_threshold, merge_distance_factor, merge_color_tol, split_sigma_max])
    cap = max(max_particles, a.shape[0]) + 1
    out = np.zeros((cap, 6))
    err = C.create_string_buffer(512)
    m = ref_lib().ref_adaptive_control_2d(a.shape[0], _p(a), _p(prm), max_particles, channels,
                                          seed, _p(out), cap, err, 512)
    if m < 0:
        raise ValueError(err.value.decode())
    return out[:m].copy()

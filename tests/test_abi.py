"""CPU tests of the drop-in boundary: libisg.so loads without a GPU, exports every symbol that
include/isg.h declares, its host-only entry points work, and device calls fail loudly (no CPU
fallback) when no GPU is present."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2403_14244_b200 import isg

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "isg.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(isg_[a-z0-9_]+)\s*\(", text)))


def test_header_declarations_are_exported():
    names = declared_symbols()
    assert len(names) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", str(isg.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (isg_[a-z0-9_]+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(isg.C_ABI_SYMBOLS) == set(names)


def test_library_loads_and_reports_version():
    L = isg.lib()
    assert L.isg_abi_version() == 2
    assert L.isg_status_string(1) == b"domain error"


def test_no_torch_types_in_header():
    text = (ROOT / "include" / "isg.h").read_text()
    for banned in (r"\bat::", r"\btorch::", r"\bTensor\b", r"\bc10\b"):
        assert not re.search(banned, text)
    assert 'extern "C"' in text


def test_synth_scene_deterministic_and_in_range():
    a = isg.synth_scene(5000, 640, 360, seed=2403)
    b = isg.synth_scene(5000, 640, 360, seed=2403)
    c = isg.synth_scene(5000, 640, 360, seed=14244)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert not np.array_equal(a[0], c[0])
    ms, co = a
    assert np.all((ms[:, 2] >= 2) & (ms[:, 2] <= 10))
    assert np.all((co[:, 3] >= 0.05) & (co[:, 3] <= 0.95))
    assert np.all((co[:, :3] >= 0) & (co[:, :3] <= 1))
    f = 1000 * 640 / 1920
    s2d = ms[:, 3] * f / ms[:, 2]
    assert np.all((s2d > 0.49) & (s2d < 8.01))
    # prefix property: the first k splats do not depend on n (counter-based RNG)
    d = isg.synth_scene(100, 640, 360, seed=2403)
    assert np.array_equal(d[0], ms[:100])


def test_synth_camera_views():
    c0 = isg.Camera.synthetic(1920, 1080)
    assert np.allclose(c0.rotation, np.eye(3)) and np.allclose(c0.translation, 0)
    assert c0.focal == 1000 and c0.principal_point == (960, 540)
    cams = [isg.Camera.synthetic(1920, 1080, k, 8) for k in range(8)]
    for k, c in enumerate(cams):
        R = c.rotation  # float32 round trip: orthonormal to float precision
        assert np.abs(R @ R.T - np.eye(3)).max() < 1e-6
        assert abs(c.translation[0] - 0.05 * (k - 3.5)) < 1e-6


def test_validation_mirrors_reference_messages():
    good = np.array([[0, 0, 2, .25, 1, .2, .1, .5]] * 2, np.float64)
    isg.validate_splats(good)
    for (j, val, msg) in [(3, 0.0, "sigma"), (0, np.inf, "mu"), (7, -0.1, "opacity"),
                          (5, np.nan, "color")]:
        bad = good.copy()
        bad[1, j] = val
        with pytest.raises(isg.DomainError, match=msg):
            isg.validate_splats(bad)
    cam = isg.Camera(np.eye(3) * 1.01, np.zeros(3), 10.0, (0, 0), 4, 4)
    with pytest.raises(isg.DomainError, match="orthonormal"):
        cam.validate()


def test_device_calls_fail_loudly_without_gpu():
    from conftest import has_cuda
    if has_cuda():
        pytest.skip("a GPU is present")
    with pytest.raises(isg.IsgError):
        isg.Renderer(0)


def _dropin(mode):
    from paper_2403_14244_b200 import build
    exe = build.build_dropin_test()
    return subprocess.run([str(exe), mode], capture_output=True, text=True, timeout=300)


def test_cpp_dropin_host_side():
    """Reference-style C++ caller code compiles against isosplat_b200.hpp; validation throws
    the reference's std::domain_error messages before any device call."""
    r = _dropin("validate")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK validate" in r.stdout


@pytest.mark.gpu
def test_cpp_dropin_render_on_gpu():
    r = _dropin("render")
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_dropin_train_on_gpu():
    r = _dropin("train")
    assert r.returncode == 0, r.stdout + r.stderr

"""Scene / camera I/O: the reference's ISPL binary + JSON and camera JSON
formats (particle_io.cpp:151-298), in Python (scene_io.py) and C++ (csrc/isosplat_io.hpp),
cross-checked against each other and against a file laid out byte-for-byte like the reference's
fixture generator (proj/tools/make_fixtures.py:79-94)."""
import json
import struct
import subprocess

import numpy as np
import pytest

from paper_2403_14244_b200 import isg, scene_io

THREE = np.array([[0.0, 0.0, 2.0, 0.25, 1.0, 0.2, 0.1, 0.5],
                  [0.35, -0.2, 3.0, 0.45, 0.2, 0.9, 0.3, 0.5],
                  [-0.3, 0.25, 4.0, 0.9, 0.1, 0.3, 1.0, 1.0]])
CAM32 = {"rotation": [[1, 0, 0], [0, 1, 0], [0, 0, 1]], "translation": [0, 0, 0], "focal": 32,
         "principal_point": [16, 16], "image_size": [32, 32]}


def write_like_make_fixtures(path):
    """Byte layout of proj/tools/make_fixtures.py:79-94 (the reference's own writer)."""
    header = json.dumps({"version": 1, "kernel_kind": "iso", "dimension": 3, "channels": 3,
                         "count": 3, "metadata": {"name": "three_splats"}}).encode()
    with open(path, "wb") as f:
        f.write(b"ISPL")
        f.write(struct.pack("<I", len(header)))
        f.write(header)
        for r in THREE:
            f.write(struct.pack("<8d", *r))


def test_load_reference_layout(tmp_path):
    p = tmp_path / "scene_three_splats.ispl"
    write_like_make_fixtures(p)
    ps = scene_io.load_particles(p)
    assert ps.count() == 3 and ps.metadata == {"name": "three_splats"}
    assert np.array_equal(ps.records, THREE)
    ms, co = ps.soa()
    assert ms.dtype == np.float32 and ms.shape == (3, 4) and co[2, 3] == 1.0


@pytest.mark.parametrize("as_json", [False, True])
def test_round_trip_exact(tmp_path, as_json):
    rng = np.random.default_rng(0)
    rec = np.concatenate([rng.normal(size=(50, 3)), rng.uniform(0.01, 1, (50, 1)),
                          rng.uniform(0, 1, (50, 3)), rng.uniform(0, 1, (50, 1))], 1)
    p = tmp_path / ("s.json" if as_json else "s.ispl")
    scene_io.save_particles(p, scene_io.ParticleSet(rec, metadata={"epoch": 3}), as_json)
    back = scene_io.load_particles(p)
    assert np.array_equal(back.records, rec) and back.metadata == {"epoch": 3}


def test_errors(tmp_path):
    with pytest.raises(RuntimeError, match="cannot open particle file"):
        scene_io.load_particles(tmp_path / "missing.ispl")
    p = tmp_path / "trunc.ispl"
    write_like_make_fixtures(p)
    p.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(RuntimeError, match="truncated particle file"):
        scene_io.load_particles(p)
    (tmp_path / "x.json").write_text('{"format": "other"}')
    with pytest.raises(RuntimeError, match="unrecognized particle file format"):
        scene_io.load_particles(tmp_path / "x.json")
    bad = dict(CAM32, quaternion=[1, 0.1, 0, 0])
    del bad["rotation"]
    (tmp_path / "c.json").write_text(json.dumps(bad))
    with pytest.raises(RuntimeError, match="quaternion norm must be 1 within 1e-9"):
        scene_io.load_camera(tmp_path / "c.json")
    bad = dict(CAM32, focal=-1)
    (tmp_path / "c2.json").write_text(json.dumps(bad))
    with pytest.raises(isg.DomainError, match="Camera.focal"):
        scene_io.load_camera(tmp_path / "c2.json")


def test_camera_quaternion_matches_rotation(tmp_path):
    th = 0.3
    q = [np.cos(th / 2), 0.0, np.sin(th / 2), 0.0]
    j = dict(CAM32, quaternion=q)
    del j["rotation"]
    (tmp_path / "q.json").write_text(json.dumps(j))
    cam = scene_io.load_camera(tmp_path / "q.json")
    R = np.array([[np.cos(th), 0, np.sin(th)], [0, 1, 0], [-np.sin(th), 0, np.cos(th)]])
    assert np.allclose(cam.rotation, R, atol=1e-15)


def test_loss_csv_and_png(tmp_path):
    scene_io.write_loss_csv(tmp_path / "loss.csv", 1.5, 10, [1.25, 1.0], [10, 9])
    assert (tmp_path / "loss.csv").read_text().splitlines() == [
        "epoch,loss,particles", "0,1.5,10", "1,1.25,10", "2,1,9"]
    img = np.zeros((4, 5, 3))
    img[1, 2] = [1.0, 0.5, 2.0]
    scene_io.write_png_rgb(tmp_path / "a.png", img)
    data = (tmp_path / "a.png").read_bytes()
    assert data[:8] == b"\x89PNG\r\n\x1a\n" and struct.unpack(">II", data[16:24]) == (5, 4)


def test_cpp_io_cross_language(tmp_path):
    from paper_2403_14244_b200 import build
    scene_io.save_particles(tmp_path / "py_scene.ispl", scene_io.ParticleSet(THREE.copy()))
    scene_io.save_particles(tmp_path / "py_scene.json", scene_io.ParticleSet(THREE.copy()), True)
    exe = build.build_dropin_test()
    r = subprocess.run([str(exe), "io", str(tmp_path)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    for f in ("cpp_scene.ispl", "cpp_scene.json"):
        ps = scene_io.load_particles(tmp_path / f)
        assert np.array_equal(ps.records, THREE) and ps.metadata == {"name": "three_splats"}
    cam = scene_io.load_camera(tmp_path / "cpp_camera.json")
    assert cam.focal == 32 and cam.width == 32


@pytest.mark.gpu
def test_render3d_flow_on_gpu(tmp_path):
    """The reference's render3d flow on B200: file -> drop-in render -> PNG, and the same scene
    through the Python API matches the known answers."""
    from paper_2403_14244_b200 import build
    write_like_make_fixtures(tmp_path / "scene.ispl")
    (tmp_path / "camera.json").write_text(json.dumps(CAM32))
    exe = build.build_dropin_test()
    r = subprocess.run([str(exe), "render3d", str(tmp_path / "scene.ispl"),
                        str(tmp_path / "camera.json"), str(tmp_path / "out.png")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "rendered 3 splats to" in r.stdout
    assert (tmp_path / "out.png").read_bytes()[:4] == b"\x89PNG"
    ps = scene_io.load_particles(tmp_path / "scene.ispl")
    img = isg.render(ps.records, scene_io.load_camera(tmp_path / "camera.json"),
                     isg.RenderOptions(t_min=0.0))
    assert abs(img[16, 16, 0] - 0.540942539951) < 1e-4
    # bad input -> the reference's exit code 2 (kExitBadInput)
    (tmp_path / "bad.ispl").write_bytes(b"ISPL\x01")
    r = subprocess.run([str(exe), "render3d", str(tmp_path / "bad.ispl"),
                        str(tmp_path / "camera.json"), str(tmp_path / "o.png")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "truncated particle file" in r.stderr

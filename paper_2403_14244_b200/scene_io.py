"""Scene and camera I/O feeding the GPU upload — the formats of the reference's particle_io
(/root/reference/proj/include/isosplat/particle_io.hpp:36-51, src/particle_io.cpp:151-298), so
scenes written by the reference's tools load unchanged and vice versa.

  ISPL binary: magic "ISPL", u32 LE header length, JSON header {version, kernel_kind,
               dimension, channels, count, metadata}, then count records of LE doubles;
               iso 3D record = mu.xyz sigma color.rgb opacity (8 doubles)
  ISPL-json:   the same header with "format": "ISPL-json" and "particles": [[8 numbers], ...]
  camera JSON: {"rotation": 3x3 rows | "quaternion": [w,x,y,z], "translation": [x,y,z],
                "focal": f, "principal_point": [cx,cy], "image_size": [w,h]}

Errors keep the reference's messages (RuntimeError here = std::runtime_error there; an invalid
camera raises DomainError like Camera::validate).  Only the isotropic 3D kind is materialised
(the hot path); other kinds are recognised and rejected with a clear message.
"""
from __future__ import annotations

import json
import math
import struct
from dataclasses import dataclass, field
from pathlib import Path
from typing import Any, Dict, Sequence

import numpy as np

from .isg import Camera

MAGIC = b"ISPL"


@dataclass
class ParticleSet:
    """particle_io.hpp:20-34 restricted to what the 3D hot path consumes."""
    records: np.ndarray  # (n, 8) float64: mu.xyz sigma color.rgb opacity
    kind: str = "iso"
    dimension: int = 3
    channels: int = 3
    format_version: int = 1
    metadata: Dict[str, Any] = field(default_factory=dict)

    def count(self) -> int:
        return int(self.records.shape[0])

    def values_per_record(self) -> int:  # particle_io.cpp:32-35
        if self.dimension == 2:
            return (3 if self.kind == "iso" else 5) + self.channels
        return 8 if self.kind == "iso" else 14

    def soa(self):
        """-> (mu_sigma (n,4) f32, rgb_opacity (n,4) f32) for Renderer.set_scene."""
        r = self.records
        return (np.ascontiguousarray(r[:, 0:4], np.float32),
                np.ascontiguousarray(r[:, 4:8], np.float32))


def _header(ps: ParticleSet) -> dict:
    return {"version": ps.format_version, "kernel_kind": ps.kind, "dimension": ps.dimension,
            "channels": ps.channels, "count": ps.count(), "metadata": ps.metadata}


def _set_from_header(h: dict, path: str) -> ParticleSet:  # particle_io.cpp:128-147
    version = h["version"]
    if version != 1:
        raise RuntimeError(f"unknown particle file version {version}")
    kind = h["kernel_kind"]
    if kind not in ("iso", "aniso"):
        raise RuntimeError("unknown kernel_kind: " + str(kind))
    dim = h["dimension"]
    if dim not in (2, 3):
        raise RuntimeError("particle file: dimension must be 2 or 3")
    ch = h["channels"]
    if ch not in (1, 3):
        raise RuntimeError("particle file: channels must be 1 or 3")
    return ParticleSet(records=np.zeros((0, 8)), kind=kind, dimension=dim, channels=ch,
                       format_version=version, metadata=h.get("metadata", {}))


def save_particles(path, ps: ParticleSet, as_json: bool = False) -> None:
    """save_particles, particle_io.cpp:151-182 (iso 3D sets)."""
    if ps.kind != "iso" or ps.dimension != 3:
        raise RuntimeError("save_particles: only isotropic 3D sets are supported here")
    rec = np.ascontiguousarray(ps.records, dtype="<f8").reshape(-1, 8)
    if as_json:
        j = _header(ps)
        j["format"] = "ISPL-json"
        j["particles"] = [[float(v) for v in row] for row in rec]
        Path(path).write_text(json.dumps(j, indent=2) + "\n")
        return
    header = json.dumps(_header(ps), separators=(",", ":")).encode()
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<I", len(header)))
        f.write(header)
        f.write(rec.tobytes())


def load_particles(path) -> ParticleSet:
    """load_particles, particle_io.cpp:184-236; returns the iso 3D set."""
    path = str(path)
    try:
        data = Path(path).read_bytes()
    except OSError:
        raise RuntimeError("cannot open particle file: " + path) from None
    if data[:4] == MAGIC:
        if len(data) < 8:
            raise RuntimeError("truncated particle file: " + path)
        (hlen,) = struct.unpack("<I", data[4:8])
        if len(data) < 8 + hlen:
            raise RuntimeError("truncated particle file: " + path)
        h = json.loads(data[8:8 + hlen].decode())
        ps = _set_from_header(h, path)
        count = int(h["count"])
        nbytes = count * ps.values_per_record() * 8
        payload = data[8 + hlen:8 + hlen + nbytes]
        if len(payload) != nbytes:
            raise RuntimeError("truncated particle file: " + path)
        values = np.frombuffer(payload, dtype="<f8").reshape(count, ps.values_per_record())
    else:
        try:
            j = json.loads(data.decode())
        except (UnicodeDecodeError, json.JSONDecodeError):
            raise RuntimeError("unrecognized particle file format: " + path) from None
        if not isinstance(j, dict) or j.get("format", "") != "ISPL-json":
            raise RuntimeError("unrecognized particle file format: " + path)
        ps = _set_from_header(j, path)
        count = int(j["count"])
        recs = j["particles"]
        if len(recs) != count:
            raise RuntimeError("particle file: count mismatch")
        if any(len(r) != ps.values_per_record() for r in recs):
            raise RuntimeError("particle file: bad record arity")
        values = np.asarray(recs, dtype=np.float64).reshape(count, ps.values_per_record())
    if ps.kind != "iso" or ps.dimension != 3:
        raise RuntimeError("scene file must hold isotropic 3D splats (kernel_kind=iso, dimension=3)")
    ps.records = np.array(values, dtype=np.float64)
    return ps


def camera_from_json(j: dict) -> Camera:
    """camera_from_json, particle_io.cpp:238-268."""
    if "rotation" in j:
        r = j["rotation"]
        if len(r) != 3:
            raise RuntimeError("camera: rotation must be 3 rows")
        R = np.array([[float(r[i][k]) for k in range(3)] for i in range(3)])
    elif "quaternion" in j:
        q = j["quaternion"]
        if len(q) != 4:
            raise RuntimeError("camera: quaternion must be [w,x,y,z]")
        w, x, y, z = (float(v) for v in q)
        if abs(math.sqrt(w * w + x * x + y * y + z * z) - 1.0) > 1e-9:
            raise RuntimeError("camera: quaternion norm must be 1 within 1e-9")
        R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                      [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                      [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])
    else:
        raise RuntimeError("camera: missing rotation or quaternion")
    t = j["translation"]
    pp = j["principal_point"]
    size = j["image_size"]
    cam = Camera(R, np.array([float(t[i]) for i in range(3)]), float(j["focal"]),
                 (float(pp[0]), float(pp[1])), int(size[0]), int(size[1]))
    cam.validate()
    return cam


def load_camera(path) -> Camera:
    """load_camera, particle_io.cpp:270-284."""
    path = str(path)
    try:
        text = Path(path).read_text()
    except OSError:
        raise RuntimeError("cannot open camera file: " + path) from None
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise RuntimeError(f"camera JSON parse error in {path}: {e}") from None
    try:
        return camera_from_json(j)
    except (KeyError, TypeError, IndexError) as e:
        raise RuntimeError(f"camera JSON field error in {path}: {e}") from None


def camera_to_json(cam: Camera) -> dict:
    R = np.asarray(cam.rotation, dtype=np.float64)
    return {"rotation": R.tolist(), "translation": [float(v) for v in cam.translation],
            "focal": float(cam.focal), "principal_point": [float(v) for v in cam.principal_point],
            "image_size": [int(cam.width), int(cam.height)]}


def write_loss_csv(path, initial_loss: float, initial_count: int,
                   loss_history: Sequence[float], count_history: Sequence[int]) -> None:
    """write_loss_csv, particle_io.cpp:286-298 (precision 17)."""
    lines = ["epoch,loss,particles", f"0,{initial_loss:.17g},{initial_count}"]
    for i, v in enumerate(loss_history):
        c = count_history[i] if i < len(count_history) else initial_count
        lines.append(f"{i + 1},{v:.17g},{c}")
    Path(path).write_text("\n".join(lines) + "\n")


def write_png_rgb(path, img: np.ndarray) -> None:
    """8-bit RGB PNG of an (H, W, 3) image with the reference's quantisation (clamp to [0,1],
    round half up: png_io.hpp:17-21)."""
    import zlib

    q = np.floor(np.clip(np.asarray(img, np.float64), 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)
    h, w = q.shape[:2]
    raw = b"".join(b"\x00" + q[y].tobytes() for y in range(h))

    def chunk(tag, payload):
        c = struct.pack(">I", len(payload)) + tag + payload
        return c + struct.pack(">I", zlib.crc32(tag + payload) & 0xFFFFFFFF)

    png = b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 8, 2, 0, 0, 0))
    png += chunk(b"IDAT", zlib.compress(raw, 6)) + chunk(b"IEND", b"")
    Path(path).write_bytes(png)

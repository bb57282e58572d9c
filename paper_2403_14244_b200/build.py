"""In-tree build of the native pieces (no JIT cache: the .so files travel with the repo).

  paper_2403_14244_b200/libisg.so   sm_100a kernels + the C-ABI (include/isg.h)
  oracle/_build/libisg_oracle.so    CPU oracle (test infrastructure only)
  oracle/_ref/libisosplat_ref.so    the reference's own splat3d.cpp/image.cpp, compiled from
                                    /root/reference when present (oracle/build_ref.sh)
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libisg.so"
ORACLE_DIR = ROOT / "oracle"
ORACLE_LIB = ORACLE_DIR / "_build" / "libisg_oracle.so"
REF_LIB = ORACLE_DIR / "_ref" / "libisosplat_ref.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["capi.cu", "k_preprocess.cu", "k_bin.cu", "k_sort.cu", "k_blend.cu",
              "k_blend_bwd.cu", "k_ssim.cu", "k_adam.cu", "k_adapt.cu", "synth.cu"]
# per-file flags: adaptive control rounds every FP64 product/sum like the oracle (no FMA)
CU_EXTRA = {"k_adapt.cu": ["-fmad=false"]}


def _digest(paths) -> str:
    h = hashlib.sha256()
    for p in sorted(paths):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()


def _run(cmd, cwd=None):
    print("+", " ".join(str(c) for c in cmd), flush=True)
    subprocess.run([str(c) for c in cmd], check=True, cwd=cwd)


def build_isg(force: bool = False) -> Path:
    srcs = [CSRC / s for s in CU_SOURCES]
    deps = srcs + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "isg.h", Path(__file__)]
    stamp = PKG / ".libisg.sha256"
    digest = _digest(deps)
    if not force and LIB.exists() and stamp.exists() and stamp.read_text() == digest:
        return LIB
    objdir = ROOT / "build" / "isg"
    objdir.mkdir(parents=True, exist_ok=True)
    objs = []
    for s in srcs:
        o = objdir / (s.stem + ".o")
        _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fopenmp",
              "-Xptxas", "-v", *CU_EXTRA.get(s.name, []), "-I", ROOT / "include", "-c", s,
              "-o", o])
        objs.append(o)
    _run([NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC,-fopenmp", "-o", LIB, *objs,
          "-ldl", "-lgomp"])
    stamp.write_text(digest)
    return LIB


def build_oracle(force: bool = False) -> Path:
    src = ORACLE_DIR / "isg_oracle.c"
    stamp = ORACLE_LIB.with_suffix(".sha256")
    digest = _digest([src])
    if not force and ORACLE_LIB.exists() and stamp.exists() and stamp.read_text() == digest:
        return ORACLE_LIB
    ORACLE_LIB.parent.mkdir(parents=True, exist_ok=True)
    # strict IEEE like the reference (proj/CMakeLists.txt:11-17): no FMA contraction, no fast-math
    _run(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
          "-shared", "-o", ORACLE_LIB, src, "-lm"])
    stamp.write_text(digest)
    return ORACLE_LIB


def build_ref(force: bool = False) -> Path | None:
    """Compile the reference's own hot-path sources when /root/reference is present."""
    script = ORACLE_DIR / "build_ref.sh"
    if not Path("/root/reference/proj/src/splat3d.cpp").exists() or not script.exists():
        return REF_LIB if REF_LIB.exists() else None
    if REF_LIB.exists() and not force:
        return REF_LIB
    _run(["bash", script])
    return REF_LIB if REF_LIB.exists() else None


DROPIN_SRC = ROOT / "tests" / "cpp" / "test_dropin.cpp"
DROPIN_BIN = ROOT / "build" / "test_dropin"


def build_dropin_test(force: bool = False) -> Path:
    """The C++ drop-in (csrc/isosplat_b200.hpp) used the way the reference's caller uses it."""
    deps = [DROPIN_SRC, CSRC / "isosplat_b200.hpp", CSRC / "isosplat_io.hpp",
            ROOT / "include" / "isg.h"]
    stamp = DROPIN_BIN.with_suffix(".sha256")
    digest = _digest(deps)
    if not force and DROPIN_BIN.exists() and stamp.exists() and stamp.read_text() == digest:
        return DROPIN_BIN
    DROPIN_BIN.parent.mkdir(parents=True, exist_ok=True)
    _run(["g++", "-std=c++20", "-O2", "-Wall", "-I", ROOT / "include", "-I", CSRC, DROPIN_SRC,
          "-L", PKG, "-lisg", "-Wl,-rpath,$ORIGIN/../paper_2403_14244_b200", "-o", DROPIN_BIN])
    stamp.write_text(digest)
    return DROPIN_BIN


def build_all(force: bool = False) -> None:
    build_isg(force)
    build_oracle(force)
    build_ref(force)
    build_dropin_test(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)

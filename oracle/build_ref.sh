#!/usr/bin/env bash
# Compile the REFERENCE's own hot-path sources, where they lie under /root/reference, into
# oracle/_ref/libisosplat_ref.so (git-ignored; travels to the GPU box with the snapshot).
#
#   /root/reference/proj/src/splat3d.cpp   render / project_iso / composite / validate
#   /root/reference/proj/src/image.cpp     ImageGrid, mse
#   /root/reference/proj/src/loss.cpp      L1 + D-SSIM loss, ssim gradient (+ reconstruct.cpp,
#                                          which loss.cpp's 2D overloads link against)
#   /root/reference/proj/src/optimize.cpp  adaptive_control (prune / merge / split), 2D
#
# The reference's build system is not used (it needs cmake + Eigen + libpng + vendored
# CLI11/json, none of which exist here).  Eigen is replaced by oracle/eigen_shim, a minimal
# from-scratch implementation of the Eigen API subset these translation units use.  The
# flags follow the reference's CMakeLists (C++20, strict IEEE: -ffp-contract=off,
# proj/CMakeLists.txt:4-17).  No reference source is copied into this repository.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF=/root/reference/proj
OUT="$HERE/_ref"
mkdir -p "$OUT"
g++ -std=c++20 -O2 -ffp-contract=off -fPIC -shared -pthread \
    -I "$HERE/eigen_shim" -I "$REF/include" \
    "$REF/src/splat3d.cpp" "$REF/src/image.cpp" "$REF/src/loss.cpp" "$REF/src/reconstruct.cpp" \
    "$REF/src/optimize.cpp" \
    "$HERE/ref_capi.cpp" \
    -o "$OUT/libisosplat_ref.so"
echo "built $OUT/libisosplat_ref.so"

"""paper_2403_14244_b200 — B200-native isotropic Gaussian-splat hot path.

The product is libisg.so (sm_100a kernels behind the C-ABI in include/isg.h).  This package
holds its Python binding (`isg`), the C++ drop-in header (csrc/isosplat_b200.hpp), the
multi-GPU view-batch driver (`view_batch`) and the in-tree build (`build`).
"""
from .isg import (AdamConfig, Camera, DomainError, IsgError, Renderer, RenderOptions,  # noqa: F401
                  render, splats_to_soa, synth_scene, validate_splats)

__all__ = ["AdamConfig", "Camera", "DomainError", "IsgError", "Renderer", "RenderOptions",
           "render", "splats_to_soa", "synth_scene", "validate_splats"]

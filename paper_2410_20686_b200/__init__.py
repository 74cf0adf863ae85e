"""B200-native ODGS rasterizer (arXiv 2410.20686): sm_100a kernels behind a C ABI.

The product is libodgs_b200.so (paper_2410_20686_b200/_lib) and its C ABI
(include/odgs_b200.h); this package is the Python mirror of the reference's
rasterizer API over that ABI.
"""
from .rasterizer import (CameraPose, Context, DomainError, GaussianCloud, GradBuffers, InvalidArgument,
                         OdgsError, OdgsRuntimeError, RenderOutput, RenderSettings, Splat2D, SplatGrads,
                         backward, cull, grad_pixels_to_splats, prepare_render, project_gaussian,
                         rasterize_splats, render, render_band)
from .densify import DensifyConfig, DensifyStats, Rng, TrainState, densify_and_prune, dynamic_threshold, reset_opacity

__all__ = ["CameraPose", "Context", "DomainError", "GaussianCloud", "GradBuffers", "InvalidArgument",
           "OdgsError", "OdgsRuntimeError", "RenderOutput", "RenderSettings", "Splat2D", "SplatGrads", "backward",
           "cull", "grad_pixels_to_splats", "project_gaussian",
           "prepare_render", "rasterize_splats", "render", "render_band", "DensifyConfig", "DensifyStats", "Rng", "TrainState",
           "densify_and_prune", "dynamic_threshold", "reset_opacity"]

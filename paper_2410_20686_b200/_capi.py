"""ctypes binding of the C ABI in include/odgs_b200.h (libodgs_b200.so).

This is plumbing for tests and bench.py; the product is the C ABI and the sm_100a
kernels behind it. Loading fails loudly if the library has not been built — there
is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("ODGS_B200_LIB", _HERE / "_lib" / "libodgs_b200.so"))

MEM_HOST = 0
MEM_DEVICE = 1
ACCUMULATE = 0x1
FRAME_KEEP_COV2D = 0x1
FRAME_PLAIN_BLEND = 0x2
FRAME_KEEP_SPLAT_GRADS = 0x4
FRAME_COUNT_WORK = 0x8

(FRAME_IMAGE, FRAME_TRANSMITTANCE, FRAME_WALKED, FRAME_TILE_OFFSETS, FRAME_TILE_ENTRIES,
 FRAME_INSTANCE_SPLAT, FRAME_INSTANCE_SHIFT, FRAME_SPLAT_INDEX, FRAME_SPLAT_MEAN, FRAME_SPLAT_COV2D,
 FRAME_SPLAT_INV, FRAME_SPLAT_DEPTH, FRAME_SPLAT_RADIUS, FRAME_SPLAT_OPACITY, FRAME_SPLAT_COLOR,
 FRAME_SPLAT_CLAMPED, FRAME_SPLATGRAD_MEAN, FRAME_SPLATGRAD_COV2D, FRAME_SPLATGRAD_OPACITY,
 FRAME_SPLATGRAD_COLOR) = range(20)

IPC_HANDLE_BYTES = 72

STATUS_OK = 0
STATUS_INVALID_ARGUMENT = 1
STATUS_RUNTIME = 2
STATUS_DOMAIN = 3
STATUS_CUDA = 4
STATUS_OUT_OF_MEMORY = 5


class Settings(C.Structure):
    _fields_ = [("near_radius", C.c_float), ("far_radius", C.c_float), ("tile_size", C.c_int32),
                ("alpha_clamp", C.c_float), ("transmittance_floor", C.c_float),
                ("cutoff_sigma", C.c_float), ("lowpass_dilation", C.c_float),
                ("max_elevation", C.c_float), ("threads", C.c_int32)]


class Camera(C.Structure):
    _fields_ = [("rotation", C.c_float * 9), ("translation", C.c_float * 3),
                ("width", C.c_int32), ("height", C.c_int32)]


class Cloud(C.Structure):
    _fields_ = [("n", C.c_int64), ("means", C.c_void_p), ("rotations", C.c_void_p),
                ("log_scales", C.c_void_p), ("raw_opacities", C.c_void_p), ("colors", C.c_void_p),
                ("memory", C.c_int32), ("sh_degree", C.c_int32), ("sh_rest", C.c_void_p)]


class Grads(C.Structure):
    _fields_ = [("means", C.c_void_p), ("rotations", C.c_void_p), ("log_scales", C.c_void_p),
                ("raw_opacities", C.c_void_p), ("colors", C.c_void_p),
                ("pixel_grad_norm", C.c_void_p), ("one_minus_cos", C.c_void_p),
                ("observed", C.c_void_p), ("memory", C.c_int32), ("sh_rest", C.c_void_p)]


class Params(C.Structure):
    _fields_ = [("n", C.c_int64), ("means", C.c_void_p), ("rotations", C.c_void_p), ("log_scales", C.c_void_p),
                ("raw_opacities", C.c_void_p), ("colors", C.c_void_p)]


class TrainState(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("means_m", "means_v", "rot_m", "rot_v", "scale_m", "scale_v", "opac_m",
                                          "opac_v", "color_m", "color_v", "grad_accum", "elev_accum",
                                          "grad_count")]


class AdamParams(C.Structure):
    _fields_ = [("lr_means", C.c_float), ("lr_rotation", C.c_float), ("lr_scale", C.c_float),
                ("lr_opacity", C.c_float), ("lr_color", C.c_float), ("step", C.c_int64)]


class DensifyConfig(C.Structure):
    _fields_ = [("grad_threshold_min", C.c_double), ("grad_threshold_max", C.c_double),
                ("percent_dense", C.c_double), ("opacity_prune_floor", C.c_double),
                ("split_scale_divisor", C.c_double)]


class DensifyStats(C.Structure):
    _fields_ = [("cloned", C.c_int64), ("split", C.c_int64), ("pruned", C.c_int64), ("n_out", C.c_int64)]


class Cloud64(C.Structure):
    _fields_ = [("n", C.c_int64), ("means", C.c_void_p), ("rotations", C.c_void_p), ("log_scales", C.c_void_p),
                ("raw_opacities", C.c_void_p), ("colors", C.c_void_p)]


class Splat(C.Structure):  # odgs_splat (Splat2D, projection.hpp:163-174)
    _fields_ = [("pixel_mean", C.c_float * 2), ("cov2d", C.c_float * 4), ("cov2d_inv", C.c_float * 4),
                ("depth", C.c_float), ("radius", C.c_float), ("opacity", C.c_float), ("color", C.c_float * 3),
                ("index", C.c_int64), ("pole_clamped", C.c_int32)]


class FrameInfo(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("tiles_x", C.c_int32),
                ("tiles_y", C.c_int32), ("n_gaussians", C.c_int64), ("n_splats", C.c_int64),
                ("n_instances", C.c_int64), ("n_entries", C.c_int64), ("row_begin", C.c_int32),
                ("row_end", C.c_int32)]


# Every symbol include/odgs_b200.h declares: name -> (restype, argtypes).
_P = C.c_void_p
SIGNATURES = {
    "odgs_default_settings": (Settings, []),
    "odgs_abi_version": (C.c_int, []),
    "odgs_ctx_create": (C.c_int, [C.c_int, _P, C.POINTER(_P)]),
    "odgs_ctx_destroy": (None, [_P]),
    "odgs_ctx_set_stream": (C.c_int, [_P, _P]),
    "odgs_ctx_stream": (_P, [_P]),
    "odgs_synchronize": (C.c_int, [_P]),
    "odgs_last_error": (C.c_int, [_P, C.POINTER(C.c_int64), C.c_char_p, C.c_size_t]),
    "odgs_ctx_launch_count": (C.c_int64, [_P]),
    "odgs_ctx_set_async": (C.c_int, [_P, C.c_int]),
    "odgs_frame_check": (C.c_int, [_P, _P, C.POINTER(C.c_int32)]),
    "odgs_frame_create": (C.c_int, [_P, C.POINTER(_P)]),
    "odgs_frame_destroy": (None, [_P]),
    "odgs_frame_set_flags": (C.c_int, [_P, C.c_uint32]),
    "odgs_frame_get_info": (C.c_int, [_P, C.POINTER(FrameInfo)]),
    "odgs_frame_download": (C.c_int, [_P, _P, C.c_int, _P, C.c_size_t]),
    "odgs_frame_work": (C.c_int, [_P, _P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "odgs_frame_backward_work": (C.c_int, [_P, _P, C.POINTER(C.c_int64), C.c_int32]),
    "odgs_frame_device_ptr": (C.c_int, [_P, C.c_int, C.POINTER(_P)]),
    "odgs_prepare_render": (C.c_int, [_P, C.POINTER(Cloud), C.POINTER(Camera), C.POINTER(Settings), _P]),
    "odgs_render": (C.c_int, [_P, C.POINTER(Cloud), C.POINTER(Camera), C.POINTER(Settings), _P]),
    "odgs_render_band": (C.c_int, [_P, C.POINTER(Cloud), C.POINTER(Camera), C.POINTER(Settings), C.c_int32,
                                   C.c_int32, _P]),
    "odgs_rasterize_splats": (C.c_int, [_P, C.c_int64, C.c_int64, _P, _P, _P, _P, _P, _P, _P, C.c_int32,
                                        C.c_int32, C.POINTER(Settings), _P]),
    "odgs_project_gaussian": (C.c_int, [_P, C.POINTER(Cloud), C.c_int64, C.POINTER(Camera), C.POINTER(Settings),
                                        C.POINTER(Splat), C.POINTER(C.c_int32)]),
    "odgs_grad_pixels_to_splats": (C.c_int, [_P, _P, _P, C.c_int32, C.POINTER(Settings), _P, _P, _P, _P]),
    "odgs_backward": (C.c_int, [_P, C.POINTER(Cloud), C.POINTER(Camera), _P, _P, C.c_int32,
                                C.POINTER(Settings), C.POINTER(Grads), C.POINTER(C.c_double), C.c_uint32]),
    "odgs_ctx_set_profiling": (C.c_int, [_P, C.c_int]),
    "odgs_ctx_stage_times": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int]),
    "odgs_ctx_reset_stage_times": (None, [_P]),
    "odgs_stage_name": (C.c_char_p, [C.c_int]),
    "odgs_measure_fp32_tflops": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "odgs_photometric_loss": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, C.c_float, _P, C.POINTER(C.c_double)]),
    "odgs_photometric_loss_async": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, C.c_float, _P, _P]),
    "odgs_adam_step": (C.c_int, [_P, C.POINTER(Params), C.POINTER(Grads), C.POINTER(TrainState),
                                 C.POINTER(AdamParams)]),
    "odgs_default_densify_config": (None, [C.POINTER(DensifyConfig)]),
    "odgs_rng_create": (_P, [C.c_uint32]),
    "odgs_rng_destroy": (None, [_P]),
    "odgs_rng_next": (C.c_uint32, [_P]),
    "odgs_rng_unit_ball": (None, [_P, C.c_int64, C.POINTER(C.c_float)]),
    "odgs_densify_plan": (C.c_int, [_P, C.POINTER(Params), C.POINTER(TrainState), C.POINTER(DensifyConfig),
                                    C.c_float, C.POINTER(DensifyStats)]),
    "odgs_densify_apply": (C.c_int, [_P, C.POINTER(Params), C.POINTER(TrainState), C.POINTER(C.c_float),
                                     C.POINTER(Params), C.POINTER(TrainState)]),
    "odgs_reset_opacity": (C.c_int, [_P, C.POINTER(Params), C.POINTER(TrainState), C.c_float]),
    "odgs_dynamic_threshold": (C.c_int, [C.c_double, C.POINTER(DensifyConfig), C.POINTER(C.c_double)]),
    "odgs_io_last_error": (C.c_size_t, [C.c_char_p, C.c_size_t]),
    "odgs_ply_vertex_count": (C.c_int, [C.c_char_p, C.POINTER(C.c_int64)]),
    "odgs_load_pointcloud": (C.c_int, [C.c_char_p, C.c_int64, _P, _P]),
    "odgs_save_pointcloud": (C.c_int, [C.c_char_p, C.c_int64, _P, _P, C.c_int32]),
    "odgs_save_checkpoint": (C.c_int, [C.c_char_p, C.POINTER(Cloud64)]),
    "odgs_load_checkpoint": (C.c_int, [C.c_char_p, C.POINTER(Cloud64)]),
    "odgs_init_from_points": (C.c_int, [_P, C.c_int64, _P, _P, C.c_int32, C.POINTER(Cloud64), _P]),
    "odgs_frame_set_image_peers": (C.c_int, [_P, C.c_int32, C.POINTER(_P)]),
    "odgs_ipc_get_handle": (C.c_int, [_P, _P]),
    "odgs_ipc_open": (C.c_int, [_P, C.POINTER(_P)]),
    "odgs_ipc_close": (C.c_int, [_P]),
    "odgs_cull": (C.c_int, [_P, C.POINTER(Cloud), C.POINTER(Camera), C.c_float, C.c_float,
                            C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
}

_lib = None


def load_library(path: Path | str | None = None) -> C.CDLL:
    """Loads libodgs_b200.so and binds every declared symbol (raises if absent)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise ImportError(f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib

"""ctypes access to the CPU oracle (oracle/libodgs_oracle.so) — test infrastructure only.

The oracle is the Eigen-free restatement of the reference hot path
(oracle/odgs_oracle.hpp); it is built from the repo's own sources with
oracle/Makefile, here and on the GPU box.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_DIR = ROOT / "oracle"
LIB = ORACLE_DIR / "_build" / "libodgs_oracle.so"
REF_TESTS = ORACLE_DIR / "_build" / "ref_tests"

_lib = None


def build():
    subprocess.run(["make", "-C", str(ORACLE_DIR), "-j4", str(LIB), str(REF_TESTS)], check=True,
                   stdout=subprocess.DEVNULL)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB))
        dp = C.POINTER(C.c_double)
        L.oracle_render.restype = C.c_int
        L.oracle_render.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int64, dp, dp, dp, dp, dp, dp, dp, C.c_int,
                                    C.c_int, dp, C.c_int, C.c_int, dp, C.POINTER(C.c_void_p), C.c_char_p, C.c_int]
        L.oracle_backward.restype = C.c_int
        L.oracle_backward.argtypes = [C.c_void_p, dp, C.c_int, C.c_char_p, C.c_int]
        L.oracle_get.restype = C.c_int64
        L.oracle_get.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
        L.oracle_free.argtypes = [C.c_void_p]
        L.oracle_rasterize_splats.restype = C.c_int
        L.oracle_rasterize_splats.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p), C.c_char_p, C.c_int]
        L.oracle_random_cloud.argtypes = [C.c_uint32, C.c_int, dp, C.c_int, dp, dp, dp, dp, dp]
        L.oracle_photometric_loss.restype = C.c_double
        L.oracle_photometric_loss.argtypes = [dp, dp, C.c_int, C.c_int, C.c_double, dp]
        L.oracle_hardware_concurrency.restype = C.c_int
        L.oracle_densify.restype = C.c_int
        L.oracle_densify.argtypes = [C.c_int, C.c_int64, dp, dp, dp, dp, C.POINTER(C.c_int32), dp, C.c_double,
                                     C.c_uint32, C.c_int64, dp, dp, C.POINTER(C.c_int64), C.POINTER(C.c_uint32),
                                     C.c_char_p, C.c_int]
        L.oracle_reset_opacity.restype = C.c_int
        L.oracle_reset_opacity.argtypes = [C.c_int, C.c_int64, dp, C.c_double, C.c_char_p, C.c_int]
        L.oracle_unit_ball.restype = C.c_uint32
        L.oracle_unit_ball.argtypes = [C.c_uint32, C.c_int64, C.POINTER(C.c_float)]
        L.oracle_dynamic_threshold.restype = C.c_int
        L.oracle_dynamic_threshold.argtypes = [C.c_double, C.c_double, C.c_double, dp]
        L.oracle_init_scales.restype = None
        L.oracle_init_scales.argtypes = [C.c_int64, dp, dp, dp]
        _lib = L
    return _lib


def init_scales(positions):
    """Brute-force init_from_points scales (io.cpp:268-296): (scale, log_scale) per point."""
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    n = pos.shape[1]
    sc = np.zeros(n)
    ls = np.zeros(n)
    dp = C.POINTER(C.c_double)
    lib().oracle_init_scales(n, pos.ctypes.data_as(dp), sc.ctypes.data_as(dp), ls.ctypes.data_as(dp))
    return sc, ls


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# ------------------------------------------------------------------ scenes (mt19937, scenes.hpp)
DEFAULT_BOUNDS = (0.5, 20.0, 1.45, 0.05, 0.95, 0.005, 0.05)


def random_cloud(seed: int, n: int, bounds=DEFAULT_BOUNDS, as_float: bool = True):
    """scenes::random_cloud<float|double>(std::mt19937(seed), n, bounds) as float64 arrays."""
    b = np.asarray(bounds, dtype=np.float64)
    means, rot, ls = np.zeros((3, n)), np.zeros((4, n)), np.zeros((3, n))
    op, col = np.zeros(n), np.zeros((3, n))
    lib().oracle_random_cloud(seed, n, _dp(b), int(as_float), _dp(means), _dp(rot), _dp(ls), _dp(op), _dp(col))
    return means, rot, ls, op, col


# ------------------------------------------------------------------ render / backward
@dataclass
class OracleSettings:
    near: float = 0.01
    far: float = 1000.0
    tile: int = 16
    alpha_clamp: float = 0.99
    floor: float = 1e-4
    cutoff: float = 3.0
    lowpass: float = 0.3
    max_elevation: float = float(np.float32(85.0) * np.float32(np.pi) / np.float32(180.0))

    def array(self):
        return np.array([self.near, self.far, self.tile, self.alpha_clamp, self.floor, self.cutoff,
                         self.lowpass, self.max_elevation], dtype=np.float64)


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class OracleFrame:
    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if self.h:
            lib().oracle_free(self.h)
            self.h = None

    def get(self, which: str):
        L = lib()
        n = L.oracle_get(self.h, which.encode(), None)
        if n < 0:
            raise KeyError(which)
        dtype = {"walked": np.int32, "tile_offsets": np.int32, "tile_entries": np.int32, "inst_splat": np.int32,
                 "splat_index": np.int64, "splat_clamped": np.int32, "stats": np.int64,
                 "g_observed": np.int32}.get(which, np.float64)
        out = np.empty(n, dtype=dtype)
        L.oracle_get(self.h, which.encode(), out.ctypes.data)
        return out

    def rasterize_splats(self, portable: bool) -> "OracleFrame":
        """This (float) frame's splats sorted, binned and blended again (the stages after
        projection), with PortableMath or StdMath blending."""
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        rc = lib().oracle_rasterize_splats(self.h, int(portable), C.byref(h), err, 512)
        if rc != 0:
            raise OracleError(rc, err.value.decode())
        return OracleFrame(h)

    def backward(self, dl_dimage: np.ndarray, mutate_term: int = -1):
        g = np.ascontiguousarray(dl_dimage, dtype=np.float64).ravel()
        err = C.create_string_buffer(512)
        rc = lib().oracle_backward(self.h, _dp(g), mutate_term, err, 512)
        if rc != 0:
            raise OracleError(rc, err.value.decode())


def render(cloud, R, t, width, height, settings: OracleSettings = OracleSettings(), dbl=False, portable=False,
           brute=False, threads=0, sh_degree: int = 0, sh_rest=None) -> OracleFrame:
    """cloud = (means, rotations, log_scales, raw_opacities, colors); sh_rest (3*nb, n)
    for the SH extension (sh_degree 1..3)."""
    means, rot, ls, op, col = [np.ascontiguousarray(a, dtype=np.float64) for a in cloud[:5]]
    sh = np.ascontiguousarray(sh_rest if sh_rest is not None else np.zeros(1), dtype=np.float64)
    R = np.ascontiguousarray(R, dtype=np.float64).reshape(9)
    t = np.ascontiguousarray(t, dtype=np.float64).reshape(3)
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    rc = lib().oracle_render(int(dbl), int(portable), int(brute), op.shape[0], _dp(means), _dp(rot), _dp(ls),
                             _dp(op), _dp(col), _dp(R), _dp(t), width, height, _dp(settings.array()), threads,
                             sh_degree, _dp(sh), C.byref(h), err, 512)
    if rc != 0:
        raise OracleError(rc, err.value.decode())
    return OracleFrame(h)


# ------------------------------------------------------------------ densify (densify.hpp:81-166)
MOMENT_WIDTHS = (("means_m", 3), ("means_v", 3), ("rot_m", 4), ("rot_v", 4), ("scale_m", 3), ("scale_v", 3),
                 ("opac_m", 1), ("opac_v", 1), ("color_m", 3), ("color_v", 3))
PARAM_WIDTHS = (("means", 3), ("rotations", 4), ("log_scales", 3), ("raw_opacities", 1), ("colors", 3))


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _split(flat, widths, m):
    out, off = {}, 0
    for name, w in widths:
        seg = flat[off * m:(off + w) * m]
        out[name] = seg.reshape(w, m) if w > 1 else seg
        off += w
    return out


def densify(params: dict, moments: dict, grad_accum, elev_accum, grad_count, cfg, extent: float, seed: int,
            portable: bool = True):
    """densify_and_prune<float, Portable|Std>(cloud, state, cfg, extent, std::mt19937(seed)).

    params / moments: dicts of [w][n] arrays (see PARAM_WIDTHS / MOMENT_WIDTHS). cfg: (grad_threshold_min,
    grad_threshold_max, percent_dense, opacity_prune_floor, split_scale_divisor). Returns
    (params_out, moments_out, (cloned, split, pruned), next_draw)."""
    n = int(np.asarray(grad_count).shape[0])
    pf = np.concatenate([np.asarray(params[k], np.float64).reshape(-1) for k, _ in PARAM_WIDTHS])
    mf = np.concatenate([np.asarray(moments[k], np.float64).reshape(-1) for k, _ in MOMENT_WIDTHS])
    ga = np.ascontiguousarray(grad_accum, np.float64)
    ea = np.ascontiguousarray(elev_accum, np.float64)
    gc = np.ascontiguousarray(grad_count, np.int32)
    cf = np.asarray(cfg, np.float64)
    cap = 3 * n + 1
    po, mo = np.zeros(14 * cap), np.zeros(28 * cap)
    stats = np.zeros(4, np.int64)
    nd = C.c_uint32()
    err = C.create_string_buffer(256)
    rc = lib().oracle_densify(int(portable), n, _dp(pf), _dp(mf), _dp(ga), _dp(ea),
                              gc.ctypes.data_as(C.POINTER(C.c_int32)), _dp(cf), float(extent), seed, cap, _dp(po),
                              _dp(mo), stats.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(nd), err, 256)
    if rc:
        raise OracleError(rc, err.value.decode())
    m = int(stats[3])
    return (_split(po[:14 * m], PARAM_WIDTHS, m), _split(mo[:28 * m], MOMENT_WIDTHS, m),
            tuple(int(x) for x in stats[:3]), nd.value)


def reset_opacity(raw_opacities, ceiling: float = 0.01, portable: bool = True):
    """reset_opacity<float> on a copy of raw_opacities (float64 array of float values)."""
    raw = np.array(raw_opacities, np.float64)
    err = C.create_string_buffer(256)
    rc = lib().oracle_reset_opacity(int(portable), raw.shape[0], _dp(raw), float(ceiling), err, 256)
    if rc:
        raise OracleError(rc, err.value.decode())
    return raw


def unit_ball(seed: int, count: int):
    """(samples (count, 3) float32, next raw draw) of unit_ball_normal<float> from mt19937(seed)."""
    out = np.empty((count, 3), np.float32)
    nxt = lib().oracle_unit_ball(seed, count, out.ctypes.data_as(C.POINTER(C.c_float)))
    return out, int(nxt)


def dynamic_threshold(elevation: float, tmin: float = 2e-5, tmax: float = 1e-4):
    out = C.c_double()
    rc = lib().oracle_dynamic_threshold(elevation, tmin, tmax, C.byref(out))
    if rc:
        raise OracleError(rc, "dynamic_threshold: elevation outside [-pi/2, pi/2]")
    return out.value

"""Scene I/O mirror over the C ABI (reference proj/include/odgs/io.hpp, src/io.cpp).

    load_pointcloud(path) -> PointCloud                 io.cpp:203-223
    save_pointcloud(points, path, binary=True)          io.cpp:225-257
    init_from_points(ctx, points) -> GaussianCloud64    io.cpp:259-297 (GPU 3-NN)
    save_checkpoint(cloud, path)                        io.cpp:299-332
    load_checkpoint(path) -> GaussianCloud64            io.cpp:334-362

Arrays are binary64 in the reference's storage: positions / colours / means (3, n),
rotations (4, n), log-scales (3, n), raw opacities (n,). File errors raise
OdgsRuntimeError (std::runtime_error) with the reference's message; init_from_points
with no points raises InvalidArgument. `GaussianCloud64.to_float()` gives the float32
GaussianCloud the rasterizer consumes.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _capi as capi
from .rasterizer import GaussianCloud, InvalidArgument, OdgsRuntimeError

KSH0 = 0.28209479177387814  # io.hpp:14
CHECKPOINT_VERSION = 1      # io.hpp:19


@dataclass
class PointCloud:  # io.hpp:22-26
    positions: np.ndarray  # (3, n) float64
    colors: np.ndarray     # (3, n) float64


@dataclass
class GaussianCloud64:  # GaussianCloud<double> (types.hpp:53-143)
    means: np.ndarray
    rotations: np.ndarray
    log_scales: np.ndarray
    raw_opacities: np.ndarray
    colors: np.ndarray

    @property
    def n(self) -> int:
        return int(self.raw_opacities.shape[0])

    @staticmethod
    def empty(n: int) -> "GaussianCloud64":
        z = lambda *s: np.zeros(s, dtype=np.float64)
        return GaussianCloud64(z(3, n), z(4, n), z(3, n), z(n), z(3, n))

    def to_c(self) -> capi.Cloud64:
        return capi.Cloud64(self.n, *(a.ctypes.data for a in (self.means, self.rotations, self.log_scales,
                                                               self.raw_opacities, self.colors)))

    def to_float(self) -> GaussianCloud:
        return GaussianCloud.from_numpy(self.means, self.rotations, self.log_scales, self.raw_opacities, self.colors)


def _path(p) -> bytes:
    return os.fsencode(os.fspath(p))


def _check(lib, status: int):
    if status == capi.STATUS_OK:
        return
    buf = C.create_string_buffer(4096)
    lib.odgs_io_last_error(buf, 4096)
    raise (InvalidArgument if status == capi.STATUS_INVALID_ARGUMENT else OdgsRuntimeError)(buf.value.decode())


def _f64(a, rows: int) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(rows, -1) if rows > 1 else a.reshape(-1)


def vertex_count(path) -> int:
    lib = capi.load_library()
    n = C.c_int64(0)
    _check(lib, lib.odgs_ply_vertex_count(_path(path), C.byref(n)))
    return int(n.value)


def load_pointcloud(path) -> PointCloud:
    lib = capi.load_library()
    n = C.c_int64(0)
    st = lib.odgs_ply_vertex_count(_path(path), C.byref(n))
    if st != capi.STATUS_OK:
        _check(lib, st)
    m = max(int(n.value), 0)
    pos = np.zeros((3, m), np.float64)
    col = np.zeros((3, m), np.float64)
    _check(lib, lib.odgs_load_pointcloud(_path(path), m, pos.ctypes.data, col.ctypes.data))
    return PointCloud(pos, col)


def save_pointcloud(points: PointCloud, path, binary: bool = True) -> None:
    lib = capi.load_library()
    pos = _f64(points.positions, 3)
    col = _f64(points.colors, 3)
    _check(lib, lib.odgs_save_pointcloud(_path(path), pos.shape[1], pos.ctypes.data, col.ctypes.data,
                                         1 if binary else 0))


def save_checkpoint(cloud: GaussianCloud64, path) -> None:
    lib = capi.load_library()
    c = GaussianCloud64(_f64(cloud.means, 3), _f64(cloud.rotations, 4), _f64(cloud.log_scales, 3),
                        _f64(cloud.raw_opacities, 1), _f64(cloud.colors, 3))
    cc = c.to_c()
    _check(lib, lib.odgs_save_checkpoint(_path(path), C.byref(cc)))


def load_checkpoint(path) -> GaussianCloud64:
    lib = capi.load_library()
    n = C.c_int64(0)
    _check(lib, lib.odgs_ply_vertex_count(_path(path), C.byref(n)))
    out = GaussianCloud64.empty(max(int(n.value), 0))
    cc = out.to_c()
    _check(lib, lib.odgs_load_checkpoint(_path(path), C.byref(cc)))
    return out


def init_from_points(ctx, points: PointCloud, return_scale: bool = False):
    """GPU init_from_points (io.cpp:259-297). Host numpy in, host numpy out. With
    return_scale also returns the per-point mean neighbour distance (before the log)."""
    pos = _f64(points.positions, 3)
    col = _f64(points.colors, 3)
    n = pos.shape[1] if pos.ndim == 2 else 0
    out = GaussianCloud64.empty(n)
    scale = np.zeros(n, np.float64)
    cc = out.to_c()
    ctx.check(ctx.lib.odgs_init_from_points(ctx.handle, n, pos.ctypes.data if n else None,
                                            col.ctypes.data if n else None, capi.MEM_HOST, C.byref(cc),
                                            scale.ctypes.data if n else None))
    return (out, scale) if return_scale else out

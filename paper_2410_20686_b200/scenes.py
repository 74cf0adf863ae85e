"""Synthetic Gaussian scenes for the benchmark configurations (BASELINE.json configs).

The draws follow the reference's test generator scenes::random_cloud
(proj/tests/scenes.hpp:20-51): azimuth U[-pi, pi], elevation U[-e, e], depth
U[dmin, dmax], a random unit quaternion, per-axis scale r * U[smin, smax], opacity
U[omin, omax] stored as a logit, colour 0.05 + 0.9 U. They are vectorised with numpy's
PCG64 (not std::mt19937), so the clouds have the reference generator's distribution,
not its exact bits; parity tests use the oracle's own mt19937 generator instead.
Arrays are float32 in the reference's SoA layout: (3, n), (4, n), (3, n), (n,), (3, n).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .rasterizer import CameraPose, GaussianCloud


@dataclass
class CloudBounds:  # scenes.hpp:11-16
    depth_min: float = 0.5
    depth_max: float = 20.0
    max_elevation: float = 1.45
    opacity_min: float = 0.05
    opacity_max: float = 0.95
    scale_min: float = 0.005
    scale_max: float = 0.05


def random_cloud_arrays(seed: int, n: int, b: CloudBounds = CloudBounds(), phi=None, theta=None):
    rng = np.random.default_rng(seed)
    if phi is None:
        phi = (2 * rng.random(n) - 1) * math.pi
    if theta is None:
        theta = (2 * rng.random(n) - 1) * b.max_elevation
    r = b.depth_min + rng.random(n) * (b.depth_max - b.depth_min)
    means = np.stack([r * np.cos(theta) * np.sin(phi), -r * np.sin(theta), r * np.cos(theta) * np.cos(phi)])
    q = rng.standard_normal((4, n))
    q /= np.maximum(np.linalg.norm(q, axis=0), 1e-3)
    s = r[None, :] * (b.scale_min + rng.random((3, n)) * (b.scale_max - b.scale_min))
    alpha = b.opacity_min + rng.random(n) * (b.opacity_max - b.opacity_min)
    colors = 0.05 + 0.9 * rng.random((3, n))
    f = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    return f(means), f(q), f(np.log(s)), f(np.log(alpha / (1 - alpha))), f(colors)


def concat(*parts):
    return tuple(np.ascontiguousarray(np.concatenate([p[k] for p in parts], axis=-1)) for k in range(5))


def cloud_c1() -> GaussianCloud:
    """C1: 100K Gaussians, default bounds (the reference's own test workload, scaled up)."""
    return GaussianCloud(*random_cloud_arrays(77, 100_000))


def cloud_c2(n: int = 500_000) -> GaussianCloud:
    """C2: 500K Gaussians with SH degree 3 (bounds of test_backward.cpp:53-63's fd_cloud:
    depth [0.8, 10], |elevation| <= 75 deg, opacity [0.1, 0.7], scale r * U[0.001, 0.01];
    45 SH coefficients N(0, 0.05^2))."""
    arrs = random_cloud_arrays(2002, n, CloudBounds(0.8, 10.0, math.radians(75.0), 0.1, 0.7, 0.001, 0.01))
    sh = np.random.default_rng(2003).normal(0.0, 0.05, (15, 3, n)).astype(np.float32)
    return GaussianCloud(*arrs, sh_degree=3, sh_rest=sh)


def cloud_c3(n: int = 1_000_000) -> GaussianCloud:
    """C3: 50% uniform + 25% near the poles + 25% at the azimuth seam."""
    n_u, n_p = n // 2, n // 4
    n_s = n - n_u - n_p
    uni = random_cloud_arrays(3001, n_u, CloudBounds(scale_min=0.001, scale_max=0.01))
    rp = np.random.default_rng(30021)
    el = np.deg2rad(75 + rp.random(n_p) * 14.5) * np.where(rp.random(n_p) < 0.5, -1.0, 1.0)
    poles = random_cloud_arrays(3002, n_p, CloudBounds(scale_min=0.0005, scale_max=0.005), theta=el)
    rs = np.random.default_rng(30031)
    az = (math.pi - rs.random(n_s) * 0.05) * np.where(rs.random(n_s) < 0.5, -1.0, 1.0)
    seam = random_cloud_arrays(3003, n_s, CloudBounds(max_elevation=1.2, scale_min=0.001, scale_max=0.01), phi=az)
    return GaussianCloud(*concat(uni, poles, seam))


def cloud_c4(n: int = 3_000_000, seed: int = 4001) -> GaussianCloud:
    """C4: 3M Gaussians, default bounds, scale r * U[0.001, 0.01]."""
    return GaussianCloud(*random_cloud_arrays(seed, n, CloudBounds(scale_min=0.001, scale_max=0.01)))


def cloud_c5(n: int = 10_000_000) -> GaussianCloud:
    """C5: 10M Gaussians, default bounds, scale r * U[0.0005, 0.005]."""
    return GaussianCloud(*random_cloud_arrays(5001, n, CloudBounds(scale_min=0.0005, scale_max=0.005)))


def identity_camera(width: int, height: int) -> CameraPose:
    return CameraPose(width, height)


def yaw_camera(yaw: float, width: int, height: int, translation=(0.0, 0.0, 0.0)) -> CameraPose:
    """synth.hpp:41-49: camera at `translation` whose forward points at azimuth `yaw`."""
    c, s = math.cos(yaw), math.sin(yaw)
    rot = np.array([[c, 0, -s], [0, 1, 0], [s, 0, c]], dtype=np.float64)
    return CameraPose(width, height, rot, np.asarray(translation, dtype=np.float64))


def c4_views(width: int = 2048, height: int = 1024, n_views: int = 8):
    """The 8 C4 training views: yaw 2*pi*v/8, small translations."""
    views = []
    for v in range(n_views):
        a = 2 * math.pi * v / n_views
        t = (0.05 * math.cos(a), 0.02 * (v % 2), 0.05 * math.sin(a))
        views.append(yaw_camera(a, width, height, t))
    return views

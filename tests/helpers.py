"""Shared helpers for the parity tests: run the same seeded scene through the GPU
(C ABI) and the CPU oracle and collect every RenderOutput field."""
from __future__ import annotations

import math

import numpy as np

import oracle_lib
from paper_2410_20686_b200 import CameraPose, GaussianCloud, RenderSettings, render
from paper_2410_20686_b200 import _capi as capi

F32 = np.float32


def to_cloud32(arrs) -> GaussianCloud:
    return GaussianCloud.from_numpy(*[np.asarray(a, dtype=np.float32) for a in arrs])


def settings_pair(**kw):
    """The same knobs as (GPU RenderSettings, oracle settings)."""
    g = RenderSettings(**kw)
    o = oracle_lib.OracleSettings(near=g.near_radius, far=g.far_radius, tile=g.tile_size, alpha_clamp=g.alpha_clamp,
                                  floor=g.transmittance_floor, cutoff=g.cutoff_sigma, lowpass=g.lowpass_dilation,
                                  max_elevation=g.max_elevation)
    return g, o


def rot_yaw(a: float) -> np.ndarray:
    return np.array([[math.cos(a), 0, math.sin(a)], [0, 1, 0], [-math.sin(a), 0, math.cos(a)]])


def angle_axis(angle: float, axis) -> np.ndarray:
    axis = np.asarray(axis, dtype=np.float64)
    axis = axis / np.linalg.norm(axis)
    k = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + math.sin(angle) * k + (1 - math.cos(angle)) * (k @ k)


def gpu_fields(ctx, cloud: GaussianCloud, cam: CameraPose, settings: RenderSettings, keep_cov=True):
    fr = render(ctx, cloud, cam, settings, flags=capi.FRAME_KEEP_COV2D if keep_cov else 0)
    info = fr.info()
    out = {
        "image": fr.image, "transmittance": fr.transmittance, "walked": fr.walked,
        "tile_offsets": fr.tile_offsets, "tile_entries": fr.tile_entries,
        "inst_splat": fr.instance_splat, "inst_shift": fr.instance_shift,
        "splat_index": fr.splat_field(capi.FRAME_SPLAT_INDEX, dtype=np.int64),
        "splat_mean": fr.splat_field(capi.FRAME_SPLAT_MEAN, 2), "splat_inv": fr.splat_field(capi.FRAME_SPLAT_INV, 4),
        "splat_depth": fr.splat_field(capi.FRAME_SPLAT_DEPTH), "splat_radius": fr.splat_field(capi.FRAME_SPLAT_RADIUS),
        "splat_opacity": fr.splat_field(capi.FRAME_SPLAT_OPACITY),
        "splat_color": fr.splat_field(capi.FRAME_SPLAT_COLOR, 3),
        "splat_clamped": fr.splat_field(capi.FRAME_SPLAT_CLAMPED, dtype=np.int32),
        "n_splats": info.n_splats, "n_instances": info.n_instances, "n_entries": info.n_entries,
        "frame": fr,
    }
    if keep_cov:
        out["splat_cov2d"] = fr.splat_field(capi.FRAME_SPLAT_COV2D, 4)
    return out


def cam32(cam: CameraPose):
    """The camera exactly as the GPU sees it (float32), widened for the oracle."""
    r = np.asarray(cam.rotation, dtype=np.float32).astype(np.float64)
    t = np.asarray(cam.translation, dtype=np.float32).astype(np.float64)
    return r, t


def oracle_fields(cloud_arrs, cam: CameraPose, osettings, portable: bool, dbl: bool = False, brute=False):
    r, t = cam32(cam)
    fr = oracle_lib.render(cloud_arrs, r, t, cam.width, cam.height, osettings,
                           dbl=dbl, portable=portable, brute=brute)
    W, H = cam.width, cam.height
    out = {k: fr.get(k) for k in ["tile_offsets", "tile_entries", "inst_splat", "inst_shift", "splat_index",
                                  "splat_depth", "splat_radius", "splat_opacity", "splat_clamped", "stats"]}
    out["image"] = fr.get("image").reshape(3, W, H)
    out["transmittance"] = fr.get("transmittance").reshape(W, H)
    out["walked"] = fr.get("walked").reshape(W, H)
    out["splat_mean"] = fr.get("splat_mean").reshape(-1, 2)
    out["splat_inv"] = fr.get("splat_inv").reshape(-1, 4)
    out["splat_cov2d"] = fr.get("splat_cov2d").reshape(-1, 4)
    out["splat_color"] = fr.get("splat_color").reshape(-1, 3)
    if brute:
        out["brute"] = fr.get("brute").reshape(3, W, H)
    out["frame"] = fr
    return out


BIT_EXACT_FIELDS = ["splat_index", "splat_mean", "splat_inv", "splat_cov2d", "splat_depth", "splat_radius",
                    "splat_opacity", "splat_color", "splat_clamped", "inst_splat", "inst_shift", "tile_offsets",
                    "tile_entries", "walked", "transmittance", "image"]


def assert_bit_exact(g, o, fields=BIT_EXACT_FIELDS):
    for k in fields:
        a = np.asarray(g[k])
        b = np.asarray(o[k])
        if a.dtype.kind == "f":
            b = b.astype(np.float32)  # oracle float results travel widened to f64 (exact)
        assert a.shape == b.shape, f"{k}: shape {a.shape} vs {b.shape}"
        bad = np.flatnonzero(~(a.ravel() == b.ravel()))
        assert bad.size == 0, f"{k}: {bad.size} mismatches, first at {bad[:5]}: {a.ravel()[bad[:5]]} vs {b.ravel()[bad[:5]]}"

"""Adaptive density control over the C ABI (reference proj/include/odgs/densify.hpp).

Mirrors the reference's `DensifyConfig`, `dynamic_threshold`, `densify_and_prune` and
`reset_opacity` (same names, argument meaning, mutation-in-place and exceptions). The
work runs in libodgs_b200.so: a device classification + compaction (csrc/densify.cu);
the split offsets come from a library-owned std::mt19937 (`Rng`) replaying the
reference's draw sequence (densify.hpp:61-69) on the host.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _capi as capi
from .rasterizer import Context, GaussianCloud, InvalidArgument, DomainError

MOMENTS = (("means_m", 3), ("means_v", 3), ("rot_m", 4), ("rot_v", 4), ("scale_m", 3), ("scale_v", 3),
           ("opac_m", 1), ("opac_v", 1), ("color_m", 3), ("color_v", 3))
PARAMS = (("means", 3), ("rotations", 4), ("log_scales", 3), ("raw_opacities", 1), ("colors", 3))


@dataclass
class DensifyConfig:  # densify.hpp:16-33
    grad_threshold_min: float = 2e-5
    grad_threshold_max: float = 1e-4
    percent_dense: float = 1e-3
    densify_interval: int = 100
    densify_until: int = 100000
    opacity_prune_floor: float = 0.005
    opacity_reset_interval: int = 3000
    split_scale_divisor: float = 1.6

    def validate(self) -> None:
        if not (self.grad_threshold_min > 0) or not (self.grad_threshold_max >= self.grad_threshold_min):
            raise InvalidArgument("DensifyConfig: need 0 < grad_threshold_min <= grad_threshold_max")
        if not (self.percent_dense > 0) or not (self.percent_dense < 1):
            raise InvalidArgument("DensifyConfig: percent_dense outside (0, 1)")

    def to_c(self) -> capi.DensifyConfig:
        return capi.DensifyConfig(self.grad_threshold_min, self.grad_threshold_max, self.percent_dense,
                                  self.opacity_prune_floor, self.split_scale_divisor)


@dataclass
class DensifyStats:  # densify.hpp:51-55
    cloned: int = 0
    split: int = 0
    pruned: int = 0


def dynamic_threshold(elevation: float, cfg: DensifyConfig) -> float:
    """densify.hpp:39-49 (binary64)."""
    out = C.c_double()
    rc = capi.load_library().odgs_dynamic_threshold(float(elevation), C.byref(cfg.to_c()), C.byref(out))
    if rc == capi.STATUS_DOMAIN:
        raise DomainError("dynamic_threshold: elevation outside [-pi/2, pi/2]")
    if rc:
        raise InvalidArgument("dynamic_threshold: bad arguments")
    return out.value


class Rng:
    """std::mt19937(seed) held by the library — the generator the reference passes to
    densify_and_prune. Same seed, same draws."""

    def __init__(self, seed: int = 5489):
        self.lib = capi.load_library()
        self.handle = self.lib.odgs_rng_create(int(seed) & 0xFFFFFFFF)
        if not self.handle:
            raise MemoryError("odgs_rng_create")

    def next(self) -> int:
        return int(self.lib.odgs_rng_next(self.handle))

    def unit_ball(self, count: int) -> np.ndarray:
        """count samples of detail::unit_ball_normal<float> (densify.hpp:61-69), (count, 3)."""
        out = np.empty((max(int(count), 0), 3), dtype=np.float32)
        if count > 0:
            self.lib.odgs_rng_unit_ball(self.handle, int(count), out.ctypes.data_as(C.POINTER(C.c_float)))
        return out

    def close(self) -> None:
        if self.handle:
            self.lib.odgs_rng_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TrainState:
    """TrainState (types.hpp:257-325) as device tensors: Adam moments per group, the
    densify window (grad_accum, elev_accum, grad_count) and the iteration."""

    def __init__(self, n: int, device, iteration: int = 0):
        import torch
        z = lambda w: torch.zeros((w, n) if w > 1 else (n,), dtype=torch.float32, device=device)
        for name, w in MOMENTS:
            setattr(self, name, z(w))
        self.grad_accum = z(1)
        self.elev_accum = z(1)
        self.grad_count = torch.zeros(n, dtype=torch.int32, device=device)
        self.iteration = iteration

    @property
    def n(self) -> int:
        return int(self.grad_count.shape[0])

    def to_c(self) -> capi.TrainState:
        return capi.TrainState(*[getattr(self, k).data_ptr() for k, _ in MOMENTS],
                               self.grad_accum.data_ptr(), self.elev_accum.data_ptr(), self.grad_count.data_ptr())

    def reset_densify_stats(self) -> None:  # types.hpp:283-287
        self.grad_accum.zero_()
        self.elev_accum.zero_()
        self.grad_count.zero_()


def params_of(cloud: GaussianCloud) -> capi.Params:
    if not cloud.on_device:
        raise InvalidArgument("densify: the cloud must live on the device")
    for name, _ in PARAMS:
        a = getattr(cloud, name)
        if not (a.is_contiguous() and str(a.dtype) == "torch.float32"):
            raise InvalidArgument("cloud tensors must be contiguous float32")
    return capi.Params(cloud.n, *[getattr(cloud, k).data_ptr() for k, _ in PARAMS])


def densify_and_prune(ctx: Context, cloud: GaussianCloud, state: TrainState, cfg: DensifyConfig,
                      scene_extent: float, rng: Rng) -> DensifyStats:
    """densify.hpp:81-153: clones / splits / prunes on the device; `cloud` and `state`
    are replaced in place by the densified rows (new tensors), like the reference."""
    import torch
    if cloud.sh_degree > 0:
        raise InvalidArgument("densify_and_prune: SH clouds (extension) are not densified")
    cfg.validate()
    if not (scene_extent > 0):
        raise InvalidArgument("densify_and_prune: scene extent must be positive")
    p_in, s_in = params_of(cloud), state.to_c()
    stats = capi.DensifyStats()
    ctx.check(ctx.lib.odgs_densify_plan(ctx.handle, C.byref(p_in), C.byref(s_in), C.byref(cfg.to_c()),
                                        float(scene_extent), C.byref(stats)))
    m = int(stats.n_out)
    dev = cloud.means.device
    new = {name: torch.empty((w, m) if w > 1 else (m,), dtype=torch.float32, device=dev) for name, w in PARAMS}
    out_cloud = GaussianCloud(new["means"], new["rotations"], new["log_scales"], new["raw_opacities"],
                              new["colors"])
    out_state = TrainState.__new__(TrainState)
    for name, w in MOMENTS:
        setattr(out_state, name, torch.empty((w, m) if w > 1 else (m,), dtype=torch.float32, device=dev))
    out_state.grad_accum = torch.empty(m, dtype=torch.float32, device=dev)
    out_state.elev_accum = torch.empty(m, dtype=torch.float32, device=dev)
    out_state.grad_count = torch.empty(m, dtype=torch.int32, device=dev)
    out_state.iteration = state.iteration
    ball = rng.unit_ball(2 * int(stats.split))
    ball_ptr = ball.ctypes.data_as(C.POINTER(C.c_float)) if ball.size else None
    p_out, s_out = params_of(out_cloud) if m > 0 else capi.Params(0), out_state.to_c()
    ctx.wait_torch()  # the new tensors come from torch's allocator / stream
    ctx.check(ctx.lib.odgs_densify_apply(ctx.handle, C.byref(p_in), C.byref(s_in), ball_ptr, C.byref(p_out),
                                         C.byref(s_out)))
    # The old tensors are released below; the library stream must be done reading them
    # before torch's allocator can hand their memory out again (densify runs every
    # ~100 iterations, so one synchronisation is free).
    ctx.synchronize()
    for name, _ in PARAMS:
        setattr(cloud, name, getattr(out_cloud, name))
    for name, _ in MOMENTS:
        setattr(state, name, getattr(out_state, name))
    state.grad_accum, state.elev_accum, state.grad_count = (out_state.grad_accum, out_state.elev_accum,
                                                           out_state.grad_count)
    return DensifyStats(int(stats.cloned), int(stats.split), int(stats.pruned))


def reset_opacity(ctx: Context, cloud: GaussianCloud, state: Optional[TrainState], ceiling: float = 0.01) -> None:
    """densify.hpp:158-166, in place on the device."""
    p = params_of(cloud)
    s = state.to_c() if state is not None else None
    ctx.check(ctx.lib.odgs_reset_opacity(ctx.handle, C.byref(p), C.byref(s) if s is not None else None,
                                         float(ceiling)))

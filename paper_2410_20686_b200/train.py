"""View-sharded training step over the C ABI (BASELINE config 4).

The reference trains on one view per step (optimizer.hpp:99-156). Per-view gradients
add (GradBuffers::accumulate, backward.hpp:364-373; test_backward.cpp:536-556), so a
batch of views partitions across GPUs: each rank renders and back-propagates its views
into one flat gradient buffer, a single all-reduce (sum) exchanges it, and every rank
applies the identical Adam update — replicas stay bit-identical because the reduced
buffer is identical everywhere.

Layout of the flat gradient buffer (float32, 16 n): means 3n | rotations 4n |
log_scales 3n | raw_opacities n | colors 3n | pixel_grad_norm n | one_minus_cos n; the
int32 `observed` counts travel in a second buffer.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _capi as capi
from .densify import DensifyConfig, DensifyStats, Rng, TrainState, densify_and_prune, reset_opacity
from .rasterizer import (CUDA_STREAM_LEGACY, CameraPose, Context, GaussianCloud, GradBuffers, RenderOutput,
                         RenderSettings, backward, render)

FLAT_LAYOUT = (("means", 3), ("rotations", 4), ("log_scales", 3), ("raw_opacities", 1), ("colors", 3),
               ("pixel_grad_norm", 1), ("one_minus_cos", 1))
FLAT_WIDTH = sum(w for _, w in FLAT_LAYOUT)  # 16


@dataclass
class TrainConfig:  # optimizer.hpp:23-48 (defaults)
    iterations: int = 5000
    lr_means_init: float = 1.6e-4
    lr_means_final: float = 1.6e-6
    lr_rotation: float = 1e-3
    lr_scale: float = 5e-3
    lr_opacity: float = 0.05
    lr_color: float = 2.5e-3
    lambda_ssim: float = 0.2
    # Density control schedule (optimizer.hpp:144-153); None = off. Every rank runs
    # it on identical inputs with an identically seeded generator, so replicas stay
    # identical without any exchange.
    densify: Optional[DensifyConfig] = None
    seed: int = 0


def means_lr_at(iteration: int, cfg: TrainConfig) -> float:
    """optimizer.hpp:61-69, evaluated in float like Scalar = float."""
    f = np.float32
    lr0, lr1 = f(cfg.lr_means_init), f(cfg.lr_means_final)
    if cfg.iterations <= 1:
        return float(lr1)
    t = min(f(1), f(iteration) / f(cfg.iterations - 1))
    return float(lr0 * np.power(lr1 / lr0, f(t), dtype=np.float32))


def assign_views(n_views: int, rank: int, world: int) -> List[int]:
    """Views of this rank: v with v % world == rank (every view exactly once)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return list(range(rank, n_views, world))


def flat_views(flat, n: int) -> dict:
    """Splits a flat (16 n) buffer into the GradBuffers members (views, no copies)."""
    out, off = {}, 0
    for name, w in FLAT_LAYOUT:
        seg = flat[off * n:(off + w) * n]
        out[name] = seg.reshape(w, n) if w > 1 else seg
        off += w
    return out


def allreduce_grads(flat, observed, group=None):
    """Sum of the per-rank gradient buffers (the one exchange step of the path)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(observed, op=dist.ReduceOp.SUM, group=group)


class _Lane:
    """One context of the trainer's view pipeline: its stream, frame, upstream-gradient
    buffer and device-side loss sum."""

    def __init__(self, torch, ctx: Context, n_px: int, device):
        self.ctx = ctx
        h = ctx.stream
        if h in (0, CUDA_STREAM_LEGACY):  # the legacy default stream: torch's default stream
            self.stream = torch.cuda.default_stream(device)
        elif h == torch.cuda.current_stream(device).cuda_stream:
            self.stream = torch.cuda.current_stream(device)
        else:
            self.stream = torch.cuda.ExternalStream(h, device=device)
        self.frame = RenderOutput(ctx)
        self.dl = torch.empty(3 * n_px, dtype=torch.float32, device=device)
        self.loss_sum = torch.zeros(1, dtype=torch.float64, device=device)


class ViewShardedTrainer:
    """C4 training step: render + photometric loss (L1 + SSIM) + backward for this rank's views, gradient
    all-reduce, Adam. Everything stays on the device.

    pipeline=True (or a lane count): views alternate between two contexts (two streams), so
    view k + 1's render, loss and front end run while view k's backward does; the backward passes —
    the only steps that touch the shared gradient buffer — stay in view order (each waits
    on the previous one's event), so the accumulated gradients are bit-identical to the
    sequential loop's."""

    def __init__(self, ctx: Context, cloud: GaussianCloud, views: Sequence[CameraPose], targets, settings,
                 cfg: TrainConfig, extent: float, rank: int = 0, world: int = 1, group=None,
                 pipeline=True):
        import torch
        self.torch = torch
        self.ctx, self.cloud, self.views, self.targets = ctx, cloud, list(views), list(targets)
        self.settings, self.cfg, self.extent = settings, cfg, float(extent)
        self.rank, self.world, self.group = rank, world, group
        self.mine = assign_views(len(self.views), rank, world)
        self.state = TrainState(cloud.n, cloud.means.device)
        self.rng = Rng(cfg.seed)
        self.last_densify: Optional[DensifyStats] = None
        H, W = views[0].height, views[0].width
        dev = cloud.means.device
        self.lanes = [_Lane(torch, ctx, W * H, dev)]
        n_lanes = min(int(pipeline) if not isinstance(pipeline, bool) else (2 if pipeline else 1), len(self.mine))
        for _ in range(1, n_lanes):
            st = torch.cuda.Stream(device=dev)
            c = Context(ctx.device, stream=st.cuda_stream)
            c.set_async(True)
            ln = _Lane(torch, c, W * H, dev)
            ln.stream = st  # the lane's torch stream (kept alive with the lane)
            self.lanes.append(ln)
        self.frame, self.dl, self.loss_sum = self.lanes[0].frame, self.lanes[0].dl, self.lanes[0].loss_sum
        self.iteration = 0
        self._alloc_grads()

    @property
    def contexts(self) -> List[Context]:
        return [ln.ctx for ln in self.lanes]

    def _alloc_grads(self) -> None:
        torch = self.torch
        n, dev = self.cloud.n, self.cloud.means.device
        self.n = n
        self.flat = torch.zeros(FLAT_WIDTH * n, dtype=torch.float32, device=dev)
        self.observed = torch.zeros(n, dtype=torch.int32, device=dev)
        fv = flat_views(self.flat, n)
        self.grads = GradBuffers(fv["means"], fv["rotations"], fv["log_scales"], fv["raw_opacities"],
                                 fv["colors"], fv["pixel_grad_norm"], fv["one_minus_cos"], self.observed)

    def step(self, read_loss: bool = True) -> Optional[float]:
        """One training step; returns this rank's summed photometric loss over its views
        (one device-to-host read per step), or None with read_loss=False."""
        torch = self.torch
        ctx, lib = self.ctx, self.ctx.lib
        for attempt in range(3):
            self.flat.zero_()
            self.observed.zero_()
            for ln in self.lanes:
                ln.loss_sum.zero_()
            start = torch.cuda.Event()
            start.record()  # the zeroed buffers, on the caller's stream
            for ln in self.lanes:
                ln.stream.wait_event(start)
            prev_bwd = None
            for k, v in enumerate(self.mine):
                ln = self.lanes[k % len(self.lanes)]
                cam = self.views[v]
                # The lane's stream is torch's current stream here, so the wrappers'
                # stream-ordering calls are no-ops and only the events below order lanes.
                with torch.cuda.stream(ln.stream):
                    render(ln.ctx, self.cloud, cam, self.settings, out=ln.frame)
                    img = ln.frame.device_ptr(capi.FRAME_IMAGE)
                    # The loss stays on the device (added into the lane's loss sum).
                    ln.ctx.check(ln.ctx.lib.odgs_photometric_loss_async(
                        ln.ctx.handle, C_void(img), C_void(self.targets[v].data_ptr()), cam.width, cam.height,
                        self.cfg.lambda_ssim, C_void(ln.dl.data_ptr()), C_void(ln.loss_sum.data_ptr())))
                    if prev_bwd is not None:
                        ln.stream.wait_event(prev_bwd)  # gradient accumulation in view order
                    backward(ln.ctx, self.cloud, cam, ln.frame, ln.dl, self.settings, grads=self.grads,
                             accumulate=True)
                    prev_bwd = torch.cuda.Event()
                    prev_bwd.record(ln.stream)
            cur = torch.cuda.current_stream(self.cloud.means.device)
            for ln in self.lanes:
                cur.wait_stream(ln.stream)
            # Asynchronous contexts: one check point per step (deferred errors). An
            # entry-buffer overflow in any view invalidates the step's gradients: the
            # views run again, with buffers grown to the largest view's entries.
            rerun = False
            for ln in self.lanes:
                rerun = ln.frame.check() or rerun
            if not rerun:
                break
        for ln in self.lanes[1:]:
            self.loss_sum += ln.loss_sum
        allreduce_grads(self.flat, self.observed, self.group)
        ctx.wait_torch()  # Adam reads the reduced gradients
        step = self.iteration + 1
        p = capi.Params(self.n, self.cloud.means.data_ptr(), self.cloud.rotations.data_ptr(),
                        self.cloud.log_scales.data_ptr(), self.cloud.raw_opacities.data_ptr(),
                        self.cloud.colors.data_ptr())
        st = self.state.to_c()
        ap = capi.AdamParams(means_lr_at(self.iteration, self.cfg) * self.extent, self.cfg.lr_rotation,
                             self.cfg.lr_scale, self.cfg.lr_opacity, self.cfg.lr_color, step)
        g = self.grads.to_c()
        ctx.check(lib.odgs_adam_step(ctx.handle, byref(p), byref(g), byref(st), byref(ap)))
        self.iteration = step
        self.state.iteration = step
        self.last_densify = None
        d = self.cfg.densify
        if d is not None and step <= d.densify_until:  # optimizer.hpp:144-153
            if d.densify_interval > 0 and step % d.densify_interval == 0:
                self.last_densify = densify_and_prune(ctx, self.cloud, self.state, d, self.extent, self.rng)
                self._alloc_grads()
            if d.opacity_reset_interval > 0 and step % d.opacity_reset_interval == 0:
                reset_opacity(ctx, self.cloud, self.state)
        if not read_loss:
            return None
        ctx.torch_wait()
        return float(self.loss_sum.item())


# ctypes shorthands
import ctypes as _C  # noqa: E402

C_double = _C.c_double
C_void = _C.c_void_p
byref = _C.byref

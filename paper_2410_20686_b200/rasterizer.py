"""Python mirror of the reference rasterizer API over the C ABI.

Names, argument meaning and error behaviour follow the reference
(proj/include/odgs/{types,rasterizer,backward}.hpp):

    render(cloud, camera, settings)            rasterizer.hpp:211-214
    prepare_render(cloud, camera, settings)    rasterizer.hpp:129-132
    backward(cloud, camera, fwd, dl_dimage, settings, signs=None)   backward.hpp:380-386
    cull(cloud, camera, near, far)             rasterizer.hpp:15-18

Exceptions: InvalidArgument (std::invalid_argument), OdgsRuntimeError
(std::runtime_error), DomainError (std::domain_error); `.index` carries the
offending Gaussian row where the reference names one.

Arrays use the reference's storage: cloud members SoA with shape (3, n)/(4, n)/(n,)
(Eigen column-major MatX3 .data()), images (3, W, H) i.e. planar channels each
column-major (ErpImage storage). Host inputs are numpy float32; device inputs are
torch CUDA float32 tensors (no copies).
"""
from __future__ import annotations

import ctypes as C
import math
import weakref
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _capi as capi


class OdgsError(Exception):
    def __init__(self, message: str, index: int = -1):
        super().__init__(message)
        self.index = index


class InvalidArgument(OdgsError, ValueError):
    pass


class OdgsRuntimeError(OdgsError, RuntimeError):
    pass


class DomainError(OdgsError, ArithmeticError):
    pass


_EXC = {capi.STATUS_INVALID_ARGUMENT: InvalidArgument, capi.STATUS_RUNTIME: OdgsRuntimeError,
        capi.STATUS_DOMAIN: DomainError}


@dataclass
class RenderSettings:  # types.hpp:229-255
    near_radius: float = 0.01
    far_radius: float = 1000.0
    tile_size: int = 16
    alpha_clamp: float = 0.99
    transmittance_floor: float = 1e-4
    cutoff_sigma: float = 3.0
    lowpass_dilation: float = 0.3
    max_elevation: float = float(np.float32(85.0) * np.float32(math.pi) / np.float32(180.0))
    threads: int = 0

    def to_c(self) -> capi.Settings:
        return capi.Settings(self.near_radius, self.far_radius, self.tile_size, self.alpha_clamp,
                             self.transmittance_floor, self.cutoff_sigma, self.lowpass_dilation,
                             self.max_elevation, self.threads)


@dataclass
class CameraPose:  # types.hpp:148-180
    width: int
    height: int
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def to_c(self) -> capi.Camera:
        c = capi.Camera()
        r = np.asarray(self.rotation, dtype=np.float32).reshape(3, 3)
        t = np.asarray(self.translation, dtype=np.float32).reshape(3)
        for k in range(9):
            c.rotation[k] = float(r.flat[k])
        for k in range(3):
            c.translation[k] = float(t[k])
        c.width = int(self.width)
        c.height = int(self.height)
        return c


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


@dataclass
class GaussianCloud:  # types.hpp:53-143
    means: object          # (3, n)
    rotations: object      # (4, n)  (w, x, y, z), unnormalised
    log_scales: object     # (3, n)
    raw_opacities: object  # (n,)
    colors: object         # (3, n)
    sh_degree: int = 0     # extension: view-dependent colour (SH degree 1..3)
    sh_rest: object = None  # ((deg+1)^2 - 1, 3, n) non-DC coefficients

    @property
    def n(self) -> int:
        return int(self.raw_opacities.shape[0])

    @property
    def on_device(self) -> bool:
        return _is_torch(self.means) and self.means.is_cuda

    @staticmethod
    def from_numpy(means, rotations, log_scales, raw_opacities, colors, sh_degree=0, sh_rest=None) -> "GaussianCloud":
        f = lambda a: np.ascontiguousarray(a, dtype=np.float32)
        return GaussianCloud(f(means), f(rotations), f(log_scales), f(raw_opacities), f(colors), sh_degree,
                             None if sh_rest is None else f(sh_rest))

    def to_c(self) -> capi.Cloud:
        arrs = (self.means, self.rotations, self.log_scales, self.raw_opacities, self.colors)
        if self.sh_degree > 0:
            arrs = arrs + (self.sh_rest,)
        if self.on_device:
            for a in arrs:
                if not (a.is_contiguous() and str(a.dtype) == "torch.float32"):
                    raise InvalidArgument("cloud tensors must be contiguous float32")
            ptrs = [a.data_ptr() for a in arrs]
            mem = capi.MEM_DEVICE
        elif _is_torch(self.means):
            ptrs = [a.data_ptr() for a in arrs]
            mem = capi.MEM_HOST
        else:
            for a in arrs:
                if not (isinstance(a, np.ndarray) and a.dtype == np.float32 and a.flags.c_contiguous):
                    raise InvalidArgument("cloud arrays must be C-contiguous float32")
            ptrs = [a.ctypes.data for a in arrs]
            mem = capi.MEM_HOST
        sh_ptr = ptrs[5] if self.sh_degree > 0 else None
        return capi.Cloud(self.n, *ptrs[:5], mem, self.sh_degree, sh_ptr)


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy


class Context:
    """One CUDA device + stream (odgs_ctx). Not thread-safe; one per host thread."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        self.lib = capi.load_library()
        h = C.c_void_p()
        # stream: a cudaStream_t handle (e.g. torch.cuda.current_stream().cuda_stream); 0 is
        # the legacy default stream (passed as cudaStreamLegacy, since a NULL handle asks the
        # library for a private non-blocking stream). None: a private stream.
        if stream is None:
            handle = None
        else:
            handle = C.c_void_p(int(stream) if int(stream) != 0 else CUDA_STREAM_LEGACY)
        st = self.lib.odgs_ctx_create(device, handle, C.byref(h))
        if st != 0:
            raise OdgsError(f"odgs_ctx_create failed with status {st}")
        self.handle = h
        self.device = device
        self._frames = weakref.WeakSet()

    def close(self):
        if self.handle:
            for fr in list(self._frames):  # frames hold device memory of this context
                fr.destroy()
            self.lib.odgs_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, status: int):
        if status == capi.STATUS_OK:
            return
        idx = C.c_int64(-1)
        msg = C.create_string_buffer(512)
        self.lib.odgs_last_error(self.handle, C.byref(idx), msg, 512)
        raise _EXC.get(status, OdgsError)(msg.value.decode(), idx.value)

    def synchronize(self):
        self.check(self.lib.odgs_synchronize(self.handle))

    @property
    def launch_count(self) -> int:
        return int(self.lib.odgs_ctx_launch_count(self.handle))

    @property
    def stream(self) -> int:
        return int(self.lib.odgs_ctx_stream(self.handle) or 0)

    def _torch_streams(self):
        """(this context's stream, torch's current stream) as torch streams, or None when they
        are the same stream (or torch / CUDA is absent)."""
        import sys as _sys
        torch = _sys.modules.get("torch")
        if torch is None or not torch.cuda.is_available():
            return None
        cur = torch.cuda.current_stream(self.device)
        mine = self.stream
        if mine == cur.cuda_stream or (mine == CUDA_STREAM_LEGACY and cur.cuda_stream == 0):
            return None
        return torch.cuda.ExternalStream(mine, device=torch.device("cuda", self.device)), cur

    def wait_torch(self):
        """Orders this context's stream after the work already queued on torch's current stream
        (call before handing torch-produced device tensors to the library)."""
        ss = self._torch_streams()
        if ss:
            ss[0].wait_stream(ss[1])

    def torch_wait(self):
        """Orders torch's current stream after the work queued on this context's stream (call
        before torch reads device memory the library wrote)."""
        ss = self._torch_streams()
        if ss:
            ss[1].wait_stream(ss[0])

    def set_async(self, enable: bool = True):
        """odgs_ctx_set_async: renders and device-buffer backward passes return without
        synchronising; errors surface at RenderOutput.check() (or any host read)."""
        self.check(self.lib.odgs_ctx_set_async(self.handle, int(enable)))

    def set_profiling(self, enable: bool):
        self.check(self.lib.odgs_ctx_set_profiling(self.handle, int(enable)))

    def reset_stage_times(self):
        self.lib.odgs_ctx_reset_stage_times(self.handle)

    def stage_times(self) -> dict:
        """{stage: (milliseconds, calls)} accumulated on the context's stream."""
        ms = (C.c_double * 16)()
        calls = (C.c_int64 * 16)()
        n = self.lib.odgs_ctx_stage_times(self.handle, ms, calls, 16)
        return {self.lib.odgs_stage_name(k).decode(): (ms[k], calls[k]) for k in range(n)}

    def measure_fp32_tflops(self) -> float:
        v = C.c_double(0)
        self.check(self.lib.odgs_measure_fp32_tflops(self.handle, C.byref(v)))
        return v.value


class RenderOutput:
    """A rendered frame (RenderOutput, rasterizer.hpp:92-102); fields download on access."""

    def __init__(self, ctx: Context, flags: int = 0):
        self.ctx = ctx
        h = C.c_void_p()
        ctx.check(ctx.lib.odgs_frame_create(ctx.handle, C.byref(h)))
        self.handle = h
        ctx._frames.add(self)
        if flags:
            ctx.lib.odgs_frame_set_flags(h, flags)

    def destroy(self):
        if self.handle and self.ctx.handle:
            self.ctx.lib.odgs_frame_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def info(self) -> capi.FrameInfo:
        i = capi.FrameInfo()
        self.ctx.check(self.ctx.lib.odgs_frame_get_info(self.handle, C.byref(i)))
        return i

    def check(self) -> bool:
        """The frame's check point (odgs_frame_check): raises the deferred error of
        asynchronous work; True if the frame had to be re-rendered (an entry-buffer
        overflow), in which case a backward enqueued on it must be repeated."""
        rr = C.c_int32(0)
        self.ctx.check(self.ctx.lib.odgs_frame_check(self.ctx.handle, self.handle, C.byref(rr)))
        return bool(rr.value)

    def _download(self, fld: int, dtype, shape) -> np.ndarray:
        out = np.empty(shape, dtype=dtype)
        self.ctx.check(self.ctx.lib.odgs_frame_download(self.ctx.handle, self.handle, fld,
                                                        out.ctypes.data, out.nbytes))
        return out

    def work(self):
        """(entries examined, entries composited) of the last blend."""
        a, b = C.c_int64(0), C.c_int64(0)
        self.ctx.check(self.ctx.lib.odgs_frame_work(self.ctx.handle, self.handle, C.byref(a), C.byref(b)))
        return a.value, b.value

    def backward_work(self):
        """(entries replayed, contributions, warp-entries walked, warp-entries with a
        contribution) of the last backward on this frame."""
        out = (C.c_int64 * 4)()
        self.ctx.check(self.ctx.lib.odgs_frame_backward_work(self.ctx.handle, self.handle, out, 4))
        return tuple(int(v) for v in out)

    def set_image_peers(self, ptrs) -> None:
        """odgs_frame_set_image_peers: the blend also writes each rendered pixel into
        these [3][W][H] float device buffers (fused band all-gather)."""
        arr = (C.c_void_p * max(len(ptrs), 1))(*[C.c_void_p(int(p)) for p in ptrs])
        st = self.ctx.lib.odgs_frame_set_image_peers(self.handle, len(ptrs), arr)
        if st != capi.STATUS_OK:
            raise InvalidArgument(f"odgs_frame_set_image_peers failed ({st})")

    def device_ptr(self, fld: int) -> int:
        p = C.c_void_p()
        self.ctx.check(self.ctx.lib.odgs_frame_device_ptr(self.handle, fld, C.byref(p)))
        return int(p.value)

    @property
    def image(self) -> np.ndarray:  # (3, W, H)
        i = self.info()
        return self._download(capi.FRAME_IMAGE, np.float32, (3, i.width, i.height))

    @property
    def transmittance(self) -> np.ndarray:  # (W, H)
        i = self.info()
        return self._download(capi.FRAME_TRANSMITTANCE, np.float32, (i.width, i.height))

    @property
    def walked(self) -> np.ndarray:  # (W, H)
        i = self.info()
        return self._download(capi.FRAME_WALKED, np.int32, (i.width, i.height))

    @property
    def tile_offsets(self) -> np.ndarray:
        i = self.info()
        return self._download(capi.FRAME_TILE_OFFSETS, np.int32, (i.tiles_x * i.tiles_y + 1,))

    @property
    def tile_entries(self) -> np.ndarray:
        return self._download(capi.FRAME_TILE_ENTRIES, np.int32, (self.info().n_entries,))

    @property
    def instance_splat(self) -> np.ndarray:
        return self._download(capi.FRAME_INSTANCE_SPLAT, np.int32, (self.info().n_instances,))

    @property
    def instance_shift(self) -> np.ndarray:
        return self._download(capi.FRAME_INSTANCE_SHIFT, np.float32, (self.info().n_instances,))

    def splat_field(self, fld: int, width: int = 1, dtype=np.float32) -> np.ndarray:
        ns = self.info().n_splats
        shape = (ns,) if width == 1 else (ns, width)
        return self._download(fld, dtype, shape)


@dataclass
class GradBuffers:  # backward.hpp:342-374
    means: np.ndarray
    rotations: np.ndarray
    log_scales: np.ndarray
    raw_opacities: np.ndarray
    colors: np.ndarray
    pixel_grad_norm: np.ndarray
    one_minus_cos: np.ndarray
    observed: np.ndarray
    sh_rest: object = None  # SH extension: gradients of the non-DC coefficients

    @staticmethod
    def zeros(n: int, sh_degree: int = 0) -> "GradBuffers":
        z = lambda *s: np.zeros(s, np.float32)
        nb = (sh_degree + 1) ** 2 - 1
        return GradBuffers(z(3, n), z(4, n), z(3, n), z(n), z(3, n), z(n), z(n), np.zeros(n, np.int32),
                           z(nb, 3, n) if sh_degree > 0 else None)

    def to_c(self) -> capi.Grads:
        arrs = (self.means, self.rotations, self.log_scales, self.raw_opacities, self.colors,
                self.pixel_grad_norm, self.one_minus_cos, self.observed)
        if _is_torch(self.means) and self.means.is_cuda:
            sh = self.sh_rest.data_ptr() if self.sh_rest is not None else None
            return capi.Grads(*[a.data_ptr() for a in arrs], capi.MEM_DEVICE, sh)
        sh = self.sh_rest.ctypes.data if self.sh_rest is not None else None
        return capi.Grads(*[a.ctypes.data for a in arrs], capi.MEM_HOST, sh)


def prepare_render(ctx: Context, cloud: GaussianCloud, camera: CameraPose, settings: RenderSettings,
                   out: Optional[RenderOutput] = None, flags: int = 0) -> RenderOutput:
    out = out or RenderOutput(ctx, flags)
    if cloud.on_device:
        ctx.wait_torch()
    cc, cam, st = cloud.to_c(), camera.to_c(), settings.to_c()
    ctx.check(ctx.lib.odgs_prepare_render(ctx.handle, C.byref(cc), C.byref(cam), C.byref(st), out.handle))
    return out


def render(ctx: Context, cloud: GaussianCloud, camera: CameraPose, settings: RenderSettings,
           out: Optional[RenderOutput] = None, flags: int = 0) -> RenderOutput:
    out = out or RenderOutput(ctx, flags)
    if cloud.on_device:
        ctx.wait_torch()
    cc, cam, st = cloud.to_c(), camera.to_c(), settings.to_c()
    ctx.check(ctx.lib.odgs_render(ctx.handle, C.byref(cc), C.byref(cam), C.byref(st), out.handle))
    return out


def rasterize_splats(ctx: Context, n_gaussians: int, index, pixel_mean, cov2d_inv, depth, radius, opacity, color,
                     width: int, height: int, settings: RenderSettings,
                     out: Optional[RenderOutput] = None, flags: int = 0) -> RenderOutput:
    """The rasterization half of render() (rasterizer.hpp:141-267) on given projected
    splats (RenderOutput::splats rows, ascending cloud index): seam instances, global
    order, tile CSR and blend. Arrays: index (ns,), pixel_mean (ns, 2), cov2d_inv (ns, 4)
    row-major, depth / radius / opacity (ns,), color (ns, 3)."""
    out = out or RenderOutput(ctx, flags)
    idx = np.ascontiguousarray(index, dtype=np.int64)
    f = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    arrs = [f(pixel_mean), f(cov2d_inv), f(depth), f(radius), f(opacity), f(color)]
    st = settings.to_c()
    ctx.check(ctx.lib.odgs_rasterize_splats(ctx.handle, int(n_gaussians), idx.shape[0], idx.ctypes.data,
                                            *[a.ctypes.data for a in arrs], width, height, C.byref(st), out.handle))
    return out


def render_band(ctx: Context, cloud: GaussianCloud, camera: CameraPose, settings: RenderSettings, row_begin: int,
                row_end: int, out: Optional[RenderOutput] = None, flags: int = 0) -> RenderOutput:
    """Rows [row_begin, row_end) of render(); bit-identical to the full render there."""
    out = out or RenderOutput(ctx, flags)
    if cloud.on_device:
        ctx.wait_torch()
    cc, cam, st = cloud.to_c(), camera.to_c(), settings.to_c()
    ctx.check(ctx.lib.odgs_render_band(ctx.handle, C.byref(cc), C.byref(cam), C.byref(st), row_begin, row_end,
                                       out.handle))
    return out


def backward(ctx: Context, cloud: GaussianCloud, camera: CameraPose, fwd: RenderOutput, dl_dimage,
             settings: RenderSettings, signs=None, grads: Optional[GradBuffers] = None,
             accumulate: bool = False) -> GradBuffers:
    grads = grads or GradBuffers.zeros(cloud.n, cloud.sh_degree)
    if (cloud.on_device or (_is_torch(dl_dimage) and dl_dimage.is_cuda)
            or (_is_torch(grads.means) and grads.means.is_cuda)):
        ctx.wait_torch()  # torch-produced inputs or torch-zeroed gradient buffers
    cc, cam, st, gc = cloud.to_c(), camera.to_c(), settings.to_c(), grads.to_c()
    if _is_torch(dl_dimage):
        dptr, dmem = dl_dimage.data_ptr(), (capi.MEM_DEVICE if dl_dimage.is_cuda else capi.MEM_HOST)
    else:
        dl_dimage = np.ascontiguousarray(dl_dimage, dtype=np.float32)
        dptr, dmem = dl_dimage.ctypes.data, capi.MEM_HOST
    sp = None
    if signs is not None:
        sp = (C.c_double * 12)(*[float(s) for s in signs])
    ctx.check(ctx.lib.odgs_backward(ctx.handle, C.byref(cc), C.byref(cam), fwd.handle, C.c_void_p(dptr), dmem,
                                    C.byref(st), C.byref(gc), sp, capi.ACCUMULATE if accumulate else 0))
    if _is_torch(grads.means) and grads.means.is_cuda:
        ctx.torch_wait()  # torch may read the gradients next
    return grads


@dataclass
class Splat2D:  # projection.hpp:163-174
    pixel_mean: np.ndarray
    cov2d: np.ndarray
    cov2d_inv: np.ndarray
    depth: float
    radius: float
    opacity: float
    color: np.ndarray
    index: int
    pole_clamped: bool


def project_gaussian(ctx: Context, cloud: GaussianCloud, i: int, camera: CameraPose,
                     settings: RenderSettings) -> Optional[Splat2D]:
    """projection.hpp:178-216: the splat of cloud row i, or None (std::nullopt)."""
    if cloud.on_device:
        ctx.wait_torch()
    cc, cam, st = cloud.to_c(), camera.to_c(), settings.to_c()
    out, projected = capi.Splat(), C.c_int32(0)
    ctx.check(ctx.lib.odgs_project_gaussian(ctx.handle, C.byref(cc), int(i), C.byref(cam), C.byref(st),
                                            C.byref(out), C.byref(projected)))
    if not projected.value:
        return None
    f = lambda a: np.array(a[:], dtype=np.float32)
    return Splat2D(f(out.pixel_mean), f(out.cov2d).reshape(2, 2), f(out.cov2d_inv).reshape(2, 2),
                   np.float32(out.depth), np.float32(out.radius), np.float32(out.opacity), f(out.color),
                   int(out.index), bool(out.pole_clamped))


@dataclass
class SplatGrads:  # backward.hpp:19-25, one row per splat of the frame
    pixel_mean: np.ndarray  # (ns, 2)
    cov2d: np.ndarray       # (ns, 2, 2), full-matrix convention
    opacity: np.ndarray     # (ns,), w.r.t. the activated opacity
    color: np.ndarray       # (ns, 3)


def grad_pixels_to_splats(ctx: Context, fwd: RenderOutput, dl_dimage, settings: RenderSettings) -> SplatGrads:
    """backward.hpp:208-339: per-splat gradients of a rendered frame (fwd) for the image
    gradient dl_dimage (3, W, H)."""
    ns = fwd.info().n_splats
    out = SplatGrads(np.zeros((ns, 2), np.float32), np.zeros((ns, 2, 2), np.float32), np.zeros(ns, np.float32),
                     np.zeros((ns, 3), np.float32))
    if _is_torch(dl_dimage):
        if dl_dimage.is_cuda:
            ctx.wait_torch()
        dptr, dmem = dl_dimage.data_ptr(), (capi.MEM_DEVICE if dl_dimage.is_cuda else capi.MEM_HOST)
    else:
        dl_dimage = np.ascontiguousarray(dl_dimage, dtype=np.float32)
        dptr, dmem = dl_dimage.ctypes.data, capi.MEM_HOST
    st = settings.to_c()
    ctx.check(ctx.lib.odgs_grad_pixels_to_splats(ctx.handle, fwd.handle, C.c_void_p(dptr), dmem, C.byref(st),
                                                 out.pixel_mean.ctypes.data, out.cov2d.ctypes.data,
                                                 out.opacity.ctypes.data, out.color.ctypes.data))
    return out


def cull(ctx: Context, cloud: GaussianCloud, camera: CameraPose, near: float, far: float) -> np.ndarray:
    out = np.empty(max(cloud.n, 1), np.int64)
    count = C.c_int64(0)
    cc, cam = cloud.to_c(), camera.to_c()
    ctx.check(ctx.lib.odgs_cull(ctx.handle, C.byref(cc), C.byref(cam), near, far,
                                out.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(count)))
    return out[: count.value].copy()

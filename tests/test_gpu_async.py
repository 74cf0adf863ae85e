"""Asynchronous rendering (odgs_ctx_set_async): no host synchronisation inside or between
renders and backward passes; tile-entry counts stay on the device, capacity-sized
buffers; errors and entry-buffer overflows surface at the frame's check point.
Results must equal the synchronous path bit for bit."""
import numpy as np
import pytest
import torch

import oracle_lib
from helpers import to_cloud32
from paper_2410_20686_b200 import (CameraPose, Context, GaussianCloud, GradBuffers, OdgsRuntimeError, RenderOutput,
                                   RenderSettings, backward, render, render_band, scenes)

pytestmark = pytest.mark.gpu


def dev_cloud(c):
    return GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(getattr(c, k))).cuda()
                           for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")])


def fields(fr):
    return fr.image, fr.transmittance, fr.walked, fr.tile_offsets, fr.tile_entries


def test_async_renders_equal_sync(gpu_ctx):
    c = dev_cloud(scenes.cloud_c3(200_000))
    s = RenderSettings()
    actx = Context(0)
    actx.set_async(True)
    fr = RenderOutput(actx)
    for k in range(6):  # the first render sizes the buffers (exact path), the rest are asynchronous
        cam = scenes.yaw_camera(0.37 * k, 1024, 512)
        render(actx, c, cam, s, out=fr)
        got = fields(fr)
        ref = fields(render(gpu_ctx, c, cam, s))
        for a, b in zip(got, ref):
            assert np.array_equal(a, b), k
    actx.close()


def test_async_queue_of_frames(gpu_ctx):
    """Several frames queued on one asynchronous context before any check."""
    c = dev_cloud(scenes.cloud_c3(100_000))
    s = RenderSettings()
    actx = Context(0)
    actx.set_async(True)
    frames = [RenderOutput(actx) for _ in range(3)]
    cams = [scenes.yaw_camera(1.1 * k, 512, 256) for k in range(3)]
    for fr, cam in zip(frames, cams):
        render(actx, c, cam, s, out=fr)   # sizing render (exact path)
    for fr, cam in zip(frames, reversed(cams)):
        render(actx, c, cam, s, out=fr)   # asynchronous
    for fr, cam in zip(frames, reversed(cams)):
        assert not fr.check()
        assert np.array_equal(fr.image, render(gpu_ctx, c, cam, s).image)
    actx.close()


def test_async_overflow_rerenders(gpu_ctx):
    """A frame sized on a sparse view, then asked for a view with many more entries: the
    check re-renders it with room for every entry and reports it."""
    n = 60_000
    base = scenes.cloud_c3(n)
    arrs = [np.array(getattr(base, k)) for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")]
    small = [a.copy() for a in arrs]
    small[2] = small[2] - 3.0  # scales / 20: few tiles per splat
    s = RenderSettings()
    cam = CameraPose(1024, 512)
    actx = Context(0)
    actx.set_async(True)
    fr = RenderOutput(actx)
    render(actx, dev_cloud(GaussianCloud(*small)), cam, s, out=fr)
    k_small = fr.info().n_entries
    big = dev_cloud(GaussianCloud(*arrs))
    render(actx, big, cam, s, out=fr)
    assert fr.check()  # re-rendered
    ref = render(gpu_ctx, big, cam, s)
    assert fr.info().n_entries == ref.info().n_entries > 2 * k_small
    for a, b in zip(fields(fr), fields(ref)):
        assert np.array_equal(a, b)
    render(actx, big, cam, s, out=fr)  # now it fits
    assert not fr.check()
    actx.close()


def test_async_errors_at_the_check_point(gpu_ctx):
    arrs = [np.array(a, dtype=np.float32) for a in oracle_lib.random_cloud(950, 3000)]
    good = to_cloud32([a.copy() for a in arrs])
    arrs[3][1777] = np.nan
    bad = to_cloud32(arrs)
    cam, s = CameraPose(256, 128), RenderSettings()
    actx = Context(0)
    actx.set_async(True)
    fr = RenderOutput(actx)
    render(actx, good, cam, s, out=fr)
    fr.check()
    render(actx, bad, cam, s, out=fr)       # returns: the error is deferred
    render(actx, good, cam, s, out=fr)      # the error survives a later render of the frame
    with pytest.raises(OdgsRuntimeError) as e:
        fr.check()
    assert e.value.index == 1777
    render(actx, good, cam, s, out=fr)      # checked: the frame is usable again
    assert not fr.check()
    assert np.array_equal(fr.image, render(gpu_ctx, good, cam, s).image)
    actx.close()


def test_async_backward_and_bands_equal_sync(gpu_ctx):
    c = dev_cloud(scenes.cloud_c3(100_000))
    s = RenderSettings()
    cam = scenes.yaw_camera(0.8, 1024, 512)
    dl = torch.from_numpy(np.random.default_rng(4).uniform(-1, 1, (3, 1024, 512)).astype(np.float32)).cuda()
    n = c.n
    z = lambda *sh: torch.zeros(sh, dtype=torch.float32, device="cuda")
    mk = lambda: GradBuffers(z(3, n), z(4, n), z(3, n), z(n), z(3, n), z(n), z(n),
                             torch.zeros(n, dtype=torch.int32, device="cuda"))
    ref = backward(gpu_ctx, c, cam, render(gpu_ctx, c, cam, s), dl, s, grads=mk())
    actx = Context(0)
    actx.set_async(True)
    fr = RenderOutput(actx)
    got = mk()
    for k in range(3):
        render(actx, c, cam, s, out=fr)
        backward(actx, c, cam, fr, dl, s, grads=got)
    fr.check()
    torch.cuda.synchronize()
    for k in ("means", "rotations", "log_scales", "raw_opacities", "colors", "observed"):
        assert torch.equal(getattr(got, k), getattr(ref, k)), k
    full = render(gpu_ctx, c, cam, s).image
    bf = RenderOutput(actx)
    for it in range(2):
        for r0 in range(0, 512, 128):
            render_band(actx, c, cam, s, r0, r0 + 128, out=bf)
            assert np.array_equal(bf.image[:, :, r0:r0 + 128], full[:, :, r0:r0 + 128]), (it, r0)
    actx.close()


def test_async_backward_on_overflowed_frame_is_memory_safe(gpu_ctx):
    """A backward enqueued on a frame whose render overflowed its entry buffers (before the
    check point) must stay inside the buffers: the fold clamps its record ranges to the
    entries actually sorted. After the check re-renders the frame, the backward equals the
    synchronous one bit for bit."""
    n = 60_000
    base = scenes.cloud_c3(n)
    arrs = [np.array(getattr(base, k)) for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")]
    small = [a.copy() for a in arrs]
    small[2] = small[2] - 3.0
    s = RenderSettings()
    cam = CameraPose(1024, 512)
    actx = Context(0)
    actx.set_async(True)
    fr = RenderOutput(actx)
    render(actx, dev_cloud(GaussianCloud(*small)), cam, s, out=fr)
    big = dev_cloud(GaussianCloud(*arrs))
    dl = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, 3 * 1024 * 512).astype(np.float32)).cuda()
    z = lambda *sh: torch.zeros(sh, dtype=torch.float32, device="cuda")
    g = GradBuffers(z(3, n), z(4, n), z(3, n), z(n), z(3, n), z(n), z(n), torch.zeros(n, dtype=torch.int32,
                                                                                      device="cuda"))
    render(actx, big, cam, s, out=fr)
    backward(actx, big, cam, fr, dl, s, grads=g)  # on the overflowed frame
    assert fr.check()  # re-rendered
    backward(actx, big, cam, fr, dl, s, grads=g)
    torch.cuda.synchronize()
    ref = backward(gpu_ctx, big, cam, render(gpu_ctx, big, cam, s), dl, s)
    for k in ("means", "rotations", "log_scales", "raw_opacities", "colors", "observed"):
        assert np.array_equal(getattr(g, k).cpu().numpy(), getattr(ref, k)), k
    actx.close()


def test_async_random_sequence_equals_sync(gpu_ctx):
    """A random sequence of clouds (sizes 0 to 40K, log-scales shifted by -3 to +1.5, so the
    entry count jumps up and down past the frame's capacity) rendered and back-propagated
    on one asynchronous frame, checked after every step against the synchronous path."""
    rng = np.random.default_rng(42)
    base = scenes.cloud_c3(40_000)
    arrs = [np.array(getattr(base, k)) for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")]
    s = RenderSettings()
    actx = Context(0)
    actx.set_async(True)
    fr = RenderOutput(actx)
    W, H = 512, 256
    for step in range(10):
        n = int(rng.choice([0, 1, 37, 5000, 40_000]))
        sub = [a[..., :n].copy() for a in arrs]
        sub[2] = sub[2] + float(rng.uniform(-3.0, 1.5))
        cloud = dev_cloud(GaussianCloud(*sub))
        cam = scenes.yaw_camera(float(rng.uniform(0, 6.28)), W, H)
        render(actx, cloud, cam, s, out=fr)
        dl = torch.from_numpy(rng.uniform(-1, 1, 3 * W * H).astype(np.float32)).cuda()
        z = lambda *sh: torch.zeros(sh, dtype=torch.float32, device="cuda")
        g = GradBuffers(z(3, n), z(4, n), z(3, n), z(n), z(3, n), z(n), z(n),
                        torch.zeros(n, dtype=torch.int32, device="cuda"))
        backward(actx, cloud, cam, fr, dl, s, grads=g)
        if fr.check():  # re-rendered: the backward ran on the overflowed frame; repeat it
            g = GradBuffers(z(3, n), z(4, n), z(3, n), z(n), z(3, n), z(n), z(n),
                            torch.zeros(n, dtype=torch.int32, device="cuda"))
            backward(actx, cloud, cam, fr, dl, s, grads=g)
        torch.cuda.synchronize()
        ref_fr = render(gpu_ctx, cloud, cam, s)
        for a, b in zip(fields(fr), fields(ref_fr)):
            assert np.array_equal(a, b), step
        if n:
            ref = backward(gpu_ctx, cloud, cam, ref_fr, dl, s)
            for k in ("means", "colors", "observed"):
                assert np.array_equal(getattr(g, k).cpu().numpy(), getattr(ref, k)), (step, k)
    actx.close()

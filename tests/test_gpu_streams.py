"""Stream ordering between the library and torch (bench.py and the trainer mix both).

* torch's default stream handle is 0; a context created with it must run on that same
  (legacy) stream, not on a private one — the bench's CUDA events and L2 flush rely on
  it (profiles/r01_kernels_v13.md).
* a context on a private stream orders itself after torch work on device inputs
  (Context.wait_torch in render / backward) and torch after the library's device
  gradients (Context.torch_wait).
"""
import numpy as np
import pytest

import oracle_lib
from paper_2410_20686_b200 import CameraPose, Context, GaussianCloud, GradBuffers, RenderSettings, backward, render
from paper_2410_20686_b200.rasterizer import CUDA_STREAM_LEGACY

pytestmark = pytest.mark.gpu


def _device_cloud(torch, seed=91, n=3000):
    arrs = oracle_lib.random_cloud(seed, n)
    return GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda() for a in arrs])


def test_default_stream_handle_is_the_legacy_stream():
    torch = pytest.importorskip("torch")
    cur = torch.cuda.current_stream().cuda_stream
    ctx = Context(0, stream=cur)
    try:
        if cur == 0:
            assert ctx.stream == CUDA_STREAM_LEGACY
        else:
            assert ctx.stream == cur
        own = Context(0)
        try:
            assert own.stream not in (0, CUDA_STREAM_LEGACY, cur)
        finally:
            own.close()
    finally:
        ctx.close()


def test_private_stream_waits_for_torch_inputs():
    torch = pytest.importorskip("torch")
    cloud = _device_cloud(torch)
    cam, s = CameraPose(256, 128), RenderSettings()
    ctx = Context(0)  # private non-blocking stream
    try:
        ref = render(ctx, cloud, cam, s).image.copy()
        assert np.abs(ref).max() > 0
        # A long GPU spin on torch's stream, then zero the colours there: the render must
        # see the zeros (it is ordered after torch's queued work), i.e. a black image.
        torch.cuda._sleep(20_000_000)
        cloud.colors.zero_()
        img = render(ctx, cloud, cam, s).image
        assert np.array_equal(img, np.zeros_like(img))
    finally:
        ctx.close()


def test_torch_reads_gradients_after_the_library():
    torch = pytest.importorskip("torch")
    cloud = _device_cloud(torch, seed=92)
    cam, s = CameraPose(256, 128), RenderSettings()
    ctx = Context(0)
    try:
        fr = render(ctx, cloud, cam, s)
        dl = torch.full((3 * 256 * 128,), 1e-3, dtype=torch.float32, device="cuda")
        n = cloud.n
        z = lambda *shape: torch.zeros(shape, dtype=torch.float32, device="cuda")
        grads = GradBuffers(z(3, n), z(4, n), z(3, n), z(n), z(3, n), z(n), z(n),
                            torch.zeros(n, dtype=torch.int32, device="cuda"))
        backward(ctx, cloud, cam, fr, dl, s, grads=grads)
        early = grads.colors.abs().sum().item()  # torch's stream, right after the call
        ctx.synchronize()
        late = grads.colors.abs().sum().item()
        assert late > 0 and early == late
    finally:
        ctx.close()


def test_concurrent_contexts_match_serial_renders():
    """The e2e path of bench.py: several contexts (own streams, programmatic dependent
    launches) rendering concurrently from host threads with a host-resident cloud give
    the same images as one context rendering the same cameras one after another."""
    import threading

    from paper_2410_20686_b200 import RenderOutput, scenes
    arrs = oracle_lib.random_cloud(95, 20000)
    cloud = GaussianCloud.from_numpy(*arrs)
    s = RenderSettings()
    cams = [scenes.yaw_camera(0.4 * k, 512, 256) for k in range(8)]
    serial = Context(0)
    try:
        ref = [render(serial, cloud, c, s).image.copy() for c in cams]
    finally:
        serial.close()
    lanes = [Context(0) for _ in range(4)]
    out = [None] * len(cams)
    errs = []

    def worker(li):
        try:
            fr = RenderOutput(lanes[li])
            for k in range(li, len(cams), len(lanes)):
                for _ in range(3):  # repeated frames into the same output
                    render(lanes[li], cloud, cams[k], s, out=fr)
                out[k] = fr.image.copy()
        except Exception as e:  # surfaced below
            errs.append(e)

    ths = [threading.Thread(target=worker, args=(i,)) for i in range(len(lanes))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for c in lanes:
        c.close()
    assert not errs, errs
    for k in range(len(cams)):
        assert np.array_equal(out[k], ref[k]), k

"""Small workloads for compute-sanitizer (racecheck / synccheck / memcheck): every kernel
of the render, backward, band, async and training paths at sizes the instrumented run
finishes in minutes. `python tools/sanitize_case.py [small|bigsort|train|overflow]`."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_20686_b200 import (CameraPose, Context, GaussianCloud, GradBuffers, RenderOutput,  # noqa: E402
                                   RenderSettings, backward, render, render_band, scenes)
from paper_2410_20686_b200 import _capi as capi  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "small"
ctx = Context(0)
dev = torch.device("cuda", 0)
if mode == "bigsort":
    # > 2^22 tile entries: the 384-thread onesweep shape
    c = scenes.cloud_c3(600_000)
    cam = CameraPose(2048, 1024)
else:
    c = scenes.cloud_c3(20_000)
    cam = scenes.yaw_camera(0.4, 512, 256, (0.05, 0.0, 0.02))
cloud = GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(getattr(c, k))).to(dev)
                        for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")])
s = RenderSettings()
W, H = cam.width, cam.height
fr = render(ctx, cloud, cam, s)
print("entries", fr.info().n_entries)
dl = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, 3 * W * H).astype(np.float32)).to(dev)
n = cloud.n
z = lambda *sh: torch.zeros(sh, dtype=torch.float32, device=dev)
g = GradBuffers(z(3, n), z(4, n), z(3, n), z(n), z(3, n), z(n), z(n), torch.zeros(n, dtype=torch.int32, device=dev))
backward(ctx, cloud, cam, fr, dl, s, grads=g)
if mode == "small":
    fp = RenderOutput(ctx, capi.FRAME_PLAIN_BLEND)  # the un-culled kernels
    render(ctx, cloud, cam, s, out=fp)
    backward(ctx, cloud, cam, fp, dl, s, grads=g, accumulate=True)
    for r0 in (0, 64, 192):  # band path
        render_band(ctx, cloud, cam, s, r0, r0 + 64)
    ctx.set_async(True)  # capacity path: device-side counts
    fa = RenderOutput(ctx)
    for k in range(3):
        render(ctx, cloud, scenes.yaw_camera(0.7 * k, W, H), s, out=fa)
        backward(ctx, cloud, scenes.yaw_camera(0.7 * k, W, H), fa, dl, s, grads=g, accumulate=True)
    fa.check()
    ctx.set_async(False)
    import ctypes as C
    loss = C.c_double()
    img = torch.from_numpy(fr.image.ravel()).to(dev)
    tgt = img.flip(0).contiguous()
    grad = torch.empty_like(img)
    ctx.check(ctx.lib.odgs_photometric_loss(ctx.handle, C.c_void_p(img.data_ptr()), C.c_void_p(tgt.data_ptr()),
                                            W, H, 0.2, C.c_void_p(grad.data_ptr()), C.byref(loss)))
if mode == "overflow":
    # a backward enqueued on an asynchronous frame whose render overflowed its entry
    # buffers (before the check point): the fold must stay inside the record buffers
    actx = Context(0)
    actx.set_async(True)
    fo = RenderOutput(actx)
    small = GaussianCloud(cloud.means, cloud.rotations, cloud.log_scales - 3.0, cloud.raw_opacities, cloud.colors)
    render(actx, small, cam, s, out=fo)
    render(actx, cloud, cam, s, out=fo)
    backward(actx, cloud, cam, fo, dl, s, grads=g)
    assert fo.check()
    backward(actx, cloud, cam, fo, dl, s, grads=g)
    actx.close()
if mode == "train":
    # the two-stream view pipeline of the trainer (four views, two steps): loss, Adam and
    # the backward passes accumulating into one buffer from two contexts
    from paper_2410_20686_b200.train import TrainConfig, ViewShardedTrainer
    views = scenes.c4_views(W, H, 4)
    targets = [img_t for img_t in (torch.from_numpy(render(ctx, cloud, scenes.yaw_camera(0.3 * k, W, H), s).image
                                                    .ravel()).to(dev) for k in range(4))]
    tr = ViewShardedTrainer(ctx, cloud, views, targets, s, TrainConfig(), extent=10.0, pipeline=2)
    assert len(tr.lanes) == 2
    for _ in range(2):
        tr.step()
torch.cuda.synchronize()
print("ok", mode)

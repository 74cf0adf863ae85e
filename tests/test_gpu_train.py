"""GPU training-step kernels vs float32 restatements of the reference formulas:
photometric_loss at lambda = 0 (metrics.hpp:152-184), adam_update + quaternion
renormalisation + densify window (optimizer.hpp:74-84, 114-139), and the
view-sharded step on one GPU (gradients add over views)."""
import ctypes as C
import math

import numpy as np
import pytest
import torch

import oracle_lib
from helpers import to_cloud32
from paper_2410_20686_b200 import CameraPose, Context, GaussianCloud, GradBuffers, RenderSettings, backward, render
from paper_2410_20686_b200 import _capi as capi
from paper_2410_20686_b200.train import TrainConfig, ViewShardedTrainer, means_lr_at

pytestmark = pytest.mark.gpu
f32 = np.float32


def test_l1_loss_and_gradient(gpu_ctx):
    W, H = 256, 128
    rng = np.random.default_rng(0)
    a = rng.random(3 * W * H, dtype=np.float32)
    b = rng.random(3 * W * H, dtype=np.float32)
    b[:100] = a[:100]  # exact zeros of the difference
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    grad = torch.empty_like(da)
    loss = C.c_double()
    gpu_ctx.check(gpu_ctx.lib.odgs_photometric_loss(gpu_ctx.handle, C.c_void_p(da.data_ptr()),
                                                    C.c_void_p(db.data_ptr()), W, H, 0.0,
                                                    C.c_void_p(grad.data_ptr()), C.byref(loss)))
    d = a - b
    pixels = f32(3 * W * H)
    expect = (f32(1) * np.sign(d).astype(np.float32)) / pixels
    assert np.array_equal(grad.cpu().numpy(), expect)
    ref = float(np.abs(d.astype(np.float64)).sum() / (3 * W * H))
    assert abs(loss.value - ref) <= 1e-12 * ref
    g64 = np.empty(3 * W * H)
    oloss = oracle_lib.lib().oracle_photometric_loss(
        a.astype(np.float64).ctypes.data_as(C.POINTER(C.c_double)),
        b.astype(np.float64).ctypes.data_as(C.POINTER(C.c_double)), H, W, 0.0,
        g64.ctypes.data_as(C.POINTER(C.c_double)))
    assert abs(loss.value - oloss) <= 1e-9 * oloss
    with pytest.raises(ValueError):  # lambda must lie in [0, 1) (metrics.hpp:160-161)
        gpu_ctx.check(gpu_ctx.lib.odgs_photometric_loss(gpu_ctx.handle, C.c_void_p(da.data_ptr()),
                                                        C.c_void_p(db.data_ptr()), W, H, 1.0,
                                                        C.c_void_p(grad.data_ptr()), C.byref(loss)))


def adam_np(p, m, v, g, lr, step):
    b1, b2, eps = f32(0.9), f32(0.999), f32(1e-15)
    m[:] = b1 * m + (f32(1) - b1) * g
    v[:] = b2 * v + (f32(1) - b2) * (g * g)
    c1 = f32(1) - np.power(b1, f32(step), dtype=np.float32)
    c2 = f32(1) - np.power(b2, f32(step), dtype=np.float32)
    p -= f32(lr) * (m / c1) / (np.sqrt(v / c2) + eps)


def test_adam_step_matches_float_restatement(gpu_ctx):
    n = 5000
    rng = np.random.default_rng(1)
    arr = lambda *s: rng.standard_normal(s).astype(np.float32)
    P = {"means": arr(3, n), "rotations": arr(4, n), "log_scales": arr(3, n), "raw_opacities": arr(n),
         "colors": arr(3, n)}
    G = {k: arr(*v.shape) * f32(1e-2) for k, v in P.items()}
    pgn, omc, obs = np.abs(arr(n)), np.abs(arr(n)), (rng.random(n) < 0.5).astype(np.int32)
    M = {k: arr(*v.shape) * f32(1e-3) for k, v in P.items()}
    V = {k: np.abs(arr(*v.shape)) * f32(1e-4) for k, v in P.items()}
    lrs = {"means": 1.6e-4, "rotations": 1e-3, "log_scales": 5e-3, "raw_opacities": 0.05, "colors": 2.5e-3}
    step = 7
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    DP, DG, DM, DV = ({k: d(v) for k, v in X.items()} for X in (P, G, M, V))
    acc = {"grad_accum": d(np.zeros(n, np.float32)), "elev_accum": d(np.zeros(n, np.float32)),
           "grad_count": d(np.zeros(n, np.int32))}
    dpgn, domc, dobs = d(pgn), d(omc), d(obs)
    params = capi.Params(n, *[DP[k].data_ptr() for k in ("means", "rotations", "log_scales", "raw_opacities",
                                                         "colors")])
    grads = capi.Grads(*[DG[k].data_ptr() for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")],
                       dpgn.data_ptr(), domc.data_ptr(), dobs.data_ptr(), capi.MEM_DEVICE)
    keys = [("means_m", "means", DM), ("means_v", "means", DV), ("rot_m", "rotations", DM),
            ("rot_v", "rotations", DV), ("scale_m", "log_scales", DM), ("scale_v", "log_scales", DV),
            ("opac_m", "raw_opacities", DM), ("opac_v", "raw_opacities", DV), ("color_m", "colors", DM),
            ("color_v", "colors", DV)]
    st = capi.TrainState(*[src[g].data_ptr() for _, g, src in keys], acc["grad_accum"].data_ptr(),
                         acc["elev_accum"].data_ptr(), acc["grad_count"].data_ptr())
    ap = capi.AdamParams(lrs["means"], lrs["rotations"], lrs["log_scales"], lrs["raw_opacities"], lrs["colors"], step)
    gpu_ctx.check(gpu_ctx.lib.odgs_adam_step(gpu_ctx.handle, C.byref(params), C.byref(grads), C.byref(st),
                                             C.byref(ap)))
    torch.cuda.synchronize()
    for k in P:
        adam_np(P[k], M[k], V[k], G[k], lrs[k], step)
    q = P["rotations"]
    norm = np.sqrt((q[0] * q[0] + q[1] * q[1]) + (q[2] * q[2] + q[3] * q[3]))
    P["rotations"] = np.where(norm > f32(1e-12), q / norm, np.array([[1], [0], [0], [0]], np.float32))
    for k in P:
        assert np.array_equal(DP[k].cpu().numpy(), P[k]), k
        assert np.array_equal(DM[k].cpu().numpy(), M[k]), k
        assert np.array_equal(DV[k].cpu().numpy(), V[k]), k
    assert np.array_equal(acc["grad_accum"].cpu().numpy(), pgn)
    assert np.array_equal(acc["grad_count"].cpu().numpy(), obs)


def test_view_sharded_step_sums_views_on_one_gpu(gpu_ctx):
    arrs = oracle_lib.random_cloud(301, 4000)
    host = to_cloud32(arrs)
    dev = lambda: GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(getattr(host, k))).cuda()
                                  for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")])
    W, H = 512, 256
    views = [CameraPose(W, H), CameraPose(W, H, np.eye(3), [0.1, 0.0, -0.2])]
    tgt = [torch.from_numpy(render(gpu_ctx, to_cloud32(oracle_lib.random_cloud(302, 4000)), v,
                                   RenderSettings()).image.ravel()).cuda() for v in views]
    cloud = dev()
    tr = ViewShardedTrainer(gpu_ctx, cloud, views, tgt, RenderSettings(), TrainConfig(lambda_ssim=0.0), extent=10.0)
    # Expected gradient: sum of per-view backward passes of the L1 loss.
    expected = None
    for v, t in zip(views, tgt):
        fr = render(gpu_ctx, cloud, v, RenderSettings())
        img = torch.from_numpy(fr.image.ravel()).cuda()
        dl = (torch.sign(img - t) / torch.tensor(3 * W * H, dtype=torch.float32, device="cuda")).float()
        g = backward(gpu_ctx, cloud, v, fr, dl, RenderSettings())
        expected = g if expected is None else GradBuffers(*[a + b for a, b in zip(
            (expected.means, expected.rotations, expected.log_scales, expected.raw_opacities, expected.colors,
             expected.pixel_grad_norm, expected.one_minus_cos, expected.observed),
            (g.means, g.rotations, g.log_scales, g.raw_opacities, g.colors, g.pixel_grad_norm, g.one_minus_cos,
             g.observed))])
    before = cloud.means.clone()
    losses = [tr.step()]
    # The trainer's buffer holds the gradient at the pre-update cloud: the view sum.
    for k in ("means", "rotations", "log_scales", "raw_opacities", "colors", "pixel_grad_norm", "one_minus_cos",
              "observed"):
        assert np.array_equal(getattr(tr.grads, k).cpu().numpy(), getattr(expected, k)), k
    losses += [tr.step() for _ in range(2)]
    assert all(math.isfinite(l) for l in losses)
    assert losses[-1] < losses[0]
    assert not torch.equal(before, cloud.means)


@pytest.mark.parametrize("lam,W,H", [(0.2, 256, 128), (0.5, 256, 128), (0.2, 203, 77), (0.2, 1030, 515)])
def test_photometric_loss_with_ssim_matches_oracle(gpu_ctx, lam, W, H):
    """metrics.hpp:83-184 (SSIM window 11, sigma 1.5, K1 .01, K2 .03) vs the fp64 oracle;
    sizes off the kernels' 56 x 16 tiles and 4-output runs included."""
    rng = np.random.default_rng(11)
    a = rng.random(3 * W * H, dtype=np.float32)
    b = np.clip(a + rng.normal(0, 0.1, a.shape).astype(np.float32), 0, 1).astype(np.float32)
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    grad = torch.empty_like(da)
    loss = C.c_double()
    gpu_ctx.check(gpu_ctx.lib.odgs_photometric_loss(gpu_ctx.handle, C.c_void_p(da.data_ptr()),
                                                    C.c_void_p(db.data_ptr()), W, H, lam,
                                                    C.c_void_p(grad.data_ptr()), C.byref(loss)))
    g64 = np.empty(3 * W * H)
    oloss = oracle_lib.lib().oracle_photometric_loss(
        a.astype(np.float64).ctypes.data_as(C.POINTER(C.c_double)),
        b.astype(np.float64).ctypes.data_as(C.POINTER(C.c_double)), H, W, lam,
        g64.ctypes.data_as(C.POINTER(C.c_double)))
    assert abs(loss.value - oloss) <= 1e-5 * abs(oloss)
    g = grad.cpu().numpy().astype(np.float64)
    assert np.abs(g - g64).max() <= 1e-4 * np.abs(g64).max()


def _trainer_setup(ctx, world, rank, group=None):
    arrs = oracle_lib.random_cloud(303, 6000)
    host = to_cloud32(arrs)
    cloud = GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(getattr(host, k))).cuda()
                            for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")])
    W, H = 512, 256
    from paper_2410_20686_b200 import scenes
    views = scenes.c4_views(W, H, 2)
    tcloud = to_cloud32(oracle_lib.random_cloud(304, 6000))
    targets = [torch.from_numpy(render(ctx, tcloud, v, RenderSettings()).image.ravel()).cuda() for v in views]
    return ViewShardedTrainer(ctx, cloud, views, targets, RenderSettings(), TrainConfig(), extent=10.0, rank=rank,
                              world=world, group=group)


def _sharded_rank(rank, world, port, q):
    try:
        import os
        import torch.distributed as dist
        from paper_2410_20686_b200 import Context
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        ctx = Context(0)
        tr = _trainer_setup(ctx, world, rank)
        losses = [tr.step() for _ in range(2)]
        torch.cuda.synchronize()
        out = {k: getattr(tr.cloud, k).cpu().numpy() for k in ("means", "rotations", "log_scales", "raw_opacities",
                                                               "colors")}
        q.put((rank, (out, losses, tr.mine)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def test_view_sharded_trainer_two_ranks_matches_one_process(gpu_ctx):
    """ViewShardedTrainer.step() on two ranks (two processes on GPU 0, gloo all-reduce of
    the CUDA gradient buffers): after two steps every rank's cloud equals the
    single-process trainer's over both views, bit for bit (the all-reduced sum g0 + g1
    adds the same floats as the local accumulation 0 + g0 + g1, and every rank runs the
    identical Adam step)."""
    import multiprocessing as mp
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    procs = [ctx_mp.Process(target=_sharded_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert not isinstance(res[r], str), res[r]
    assert res[0][2] == [0] and res[1][2] == [1]
    tr = _trainer_setup(gpu_ctx, 1, 0)
    losses = [tr.step() for _ in range(2)]
    torch.cuda.synchronize()
    for k in ("means", "rotations", "log_scales", "raw_opacities", "colors"):
        ref = getattr(tr.cloud, k).cpu().numpy()
        for r in range(2):
            assert np.array_equal(res[r][0][k], ref), (r, k)
    # the per-rank losses add up to the single-process loss (each rank sums its views)
    for step in range(2):
        assert abs(res[0][1][step] + res[1][1][step] - losses[step]) <= 1e-12 * abs(losses[step])


def test_pipelined_trainer_matches_sequential(gpu_ctx):
    """pipeline=True (views alternate between two contexts / streams; the backward passes
    stay in view order through events) gives the sequential trainer's clouds bit for bit
    after two steps of four views; the losses agree up to the order of the two lanes'
    float64 sums."""
    arrs = oracle_lib.random_cloud(305, 6000)
    host = to_cloud32(arrs)
    W, H = 512, 256
    from paper_2410_20686_b200 import scenes
    views = scenes.c4_views(W, H, 4)
    tcloud = to_cloud32(oracle_lib.random_cloud(306, 6000))
    targets = [torch.from_numpy(render(gpu_ctx, tcloud, v, RenderSettings()).image.ravel()).cuda() for v in views]
    out = []
    for pipe in (False, True):
        cloud = GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(getattr(host, k))).cuda()
                                for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")])
        tr = ViewShardedTrainer(gpu_ctx, cloud, views, targets, RenderSettings(), TrainConfig(), extent=10.0,
                                pipeline=pipe)
        assert len(tr.lanes) == (2 if pipe else 1)
        losses = [tr.step() for _ in range(2)]
        torch.cuda.synchronize()
        out.append(({k: getattr(cloud, k).cpu().numpy() for k in ("means", "rotations", "log_scales",
                                                                   "raw_opacities", "colors")}, losses))
    for k in out[0][0]:
        assert np.array_equal(out[0][0][k], out[1][0][k]), k
    for a, b in zip(out[0][1], out[1][1]):
        assert abs(a - b) <= 1e-12 * abs(a)


def test_pipelined_trainer_overflow_rerun_matches_sequential(gpu_ctx):
    """A step whose views need more tile entries than the lanes' frames were sized for
    (log-scales grown by 2 after the first step): both lanes' check points report the
    overflow, the step runs again with grown buffers, and the pipelined trainer still
    ends with the sequential trainer's cloud bit for bit."""
    arrs = oracle_lib.random_cloud(307, 5000)
    host = to_cloud32(arrs)
    W, H = 512, 256
    from paper_2410_20686_b200 import scenes
    views = scenes.c4_views(W, H, 4)
    tcloud = to_cloud32(oracle_lib.random_cloud(308, 5000))
    targets = [torch.from_numpy(render(gpu_ctx, tcloud, v, RenderSettings()).image.ravel()).cuda() for v in views]
    out = []
    for pipe in (False, True):
        ls = np.ascontiguousarray(host.log_scales) - 2.0  # small splats: few entries per view
        cloud = GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(a)).cuda()
                                for a in (host.means, host.rotations, ls, host.raw_opacities, host.colors)])
        ctx = Context(0)
        ctx.set_async(True)
        tr = ViewShardedTrainer(ctx, cloud, views, targets, RenderSettings(), TrainConfig(), extent=10.0,
                                pipeline=pipe)
        tr.step()
        k0 = [ln.frame.info().n_entries for ln in tr.lanes]
        with torch.no_grad():
            cloud.log_scales += 2.0  # many more entries than the frames hold
        tr.step()
        torch.cuda.synchronize()
        k1 = [ln.frame.info().n_entries for ln in tr.lanes]
        assert all(b > 2 * a for a, b in zip(k0, k1)), (k0, k1)
        out.append({k: getattr(cloud, k).cpu().numpy() for k in ("means", "rotations", "log_scales",
                                                                  "raw_opacities", "colors")})
        ctx.close()
    for k in out[0]:
        assert np.array_equal(out[0][k], out[1][k]), k

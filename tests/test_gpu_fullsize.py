"""Parity at the BASELINE configs' full sizes (BASELINE.json configs 1, 4, 5; C2 and C3
are covered in test_gpu_sh.py / test_gpu_stages.py / test_gpu_forward.py).

  C1  100K Gaussians (scenes::random_cloud<float>(mt19937(77)), default bounds) at
      1024x512 — the reference's own test workload (test_rasterizer.cpp:148-157):
      every RenderOutput field bit-exact vs oracle::render<float, PortableMath>.
  C5  10M Gaussians at 4096x2048: tile CSR, tile entries, walk lengths, transmittance
      and image bit-exact vs the oracle; each of the 8 row bands equal to its rows.
  C4  3M Gaussians, 8 views at 2048x1024, photometric loss (lambda 0.2): every view's
      forward bit-exact vs the oracle and its gradients within group-relative 1e-3 of
      the float oracle's backward (backward.hpp:380-448) on the same upstream gradient;
      the trainer's summed buffer equals the per-view sum (GradBuffers::accumulate,
      backward.hpp:364-373) bit for bit and the oracle's sum within 1e-3; the Adam step
      (optimizer.hpp:74-84, 114-139) bit-exact vs the float restatement.
The clouds come from the oracle's std::mt19937 generator (SURVEY.md §8d seeds).
"""
import ctypes as C
import math

import numpy as np
import pytest
import torch

import oracle_lib
from helpers import assert_bit_exact, cam32, gpu_fields, oracle_fields, settings_pair, to_cloud32
from paper_2410_20686_b200 import CameraPose, GaussianCloud, RenderSettings, backward, render, render_band, scenes
from paper_2410_20686_b200 import _capi as capi

pytestmark = pytest.mark.gpu

GROUPS = ["means", "rotations", "log_scales", "raw_opacities", "colors"]


def group_rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return np.abs(a - b).max() / max(np.abs(a).max(), np.abs(b).max(), 1e-12)


def to_device(arrs):
    return GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda() for a in arrs])


def test_c1_full_size_bit_exact(gpu_ctx):
    arrs = oracle_lib.random_cloud(77, 100_000)
    cam = CameraPose(1024, 512)
    gs, os_ = settings_pair()
    g = gpu_fields(gpu_ctx, to_cloud32(arrs), cam, gs)
    o = oracle_fields(arrs, cam, os_, portable=True)
    assert (g["n_splats"], g["n_instances"], g["n_entries"]) == tuple(o["stats"][:3])
    assert_bit_exact(g, o)


C5_BOUNDS = (0.5, 20.0, 1.45, 0.05, 0.95, 0.0005, 0.005)


def test_c5_full_size_bit_exact_and_bands(gpu_ctx):
    arrs = oracle_lib.random_cloud(5001, 10_000_000, C5_BOUNDS)
    W, H = 4096, 2048
    cam = CameraPose(W, H)
    gs, os_ = settings_pair()
    cloud = to_device(arrs)
    fr = render(gpu_ctx, cloud, cam, gs)
    info = fr.info()
    r, t = cam32(cam)
    of = oracle_lib.render(arrs, r, t, W, H, os_, portable=True)
    del arrs
    st = of.get("stats")
    assert (info.n_splats, info.n_instances, info.n_entries) == (st[0], st[1], st[2])
    assert np.array_equal(fr.tile_offsets, of.get("tile_offsets"))
    assert np.array_equal(fr.tile_entries, of.get("tile_entries"))
    walked = fr.walked
    assert np.array_equal(walked.ravel(), of.get("walked"))
    tr = fr.transmittance
    assert np.array_equal(tr.ravel(), of.get("transmittance").astype(np.float32))
    img = fr.image
    assert np.array_equal(img.ravel(), of.get("image").astype(np.float32))
    del of
    rows = H // 8
    entries = 0
    for b in range(8):
        r0, r1 = b * rows, (b + 1) * rows
        bf = render_band(gpu_ctx, cloud, cam, gs, r0, r1)
        assert np.array_equal(bf.image[:, :, r0:r1], img[:, :, r0:r1]), b
        assert np.array_equal(bf.transmittance[:, r0:r1], tr[:, r0:r1]), b
        assert np.array_equal(bf.walked[:, r0:r1], walked[:, r0:r1]), b
        entries += bf.info().n_entries
        bf.destroy()
    assert entries == info.n_entries


C4_BOUNDS = (0.5, 20.0, 1.45, 0.05, 0.95, 0.001, 0.01)


def test_c4_full_size_train_step(gpu_ctx):
    from test_gpu_train import adam_np
    from paper_2410_20686_b200.train import TrainConfig, ViewShardedTrainer, means_lr_at
    n, W, H = 3_000_000, 2048, 1024
    arrs = oracle_lib.random_cloud(4001, n, C4_BOUNDS)
    tarrs = oracle_lib.random_cloud(4002, n, C4_BOUNDS)
    views = scenes.c4_views(W, H, 8)
    gs, os_ = settings_pair()
    tcloud = to_device(tarrs)
    targets = [torch.from_numpy(render(gpu_ctx, tcloud, v, gs).image.ravel()).cuda() for v in views]
    del tcloud, tarrs
    cloud = to_device(arrs)
    cfg = TrainConfig()  # lambda_ssim 0.2
    dl = torch.empty(3 * W * H, dtype=torch.float32, device="cuda")
    gpu_sum = None
    oracle_sum = None
    for v, (cam, tgt) in enumerate(zip(views, targets)):
        fr = render(gpu_ctx, cloud, cam, gs)
        loss = C.c_double()
        gpu_ctx.wait_torch()  # the target was uploaded on torch's stream
        gpu_ctx.check(gpu_ctx.lib.odgs_photometric_loss(
            gpu_ctx.handle, C.c_void_p(fr.device_ptr(capi.FRAME_IMAGE)), C.c_void_p(tgt.data_ptr()), W, H,
            cfg.lambda_ssim, C.c_void_p(dl.data_ptr()), C.byref(loss)))
        g = backward(gpu_ctx, cloud, cam, fr, dl, gs)  # host GradBuffers
        # The float oracle's isZero() skips pixels with |dL/dpixel| <= 1e-5
        # (backward.hpp:248); the photometric gradient is ~1e-7 per pixel, so the oracle
        # would drop every pixel. The comparison runs on dl * 2^20 (an
        # exact scaling; the gradients are linear in dl) on both sides.
        dl_big = dl * float(2 ** 20)
        g_big = backward(gpu_ctx, cloud, cam, fr, dl_big, gs)
        r, t = cam32(cam)
        of = oracle_lib.render(arrs, r, t, W, H, os_, portable=True)
        assert np.array_equal(fr.walked.ravel(), of.get("walked")), v
        assert np.array_equal(fr.image.ravel(), of.get("image").astype(np.float32)), v
        of.backward(dl_big.cpu().numpy().astype(np.float64))
        o = {"means": of.get("g_means"), "rotations": of.get("g_rotations"), "log_scales": of.get("g_log_scales"),
             "raw_opacities": of.get("g_raw_opacities"), "colors": of.get("g_colors")}
        for k in GROUPS:
            assert group_rel(getattr(g_big, k), o[k]) < 1e-3, (v, k, group_rel(getattr(g_big, k), o[k]))
        assert np.array_equal(g_big.observed, of.get("g_observed")), v
        assert np.abs(g_big.one_minus_cos - of.get("g_one_minus_cos")).max() < 1e-5, v
        assert group_rel(g_big.pixel_grad_norm, of.get("g_pixel_grad_norm")) < 1e-3, v
        cur = {k: getattr(g, k).copy() for k in GROUPS + ["pixel_grad_norm", "one_minus_cos", "observed"]}
        osum = {k: (o[k] / 2.0 ** 20).astype(np.float32).reshape(cur[k].shape) for k in GROUPS}
        if gpu_sum is None:
            gpu_sum, oracle_sum = cur, osum
        else:
            for k in cur:
                gpu_sum[k] = gpu_sum[k] + cur[k]
            for k in osum:
                oracle_sum[k] = oracle_sum[k] + osum[k]
        del of, fr
    for k in GROUPS:
        assert group_rel(gpu_sum[k], oracle_sum[k]) < 1e-3, k
    # The trainer: all 8 views on this GPU, one step. Its buffer must hold the same sum.
    extent = float(np.sqrt(((arrs[0] - arrs[0].mean(axis=1, keepdims=True)) ** 2).sum(axis=0).max()))
    tr = ViewShardedTrainer(gpu_ctx, cloud, views, targets, gs, cfg, extent)
    P = {k: np.asarray(a, np.float32).copy() for k, a in zip(GROUPS, arrs)}
    tr.step()
    torch.cuda.synchronize()
    for k in gpu_sum:
        assert np.array_equal(getattr(tr.grads, k).cpu().numpy(), gpu_sum[k]), k
    lrs = {"means": np.float32(means_lr_at(0, cfg) * extent), "rotations": cfg.lr_rotation,
           "log_scales": cfg.lr_scale, "raw_opacities": cfg.lr_opacity, "colors": cfg.lr_color}
    for k in GROUPS:
        m = np.zeros_like(P[k])
        v = np.zeros_like(P[k])
        adam_np(P[k], m, v, gpu_sum[k], lrs[k], 1)
    q = P["rotations"]
    norm = np.sqrt((q[0] * q[0] + q[1] * q[1]) + (q[2] * q[2] + q[3] * q[3]))
    P["rotations"] = np.where(norm > np.float32(1e-12), q / norm, np.array([[1], [0], [0], [0]], np.float32))
    for k in GROUPS:
        assert np.array_equal(getattr(cloud, k).cpu().numpy(), P[k]), k

"""SH colour extension (BASELINE config C2). The reference
colour is RGB only, so there is no reference to pin against: the oracle
restates this build's definition (oracle::sh_color — real SH degree 1..3 at the
world-space view direction, c = rgb + sum_k Y_k coef_k, degree 0 = passthrough) and
its backward is pinned by finite differences in oracle/ref_tests.cpp. Here the GPU
must be bit-exact with the portable oracle in the forward and within the gradient
tolerance of the fp64 oracle in the backward, up to the full C2 size."""
import math

import numpy as np
import pytest

import oracle_lib
from helpers import assert_bit_exact, cam32, gpu_fields, oracle_fields, settings_pair
from paper_2410_20686_b200 import CameraPose, GaussianCloud, RenderSettings, backward, render

pytestmark = pytest.mark.gpu
GROUPS = ["means", "rotations", "log_scales", "raw_opacities", "colors"]


def group_rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return np.abs(a - b).max() / max(np.abs(a).max(), np.abs(b).max(), 1e-12)


def sh_cloud(seed, n, degree, bounds=oracle_lib.DEFAULT_BOUNDS):
    arrs = oracle_lib.random_cloud(seed, n, bounds)
    nb = (degree + 1) ** 2 - 1
    sh = np.random.default_rng(seed + 1).normal(0, 0.05, (nb, 3, n)).astype(np.float32).astype(np.float64)
    return arrs, sh


def gpu_cloud(arrs, degree, sh):
    return GaussianCloud.from_numpy(*arrs, sh_degree=degree, sh_rest=sh)


@pytest.mark.parametrize("degree", [1, 2, 3])
def test_sh_forward_bit_exact(gpu_ctx, degree):
    arrs, sh = sh_cloud(700 + degree, 3000, degree)
    cam = CameraPose(512, 256, np.array([[0.8775826, 0.0, 0.4794255], [0.0, 1.0, 0.0], [-0.4794255, 0.0, 0.8775826]]),
                     [0.3, -0.1, 0.2])
    gs, os_ = settings_pair()
    g = gpu_fields(gpu_ctx, gpu_cloud(arrs, degree, sh), cam, gs)
    r, t = cam32(cam)
    fr = oracle_lib.render(arrs, r, t, cam.width, cam.height, os_, portable=True, sh_degree=degree,
                           sh_rest=sh.reshape(-1, arrs[3].shape[0]))
    o = {"image": fr.get("image").reshape(3, 512, 256), "walked": fr.get("walked").reshape(512, 256),
         "splat_color": fr.get("splat_color").reshape(-1, 3), "tile_offsets": fr.get("tile_offsets")}
    assert_bit_exact(g, o, ["splat_color", "tile_offsets", "walked", "image"])
    # The SH term changes colours (not a silent passthrough).
    assert np.abs(g["splat_color"] - (np.asarray(arrs[4]).T[:len(g["splat_color"])])).max() > 1e-3


@pytest.mark.parametrize("degree", [1, 3])
def test_sh_gradients_match_fp64_oracle(gpu_ctx, degree):
    bounds = (0.8, 10.0, 75.0 * math.pi / 180.0, 0.1, 0.7, 0.02, 0.12)
    arrs, sh = sh_cloud(720 + degree, 10, degree, bounds)
    cam = CameraPose(64, 32, np.eye(3), [0.1, -0.05, 0.2])
    gs, os_ = settings_pair(cutoff_sigma=8.0)
    dl = np.random.default_rng(5).uniform(-1, 1, (3, 64, 32)).astype(np.float32)
    cloud = gpu_cloud(arrs, degree, sh)
    g = backward(gpu_ctx, cloud, cam, render(gpu_ctx, cloud, cam, gs), dl, gs)
    r, t = cam32(cam)
    n = arrs[3].shape[0]
    fr = oracle_lib.render(arrs, r, t, 64, 32, os_, dbl=True, sh_degree=degree, sh_rest=sh.reshape(-1, n))
    fr.backward(dl.astype(np.float64))
    assert group_rel(g.sh_rest, fr.get("g_sh_rest")) < 1e-3
    for k in GROUPS:
        assert group_rel(getattr(g, k), fr.get("g_" + k)) < 1e-3, k


def test_c2_full_size_sh3_forward_and_gradients(gpu_ctx):
    """BASELINE config 2 at full size: 500K Gaussians, SH degree 3, 2048x1024, fwd + bwd
    (bounds of SURVEY.md §8d), against the float oracle that makes the same forward
    decisions; forward bit-exact."""
    n = 500_000
    bounds = (0.8, 10.0, 75.0 * math.pi / 180.0, 0.1, 0.7, 0.001, 0.01)
    arrs = oracle_lib.random_cloud(2002, n, bounds)
    sh = np.random.default_rng(2003).normal(0, 0.05, (15, 3, n)).astype(np.float32).astype(np.float64)
    dl = np.random.default_rng(2004).uniform(-1, 1, (3, 2048, 1024)).astype(np.float32)
    cam = CameraPose(2048, 1024)
    gs, os_ = settings_pair()
    cloud = gpu_cloud(arrs, 3, sh)
    fr = render(gpu_ctx, cloud, cam, gs)
    g = backward(gpu_ctx, cloud, cam, fr, dl, gs)
    of = oracle_lib.render(arrs, np.eye(3), np.zeros(3), 2048, 1024, os_, portable=True, sh_degree=3,
                           sh_rest=sh.reshape(-1, n))
    assert np.array_equal(fr.image.ravel(), of.get("image").astype(np.float32))
    assert np.array_equal(fr.walked.ravel(), of.get("walked"))
    of.backward(dl.astype(np.float64))
    for k in GROUPS:
        assert group_rel(getattr(g, k), of.get("g_" + k)) < 1e-3, k
    assert group_rel(g.sh_rest, of.get("g_sh_rest")) < 1e-3

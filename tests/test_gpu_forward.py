"""GPU forward parity: the sm_100a path through the C ABI vs the CPU oracle.

Contract: against oracle::render<float, PortableMath> the GPU is
bit-exact on every RenderOutput field — splats, instance order, tile CSR, tile
entries, walk lengths, transmittance, image. Against the literal libm oracle
(StdMath, float and double) the image matches within 1e-4 max-abs.
Cases follow the reference tests (proj/tests/test_rasterizer.cpp, acceptance.cpp).
"""
import math

import numpy as np
import pytest

import oracle_lib
from helpers import (angle_axis, assert_bit_exact, gpu_fields, oracle_fields, rot_yaw, settings_pair, to_cloud32)
from paper_2410_20686_b200 import (CameraPose, DomainError, GaussianCloud, InvalidArgument, OdgsRuntimeError,
                                   RenderSettings, cull, render)
from paper_2410_20686_b200 import scenes

pytestmark = pytest.mark.gpu


def f32(arrs):
    return tuple(np.asarray(a, dtype=np.float32).astype(np.float64) for a in arrs)


SCENES = [
    # (name, cloud factory, camera, settings kwargs)
    ("ref77_256x128", lambda: oracle_lib.random_cloud(77, 100), CameraPose(256, 128), {}),
    ("ref77_2000_yawed", lambda: oracle_lib.random_cloud(78, 2000),
     CameraPose(512, 256, angle_axis(0.8, [1, 2, 3]), [0.1, -0.2, 0.15]), {}),
    ("c3_small_1024", lambda: f32(tuple(a for a in [getattr(scenes.cloud_c3(20000), k) for k in
                                                  ("means", "rotations", "log_scales", "raw_opacities",
                                                   "colors")])), CameraPose(1024, 512), {}),
    ("tile8_cutoff8", lambda: oracle_lib.random_cloud(404, 500), CameraPose(256, 128),
     {"tile_size": 8, "cutoff_sigma": 8.0}),
    ("tile32", lambda: oracle_lib.random_cloud(405, 500), CameraPose(512, 256), {"tile_size": 32}),
    ("tile20_ragged", lambda: oracle_lib.random_cloud(406, 300), CameraPose(250, 125), {"tile_size": 20}),
    # tiles above 64 px: blended in 4096-pixel chunks per CTA
    ("tile80_ragged", lambda: oracle_lib.random_cloud(408, 600), CameraPose(300, 150), {"tile_size": 80}),
    ("tile128", lambda: oracle_lib.random_cloud(409, 600), CameraPose(512, 256), {"tile_size": 128}),
    ("near_far_shell", lambda: oracle_lib.random_cloud(407, 800), CameraPose(256, 128),
     {"near_radius": 3.0, "far_radius": 12.0}),
]


@pytest.mark.parametrize("name,make,cam,kw", SCENES, ids=[s[0] for s in SCENES])
def test_bit_exact_vs_portable_oracle(gpu_ctx, name, make, cam, kw):
    cloud = make()
    gs, os_ = settings_pair(**kw)
    g = gpu_fields(gpu_ctx, to_cloud32(cloud), cam, gs)
    o = oracle_fields(cloud, cam, os_, portable=True)
    assert g["n_splats"] == o["stats"][0]
    assert g["n_instances"] == o["stats"][1]
    assert g["n_entries"] == o["stats"][2]
    assert_bit_exact(g, o)


@pytest.mark.parametrize("name,make,cam,kw", SCENES[:3], ids=[s[0] for s in SCENES[:3]])
def test_image_tolerance_vs_libm_oracle(gpu_ctx, name, make, cam, kw):
    """Against the literal libm oracle (float and double). The compositing rule has
    two discontinuities — the d2 > cutoff^2 skip (rasterizer.hpp:247), where alpha jumps
    by opacity*exp(-cutoff^2/2), and the tile box edge — so a last-bit difference in a
    transcendental can move a pixel across them. With the reference's finite-difference
    cutoff (8 sigma, test_backward.cpp:42-49) the jump is ~1e-14 and every pixel is
    within 1e-4; at the default 3 sigma only isolated pixels may exceed it (the
    reference's own float vs double renders show the same)."""
    cloud = make()
    gs8, os8 = settings_pair(**{**kw, "cutoff_sigma": 8.0})
    g = gpu_fields(gpu_ctx, to_cloud32(cloud), cam, gs8, keep_cov=False)
    for dbl in (False, True):
        o = oracle_fields(cloud, cam, os8, portable=False, dbl=dbl)
        assert np.abs(g["image"] - o["image"]).max() <= 1e-4, dbl
    gs, os_ = settings_pair(**kw)
    g = gpu_fields(gpu_ctx, to_cloud32(cloud), cam, gs, keep_cov=False)
    for dbl in (False, True):
        o = oracle_fields(cloud, cam, os_, portable=False, dbl=dbl)
        px_err = np.abs(g["image"] - o["image"]).max(axis=0)
        assert np.mean(px_err > 1e-4) <= 1e-4, (dbl, np.mean(px_err > 1e-4), px_err.max())
        assert np.mean(g["walked"] != o["walked"]) <= 1e-3


def test_brute_force_oracle_equivalence(gpu_ctx):
    """acceptance.cpp:219-242 / test_rasterizer.cpp:131-158: tiled == brute force within 1e-5."""
    gs, os_ = settings_pair()
    worst = 0.0
    for seed in range(3):
        cloud = oracle_lib.random_cloud(77 + seed, 100)
        cam = CameraPose(256, 128)
        g = gpu_fields(gpu_ctx, to_cloud32(cloud), cam, gs, keep_cov=False)
        o = oracle_fields(cloud, cam, os_, portable=True, brute=True)
        worst = max(worst, float(np.abs(g["image"] - o["brute"]).max()))
    assert worst <= 1e-5


def test_single_opaque_gaussian_on_axis(gpu_ctx):
    """test_rasterizer.cpp:134-145."""
    means = np.array([[0.0], [0.0], [2.0]])
    rot = np.array([[1.0], [0], [0], [0]])
    ls = np.full((3, 1), math.log(np.float32(0.05)))
    op = np.array([math.log(0.95 / 0.05)])
    col = np.array([[1.0], [0.5], [0.25]])
    cloud = f32((means, rot, ls, op, col))
    gs, os_ = settings_pair()
    cam = CameraPose(256, 128)
    g = gpu_fields(gpu_ctx, to_cloud32(cloud), cam, gs)
    o = oracle_fields(cloud, cam, os_, portable=True, brute=True)
    assert_bit_exact(g, o)
    assert np.abs(g["image"] - o["brute"]).max() <= 1e-5


def test_empty_cloud_is_black(gpu_ctx):
    """test_rasterizer.cpp:110-116."""
    z = np.zeros((3, 0), np.float32)
    cloud = GaussianCloud(z, np.zeros((4, 0), np.float32), z.copy(), np.zeros(0, np.float32), z.copy())
    fr = render(gpu_ctx, cloud, CameraPose(64, 32), RenderSettings())
    assert np.all(fr.image == 0)
    assert np.all(fr.transmittance == 1)
    assert np.all(fr.walked == 0)
    assert np.all(fr.tile_offsets == 0)


def test_nonfinite_parameter_names_the_gaussian(gpu_ctx):
    """test_rasterizer.cpp:118-129."""
    cloud = list(oracle_lib.random_cloud(5, 4))
    cloud[0] = cloud[0].copy()
    cloud[0][1, 2] = np.nan
    with pytest.raises(OdgsRuntimeError) as e:
        render(gpu_ctx, to_cloud32(cloud), CameraPose(64, 32), RenderSettings())
    assert e.value.index == 2
    assert "2" in str(e.value)


def test_invalid_camera_and_quaternion(gpu_ctx):
    cloud = to_cloud32(oracle_lib.random_cloud(5, 8))
    with pytest.raises(InvalidArgument):
        render(gpu_ctx, cloud, CameraPose(64, 64), RenderSettings())
    with pytest.raises(InvalidArgument):
        render(gpu_ctx, cloud, CameraPose(64, 32, np.diag([1.0, 1.0, 1.1])), RenderSettings())
    arrs = [np.array(a) for a in oracle_lib.random_cloud(5, 8)]
    arrs[1][:, 3] = 0.0
    arrs[1][:, 6] = 0.0
    with pytest.raises(InvalidArgument) as e:
        render(gpu_ctx, to_cloud32(arrs), CameraPose(64, 32), RenderSettings())
    assert e.value.index == 3  # lowest offending row wins, as in the reference's serial loop


def test_zero_distance_with_zero_near_is_domain_error(gpu_ctx):
    arrs = [np.array(a) for a in oracle_lib.random_cloud(6, 4)]
    arrs[0][:, 1] = 0.0
    with pytest.raises(DomainError) as e:
        render(gpu_ctx, to_cloud32(arrs), CameraPose(64, 32), RenderSettings(near_radius=0.0))
    assert e.value.index == 1


def test_permutation_invariance(gpu_ctx):
    """test_rasterizer.cpp:160-173 (<= 1e-6)."""
    arrs = oracle_lib.random_cloud(83, 60)
    cam = CameraPose(128, 64)
    base = render(gpu_ctx, to_cloud32(arrs), cam, RenderSettings()).image
    perm = np.random.default_rng(0).permutation(60)
    shuffled = tuple(a[..., perm] for a in arrs)
    img = render(gpu_ctx, to_cloud32(shuffled), cam, RenderSettings()).image
    assert np.abs(base - img).max() <= 1e-6


@pytest.mark.parametrize("k", [1, 17, 64, 200])
def test_yaw_by_whole_pixels_shifts_the_image(gpu_ctx, k):
    """test_rasterizer.cpp:175-196 (<= 1e-4)."""
    arrs = oracle_lib.random_cloud(89, 80)
    W, H = 256, 128
    base = render(gpu_ctx, to_cloud32(arrs), CameraPose(W, H), RenderSettings()).image
    delta = np.float32(k) * np.float32(2.0) * np.float32(math.pi) / np.float32(W)
    yawed = render(gpu_ctx, to_cloud32(arrs), CameraPose(W, H, rot_yaw(float(delta))), RenderSettings()).image
    src = (np.arange(W) - k % W + W) % W
    assert np.abs(yawed - base[:, src, :]).max() <= 1e-4


def test_device_resident_cloud_matches_host(gpu_ctx):
    import torch
    arrs = oracle_lib.random_cloud(91, 3000)
    host = to_cloud32(arrs)
    dev = GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(getattr(host, k))).cuda()
                          for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")])
    cam = CameraPose(512, 256)
    a = render(gpu_ctx, host, cam, RenderSettings())
    b = render(gpu_ctx, dev, cam, RenderSettings())
    assert np.array_equal(a.image, b.image)
    assert np.array_equal(a.walked, b.walked)


def test_cull_matches_oracle_shell(gpu_ctx):
    """rasterizer.hpp:15-28 / test_rasterizer.cpp:30-51."""
    means = np.array([[0, 0, 0.05], [0, 1, 0], [500, 0, 0]], dtype=np.float32).T.copy()
    n = 3
    cloud = GaussianCloud(means, np.tile(np.array([[1], [0], [0], [0]], np.float32), (1, n)),
                          np.zeros((3, n), np.float32), np.zeros(n, np.float32), np.zeros((3, n), np.float32))
    assert list(cull(gpu_ctx, cloud, CameraPose(64, 32), 0.1, 100.0)) == [1]
    with pytest.raises(InvalidArgument):
        cull(gpu_ctx, cloud, CameraPose(64, 32), 1.0, 0.5)


def test_full_size_c3_bit_exact(gpu_ctx):
    """BASELINE config 3 at full size (1M Gaussians, 2048x1024, poles + seam)."""
    c = scenes.cloud_c3()
    arrs = tuple(np.asarray(getattr(c, k), dtype=np.float64) for k in
                 ("means", "rotations", "log_scales", "raw_opacities", "colors"))
    cam = CameraPose(2048, 1024)
    gs, os_ = settings_pair()
    g = gpu_fields(gpu_ctx, c, cam, gs, keep_cov=False)
    o = oracle_fields(arrs, cam, os_, portable=True)
    assert_bit_exact(g, o, ["tile_offsets", "walked", "transmittance", "image"])
    # Size-independent properties.
    offs = g["tile_offsets"]
    assert offs[0] == 0 and np.all(np.diff(offs) >= 0) and offs[-1] == g["n_entries"]
    assert np.all(g["transmittance"] >= 1e-4 * (1 - 1e-6))


@pytest.mark.parametrize("tile", [8, 16])
def test_warp_culled_blend_equals_plain_blend(gpu_ctx, tile):
    """The culled blend (conservative per-warp ellipse test) changes no output bit."""
    from paper_2410_20686_b200 import _capi as capi
    c = scenes.cloud_c3(200_000)
    cam = CameraPose(2048, 1024, rot_yaw(0.3))
    s = RenderSettings(tile_size=tile)
    a = render(gpu_ctx, c, cam, s, flags=capi.FRAME_COUNT_WORK)
    b = render(gpu_ctx, c, cam, s, flags=capi.FRAME_PLAIN_BLEND | capi.FRAME_COUNT_WORK)
    assert np.array_equal(a.image, b.image)
    assert np.array_equal(a.walked, b.walked)
    assert np.array_equal(a.transmittance, b.transmittance)
    assert a.work() == b.work()
    assert a.work()[1] > 0
    # without ODGS_FRAME_COUNT_WORK the blend counts nothing (and its outputs are the same)
    d = render(gpu_ctx, c, cam, s)
    assert d.work() == (0, 0)
    assert np.array_equal(a.image, d.image) and np.array_equal(a.walked, d.walked)

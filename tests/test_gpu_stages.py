"""Stage-isolated parity (parity-contract bullet 2): the GPU's sort, bin
and blend stages fed the literal-libm oracle's projected splats.

oracle::render<float, StdMath> (libm transcendentals, the reference's arithmetic)
projects the cloud; its Splat2D records go through odgs_rasterize_splats, i.e. the GPU's
seam-instance emission, (depth, index, shift) radix sorts, tile CSR and blend. Then
  * the instance order, tile_offsets (empty tiles included) and tile_entries are
    bit-exact against the StdMath oracle — integer work that depends on the splats only
    (rasterizer.hpp:141-205);
  * image, transmittance and walked are bit-exact against the oracle's blend of the
    same splats (rasterizer.hpp:216-267, PortableMath's exponential, which the GPU
    shares; the StdMath blend differs only by expf's last bit, checked at tolerance).
"""
import numpy as np
import pytest

import oracle_lib
from helpers import angle_axis, cam32, settings_pair
from paper_2410_20686_b200 import CameraPose, InvalidArgument, rasterize_splats, scenes
from paper_2410_20686_b200 import _capi as capi

pytestmark = pytest.mark.gpu


def c3_prefix(n):
    c = scenes.cloud_c3(n)
    return tuple(np.asarray(getattr(c, k), np.float32).astype(np.float64)
                 for k in ("means", "rotations", "log_scales", "raw_opacities", "colors"))


SCENES = [
    ("ref77_256x128", lambda: oracle_lib.random_cloud(77, 100), CameraPose(256, 128), {}),
    ("pitched_2000", lambda: oracle_lib.random_cloud(78, 2000),
     CameraPose(512, 256, angle_axis(0.8, [1, 2, 3]), [0.1, -0.2, 0.15]), {}),
    ("c3_poles_seam_50k", lambda: c3_prefix(50_000), CameraPose(1024, 512), {}),
    ("tile8_cutoff8", lambda: oracle_lib.random_cloud(404, 500), CameraPose(256, 128),
     {"tile_size": 8, "cutoff_sigma": 8.0}),
    ("tile20_ragged", lambda: oracle_lib.random_cloud(406, 300), CameraPose(250, 125), {"tile_size": 20}),
    ("tile32_yawed", lambda: oracle_lib.random_cloud(405, 3000), scenes.yaw_camera(2.5, 512, 256), {"tile_size": 32}),
]


def splats_of(of):
    g = of.get
    return dict(index=g("splat_index"), pixel_mean=g("splat_mean").reshape(-1, 2),
                cov2d_inv=g("splat_inv").reshape(-1, 4), depth=g("splat_depth"), radius=g("splat_radius"),
                opacity=g("splat_opacity"), color=g("splat_color").reshape(-1, 3))


def check_stages(ctx, arrs, cam, kw):
    gs, os_ = settings_pair(**kw)
    r, t = cam32(cam)
    W, H = cam.width, cam.height
    std = oracle_lib.render(arrs, r, t, W, H, os_, portable=False)  # libm projection + blend
    sp = splats_of(std)
    n = arrs[3].shape[0]
    fr = rasterize_splats(ctx, n, sp["index"], sp["pixel_mean"], sp["cov2d_inv"], sp["depth"], sp["radius"],
                          sp["opacity"], sp["color"], W, H, gs)
    info = fr.info()
    st = std.get("stats")
    assert (info.n_splats, info.n_instances, info.n_entries) == (st[0], st[1], st[2])
    # the injected splats come back unchanged
    assert np.array_equal(fr.splat_field(capi.FRAME_SPLAT_INDEX, dtype=np.int64), sp["index"])
    assert np.array_equal(fr.splat_field(capi.FRAME_SPLAT_DEPTH), sp["depth"].astype(np.float32))
    # integer stages: bit-exact against the libm oracle
    assert np.array_equal(fr.instance_splat, std.get("inst_splat"))
    assert np.array_equal(fr.instance_shift, std.get("inst_shift").astype(np.float32))
    assert np.array_equal(fr.tile_offsets, std.get("tile_offsets"))
    assert np.array_equal(fr.tile_entries, std.get("tile_entries"))
    # blend: bit-exact against the oracle's blend of the same splats
    pb = std.rasterize_splats(portable=True)
    assert np.array_equal(pb.get("tile_entries"), std.get("tile_entries"))
    assert np.array_equal(fr.walked.ravel(), pb.get("walked"))
    assert np.array_equal(fr.transmittance.ravel(), pb.get("transmittance").astype(np.float32))
    assert np.array_equal(fr.image.ravel(), pb.get("image").astype(np.float32))
    # and within the image tolerance of the libm blend (expf's last bit moves at most
    # isolated pixels across the termination threshold)
    walked_std = std.get("walked")
    assert np.mean(fr.walked.ravel() != walked_std) <= 1e-3
    same = np.tile(fr.walked.ravel() == walked_std, 3)
    assert np.abs(fr.image.ravel()[same] - std.get("image")[same]).max(initial=0.0) <= 1e-4


@pytest.mark.parametrize("name,make,cam,kw", SCENES, ids=[s[0] for s in SCENES])
def test_sort_bin_blend_on_libm_splats(gpu_ctx, name, make, cam, kw):
    check_stages(gpu_ctx, make(), cam, kw)


def test_sort_bin_blend_on_libm_splats_full_c3(gpu_ctx):
    """BASELINE config 3 at full size: 1M Gaussians (poles + seam), 2048x1024."""
    check_stages(gpu_ctx, c3_prefix(1_000_000), CameraPose(2048, 1024), {})


def test_rasterize_splats_argument_checks(gpu_ctx):
    from paper_2410_20686_b200 import RenderSettings
    s = RenderSettings()
    one = dict(pixel_mean=np.zeros((2, 2)), cov2d_inv=np.tile([1.0, 0, 0, 1.0], (2, 1)), depth=np.ones(2),
               radius=np.ones(2), opacity=np.full(2, 0.5), color=np.ones((2, 3)))
    with pytest.raises(InvalidArgument):  # indices must ascend
        rasterize_splats(gpu_ctx, 4, [2, 1], **one, width=64, height=32, settings=s)
    with pytest.raises(InvalidArgument):  # inside the cloud
        rasterize_splats(gpu_ctx, 2, [0, 2], **one, width=64, height=32, settings=s)
    bad = dict(one, depth=np.array([1.0, np.nan]))
    with pytest.raises(InvalidArgument) as e:
        rasterize_splats(gpu_ctx, 4, [0, 1], **bad, width=64, height=32, settings=s)
    assert e.value.index == 1
    fr = rasterize_splats(gpu_ctx, 4, np.zeros(0, np.int64), **{k: v[:0] for k, v in one.items()}, width=64,
                          height=32, settings=s)
    assert np.all(fr.image == 0) and np.all(fr.transmittance == 1)

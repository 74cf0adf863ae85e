"""Row-band renders: every band equals the same rows of the
full render bit for bit, and band backward passes add up to the full gradient."""
import numpy as np
import pytest

import oracle_lib
from helpers import to_cloud32
from paper_2410_20686_b200 import CameraPose, InvalidArgument, RenderSettings, backward, render, render_band
from paper_2410_20686_b200 import scenes

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bands", [2, 4, 8])
def test_bands_are_bit_identical_to_full_render(gpu_ctx, bands):
    c = scenes.cloud_c3(100_000)
    cam = CameraPose(2048, 1024)
    s = RenderSettings()
    full = render(gpu_ctx, c, cam, s)
    img, tr, wk = full.image, full.transmittance, full.walked
    rows = 1024 // bands
    total_entries = 0
    for b in range(bands):
        r0, r1 = b * rows, (b + 1) * rows
        fr = render_band(gpu_ctx, c, cam, s, r0, r1)
        assert np.array_equal(fr.image[:, :, r0:r1], img[:, :, r0:r1])
        assert np.array_equal(fr.transmittance[:, r0:r1], tr[:, r0:r1])
        assert np.array_equal(fr.walked[:, r0:r1], wk[:, r0:r1])
        info = fr.info()
        assert (info.row_begin, info.row_end) == (r0, r1)
        total_entries += info.n_entries
    assert total_entries == full.info().n_entries


def test_band_gradients_add_to_the_full_gradient(gpu_ctx):
    arrs = oracle_lib.random_cloud(401, 3000)
    cloud = to_cloud32(arrs)
    cam = CameraPose(512, 256)
    s = RenderSettings()
    dl = np.random.default_rng(3).uniform(-1, 1, (3, 512, 256)).astype(np.float32)
    full = backward(gpu_ctx, cloud, cam, render(gpu_ctx, cloud, cam, s), dl, s)
    acc = None
    for r0 in range(0, 256, 64):
        fr = render_band(gpu_ctx, cloud, cam, s, r0, r0 + 64)
        acc = backward(gpu_ctx, cloud, cam, fr, dl, s, grads=acc, accumulate=acc is not None)
    for k in ("means", "rotations", "log_scales", "raw_opacities", "colors"):
        a, b = getattr(acc, k), getattr(full, k)
        assert np.abs(a - b).max() <= 1e-5 * max(np.abs(b).max(), 1e-12), k


def test_band_rows_must_be_tile_aligned(gpu_ctx):
    cloud = to_cloud32(oracle_lib.random_cloud(5, 10))
    with pytest.raises(InvalidArgument):
        render_band(gpu_ctx, cloud, CameraPose(256, 128), RenderSettings(), 8, 64)
    with pytest.raises(InvalidArgument):
        render_band(gpu_ctx, cloud, CameraPose(256, 128), RenderSettings(), 64, 32)


def test_band_without_gaussians_is_empty(gpu_ctx):
    """A band no Gaussian reaches (band compaction leaves nothing to sort): black image,
    transmittance 1, no walks, no entries — as the same rows of the full render."""
    arrs = oracle_lib.random_cloud(77, 200, (1.0, 5.0, 0.05, 0.2, 0.9, 0.001, 0.005))  # |elevation| <= 0.05
    cloud = to_cloud32(arrs)
    cam = CameraPose(256, 128)
    s = RenderSettings()
    full = render(gpu_ctx, cloud, cam, s)
    fr = render_band(gpu_ctx, cloud, cam, s, 0, 16)
    assert fr.info().n_entries == 0
    assert np.array_equal(fr.image[:, :, 0:16], full.image[:, :, 0:16])
    assert np.all(fr.image[:, :, 0:16] == 0) and np.all(fr.transmittance[:, 0:16] == 1)
    assert np.all(fr.walked[:, 0:16] == 0)


def test_band_renders_write_peer_images(gpu_ctx):
    """odgs_frame_set_image_peers: every band render also writes its rows into the peer
    buffers, so after all bands each peer holds the full frame, bit for bit."""
    import torch
    from paper_2410_20686_b200 import RenderOutput
    c = scenes.cloud_c3(100_000)
    cam = CameraPose(1024, 512)
    s = RenderSettings()
    full = render(gpu_ctx, c, cam, s).image
    peers = [torch.full((3 * 1024 * 512,), float("nan"), device="cuda") for _ in range(2)]
    fr = RenderOutput(gpu_ctx)
    fr.set_image_peers([p.data_ptr() for p in peers])
    for r0 in range(0, 512, 128):
        render_band(gpu_ctx, c, cam, s, r0, r0 + 128, out=fr)
    torch.cuda.synchronize()
    for p in peers:
        assert np.array_equal(p.cpu().numpy().reshape(3, 1024, 512), full)
    fr.set_image_peers([])
    with pytest.raises(InvalidArgument):
        fr.set_image_peers([0] * 9)


def _ipc_child(handle, q):
    try:
        import torch
        from paper_2410_20686_b200 import Context, RenderOutput, RenderSettings, render_band, scenes
        from paper_2410_20686_b200.peers import ipc_open
        ctx = Context(0)
        ptr = ipc_open(ctx.lib, handle)
        fr = RenderOutput(ctx)
        fr.set_image_peers([ptr])
        render_band(ctx, scenes.cloud_c3(20_000), CameraPose(512, 256), RenderSettings(), 64, 192, out=fr)
        ctx.synchronize()
        fr.set_image_peers([])
        ctx.lib.odgs_ipc_close(__import__("ctypes").c_void_p(ptr))
        q.put("ok")
    except Exception as e:  # reported to the parent
        q.put(repr(e))


@pytest.mark.parametrize("pad", [0, 12345])
def test_band_written_into_another_process_buffer(gpu_ctx, pad):
    """CUDA IPC path of the fused band all-gather, two processes on one GPU: the child
    renders rows [64, 192) straight into the parent's buffer. pad > 0 exports a pointer
    inside a larger allocation (as a caching allocator hands out): the handle carries the
    offset, and the floats before it stay untouched."""
    import multiprocessing as mp
    import torch
    from paper_2410_20686_b200.peers import ipc_handle
    whole = torch.full((pad + 3 * 512 * 256,), -1.0, device="cuda")
    buf = whole[pad:]
    torch.cuda.synchronize()
    h = ipc_handle(gpu_ctx.lib, buf.data_ptr())
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    p = ctx_mp.Process(target=_ipc_child, args=(h, q))
    p.start()
    msg = q.get(timeout=300)
    p.join(timeout=60)
    assert msg == "ok", msg
    ref = render(gpu_ctx, scenes.cloud_c3(20_000), CameraPose(512, 256), RenderSettings()).image
    got = buf.cpu().numpy().reshape(3, 512, 256)
    assert np.array_equal(got[:, :, 64:192], ref[:, :, 64:192])
    assert np.all(got[:, :, :64] == -1.0) and np.all(got[:, :, 192:] == -1.0)
    assert np.all(whole[:pad].cpu().numpy() == -1.0)


def _gather_rank(rank, world, port, q):
    try:
        import os
        import torch
        import torch.distributed as dist
        from paper_2410_20686_b200 import Context, RenderOutput, RenderSettings, render_band, scenes
        from paper_2410_20686_b200.peers import BandGather
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        ctx = Context(0)
        fr = RenderOutput(ctx)
        W, H = 512, 256
        g = BandGather(ctx, fr, W, H, torch.device("cuda", 0))
        rows = H // world
        frames = []
        for k in range(3):  # consecutive frames alternate between the two image buffers
            g.begin()
            render_band(ctx, scenes.cloud_c3(20_000), scenes.yaw_camera(0.5 * k, W, H), RenderSettings(),
                        rank * rows, (rank + 1) * rows, out=fr)
            g.sync(0)
            frames.append(g.full.cpu().numpy())
        q.put((rank, frames))
        dist.barrier()
        g.close()
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, repr(e)))


def test_band_gather_two_ranks_on_one_gpu(gpu_ctx):
    """BandGather end to end with two ranks (gloo for the handle exchange, both on GPU 0):
    each renders half of the rows into both ranks' full images; both end up with the
    whole frame."""
    import multiprocessing as mp
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    procs = [ctx_mp.Process(target=_gather_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert not isinstance(res[r], str), res[r]
    for k in range(3):
        ref = render(gpu_ctx, scenes.cloud_c3(20_000), scenes.yaw_camera(0.5 * k, 512, 256), RenderSettings()).image
        for r in range(2):
            assert np.array_equal(res[r][k].reshape(3, 512, 256), ref), (r, k)


@pytest.mark.parametrize("tile,yaw", [(16, 0.0), (8, 0.7), (32, -1.3)])
def test_bands_bit_identical_sh3_and_tile_sizes(gpu_ctx, tile, yaw):
    # The fused band pass (pre-cull, survivor queues, segment compaction) on an SH
    # degree-3 cloud, a yawed camera and tile sizes other than 16.
    from paper_2410_20686_b200 import GaussianCloud
    arrs = oracle_lib.random_cloud(930 + tile, 20000)
    sh = np.random.default_rng(tile).normal(0, 0.05, (15, 3, 20000)).astype(np.float32)
    cloud = GaussianCloud.from_numpy(*arrs, sh_degree=3, sh_rest=sh)
    cam = scenes.yaw_camera(yaw, 512, 256)
    s = RenderSettings(tile_size=tile)
    full = render(gpu_ctx, cloud, cam, s)
    img, wk = full.image, full.walked
    rows = 256 // 4 if tile != 32 else 64
    for r0 in range(0, 256, rows):
        fr = render_band(gpu_ctx, cloud, cam, s, r0, r0 + rows)
        assert np.array_equal(fr.image[:, :, r0:r0 + rows], img[:, :, r0:r0 + rows])
        assert np.array_equal(fr.walked[:, r0:r0 + rows], wk[:, r0:r0 + rows])


def test_band_reports_non_finite_like_the_full_render(gpu_ctx):
    from paper_2410_20686_b200 import OdgsRuntimeError
    arrs = [np.array(a, dtype=np.float32) for a in oracle_lib.random_cloud(940, 5000)]
    arrs[0][1, 1234] = np.nan  # a NaN mean: the pre-cull must pass it to the exact path
    cloud = to_cloud32(arrs)
    cam, s = CameraPose(256, 128), RenderSettings()
    with pytest.raises(OdgsRuntimeError) as full_err:
        render(gpu_ctx, cloud, cam, s)
    with pytest.raises(OdgsRuntimeError) as band_err:
        render_band(gpu_ctx, cloud, cam, s, 64, 96)
    assert full_err.value.index == band_err.value.index == 1234


@pytest.mark.parametrize("field,row,col", [("raw_opacities", None, 4321), ("colors", 2, 4321),
                                           ("log_scales", 1, 4321), ("rotations", 3, 4321)])
@pytest.mark.parametrize("value", [np.nan, np.inf, -np.inf])
def test_band_checks_every_parameter_outside_the_band(gpu_ctx, field, row, col, value):
    """first_non_finite (rasterizer.hpp:133-136) covers every parameter of every row: a
    Gaussian far outside the band with a non-finite opacity, colour, single log-scale or
    quaternion component fails the band render exactly as it fails the full render."""
    from paper_2410_20686_b200 import OdgsRuntimeError
    arrs = [np.array(a, dtype=np.float32) for a in oracle_lib.random_cloud(941, 6000)]
    arrs[0][:, col] = [0.0, -5.0, 1.0]  # high above the horizon: never in the bottom band
    names = ["means", "rotations", "log_scales", "raw_opacities", "colors"]
    a = arrs[names.index(field)]
    if row is None:
        a[col] = value
    else:
        a[row, col] = value
    cloud = to_cloud32(arrs)
    cam, s = CameraPose(256, 128), RenderSettings()
    with pytest.raises(OdgsRuntimeError) as full_err:
        render(gpu_ctx, cloud, cam, s)
    with pytest.raises(OdgsRuntimeError) as band_err:
        render_band(gpu_ctx, cloud, cam, s, 96, 128)
    assert full_err.value.index == band_err.value.index == col


def test_band_checks_sh_coefficients_outside_the_band(gpu_ctx):
    from paper_2410_20686_b200 import GaussianCloud, OdgsRuntimeError
    arrs = [np.array(a, dtype=np.float32) for a in oracle_lib.random_cloud(942, 3000)]
    arrs[0][:, 77] = [0.0, -5.0, 1.0]
    sh = np.zeros((3, 3, 3000), np.float32)
    sh[2, 1, 77] = np.nan
    cloud = GaussianCloud.from_numpy(*arrs, sh_degree=1, sh_rest=sh)
    cam, s = CameraPose(256, 128), RenderSettings()
    with pytest.raises(OdgsRuntimeError) as band_err:
        render_band(gpu_ctx, cloud, cam, s, 96, 128)
    assert band_err.value.index == 77


@pytest.mark.parametrize("tile,plain", [(16, True), (32, False), (80, False)])
def test_peer_images_written_on_every_blend_path(gpu_ctx, tile, plain):
    """The fused band all-gather also runs in the un-culled blend (ODGS_FRAME_PLAIN_BLEND)
    and for tiles above 16 px, set before or after the flags."""
    import torch
    from paper_2410_20686_b200 import RenderOutput
    from paper_2410_20686_b200 import _capi as capi
    c = scenes.cloud_c3(30_000)
    W, H = 640, 320
    cam = CameraPose(W, H)
    s = RenderSettings(tile_size=tile)
    full = render(gpu_ctx, c, cam, s).image
    peer = torch.full((3 * W * H,), float("nan"), device="cuda")
    fr = RenderOutput(gpu_ctx)
    fr.set_image_peers([peer.data_ptr()])
    if plain:
        gpu_ctx.lib.odgs_frame_set_flags(fr.handle, capi.FRAME_PLAIN_BLEND)
    rows = 160 if tile == 80 else tile * (160 // tile)
    for r0 in range(0, H, rows):
        render_band(gpu_ctx, c, cam, s, r0, min(H, r0 + rows), out=fr)
    torch.cuda.synchronize()
    assert np.array_equal(peer.cpu().numpy().reshape(3, W, H), full)

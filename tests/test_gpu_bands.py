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

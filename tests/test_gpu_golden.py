"""GPU vs the committed golden fixtures (tests/golden/*.npz, made by make_golden.py from
the oracle): walk lengths, tile CSR, tile entries and image bit-exact against the
PortableMath outputs; image within 1e-4 of the libm (StdMath) outputs."""
from pathlib import Path

import numpy as np
import pytest

from paper_2410_20686_b200 import CameraPose, GaussianCloud, RenderSettings, render

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("path", sorted(GOLDEN.glob("*.npz")), ids=lambda p: p.stem)
def test_gpu_reproduces_golden(gpu_ctx, path):
    g = np.load(path)
    cloud = GaussianCloud.from_numpy(g["means"], g["rotations"], g["log_scales"], g["raw_opacities"], g["colors"])
    W, H = int(g["width"]), int(g["height"])
    s = [float(x) for x in g["settings"]]
    settings = RenderSettings(near_radius=s[0], far_radius=s[1], tile_size=int(s[2]), alpha_clamp=s[3],
                              transmittance_floor=s[4], cutoff_sigma=s[5], lowpass_dilation=s[6],
                              max_elevation=s[7])
    fr = render(gpu_ctx, cloud, CameraPose(W, H, g["rotation"], g["translation"]), settings)
    assert np.array_equal(fr.walked.ravel(), g["walked_portable"])
    assert np.array_equal(fr.tile_offsets, g["tile_offsets_portable"])
    assert np.array_equal(fr.tile_entries, g["tile_entries_portable"])
    assert np.array_equal(fr.image.ravel(), g["image_portable"])
    assert np.abs(fr.image.ravel() - g["image_std"]).max() <= 1e-4

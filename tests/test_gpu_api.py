"""The rest of the reference's hot-path API through the C ABI: project_gaussian
(projection.hpp:178-216) and grad_pixels_to_splats (backward.hpp:208-339), against the
oracle restatement."""
import numpy as np
import pytest

import oracle_lib
from helpers import cam32, settings_pair, to_cloud32
from paper_2410_20686_b200 import (CameraPose, DomainError, InvalidArgument, grad_pixels_to_splats,
                                   project_gaussian, render, scenes)

pytestmark = pytest.mark.gpu


def test_project_gaussian_matches_the_splats_of_render(gpu_ctx):
    """Every row: None exactly where the oracle culls, otherwise the oracle's Splat2D bit for bit."""
    arrs = oracle_lib.random_cloud(610, 600)
    cam = scenes.yaw_camera(0.9, 512, 256, (0.1, 0.0, -0.2))
    gs, os_ = settings_pair()
    r, t = cam32(cam)
    of = oracle_lib.render(arrs, r, t, cam.width, cam.height, os_, portable=True)
    idx = of.get("splat_index")
    mean, inv, cov = of.get("splat_mean").reshape(-1, 2), of.get("splat_inv").reshape(-1, 4), of.get(
        "splat_cov2d").reshape(-1, 4)
    depth, radius, opac = of.get("splat_depth"), of.get("splat_radius"), of.get("splat_opacity")
    col, clamped = of.get("splat_color").reshape(-1, 3), of.get("splat_clamped")
    cloud = to_cloud32(arrs)
    pos = {int(i): k for k, i in enumerate(idx)}
    for i in range(600):
        sp = project_gaussian(gpu_ctx, cloud, i, cam, gs)
        if i not in pos:
            assert sp is None, i
            continue
        k = pos[i]
        assert sp is not None and sp.index == i
        f = np.float32
        assert np.array_equal(sp.pixel_mean, mean[k].astype(f))
        assert np.array_equal(sp.cov2d_inv.ravel(), inv[k].astype(f))
        assert np.array_equal(sp.cov2d.ravel(), cov[k].astype(f))
        assert (sp.depth, sp.radius, sp.opacity) == (f(depth[k]), f(radius[k]), f(opac[k]))
        assert np.array_equal(sp.color, col[k].astype(f))
        assert sp.pole_clamped == bool(clamped[k])


def test_project_gaussian_errors_as_the_reference(gpu_ctx):
    arrs = [np.array(a) for a in oracle_lib.random_cloud(611, 4)]
    arrs[1][:, 1] = 0.0                      # near-zero quaternion (covariance.hpp:14-15)
    arrs[2][0, 2] = np.inf                   # non-finite log-scale (covariance.hpp:31-32)
    arrs[0][:, 3] = [np.nan, 0.0, 1.0]       # NaN depth: outside the shell, no throw
    cloud = to_cloud32(arrs)
    cam = CameraPose(256, 128)
    gs, _ = settings_pair()
    assert project_gaussian(gpu_ctx, cloud, 0, cam, gs) is not None
    with pytest.raises(InvalidArgument):
        project_gaussian(gpu_ctx, cloud, 1, cam, gs)
    with pytest.raises(InvalidArgument):
        project_gaussian(gpu_ctx, cloud, 2, cam, gs)
    assert project_gaussian(gpu_ctx, cloud, 3, cam, gs) is None
    with pytest.raises(InvalidArgument):
        project_gaussian(gpu_ctx, cloud, 4, cam, gs)
    gs_near0, _ = settings_pair(near_radius=0.0)
    z = [np.array(a) for a in oracle_lib.random_cloud(612, 1)]
    z[0][:, 0] = 0.0                         # at the camera centre: to_spherical's domain error
    with pytest.raises(DomainError):
        project_gaussian(gpu_ctx, to_cloud32(z), 0, cam, gs_near0)


@pytest.mark.parametrize("cutoff", [3.0, 8.0])
def test_grad_pixels_to_splats_matches_oracle(gpu_ctx, cutoff):
    arrs = oracle_lib.random_cloud(613, 3000)
    W, H = 512, 256
    cam = CameraPose(W, H)
    gs, os_ = settings_pair(cutoff_sigma=cutoff)
    fr = render(gpu_ctx, to_cloud32(arrs), cam, gs)
    dl = np.random.default_rng(5).uniform(-1, 1, (3, W, H)).astype(np.float32)
    sg = grad_pixels_to_splats(gpu_ctx, fr, dl, gs)
    r, t = cam32(cam)
    of = oracle_lib.render(arrs, r, t, W, H, os_, portable=True)
    of.backward(dl.astype(np.float64))
    rel = lambda a, b: np.abs(a.ravel() - b.ravel()).max() / max(np.abs(a).max(), np.abs(b).max(), 1e-12)
    assert rel(sg.pixel_mean, of.get("sg_mean")) < 1e-3
    assert rel(sg.cov2d, of.get("sg_cov2d")) < 1e-3
    assert rel(sg.opacity, of.get("sg_opacity")) < 1e-3
    assert rel(sg.color, of.get("sg_color")) < 1e-3

"""init_from_points on the GPU (reference io.cpp:259-297) against
the brute-force oracle restatement (oracle::init_scales_brute) and the reference's own
test_io.cpp cases. The per-point mean neighbour distance must be bit-identical (same
binary64 distances, same ascending sum); the log-scale is CUDA's log of that value,
within 1 ulp of glibc's."""
import math

import numpy as np
import pytest

import oracle_lib
from paper_2410_20686_b200 import io
from paper_2410_20686_b200.rasterizer import InvalidArgument

pytestmark = pytest.mark.gpu


def run(ctx, pos, col=None):
    pos = np.ascontiguousarray(pos, np.float64)
    n = pos.shape[1]
    col = np.full((3, n), 0.5) if col is None else col
    return io.init_from_points(ctx, io.PointCloud(pos, col), return_scale=True)


def check_against_oracle(ctx, pos):
    cloud, scale = run(ctx, pos)
    o_scale, o_ls = oracle_lib.init_scales(pos)
    assert np.array_equal(scale, o_scale), np.flatnonzero(scale != o_scale)[:10]
    ulp = np.abs(cloud.log_scales - o_ls[None]) / np.spacing(np.abs(o_ls))[None]
    assert ulp.max() <= 1.0
    assert np.array_equal(cloud.log_scales[0], cloud.log_scales[1]) and np.array_equal(cloud.log_scales[0],
                                                                                       cloud.log_scales[2])
    return cloud, scale


def test_one_point_gets_the_fallback_scale(gpu_ctx):  # test_io.cpp:71-92
    cloud, scale = run(gpu_ctx, np.zeros((3, 1)), np.ones((3, 1)))
    assert np.array_equal(cloud.colors[:, 0], [1, 1, 1])
    assert cloud.raw_opacities[0] == pytest.approx(math.log(0.1 / 0.9), rel=1e-15)
    assert np.array_equal(cloud.rotations[:, 0], [1, 0, 0, 0])
    assert scale[0] == 0.1
    assert cloud.log_scales[0, 0] == pytest.approx(math.log(0.1), rel=1e-15)


def test_neighbor_distances_set_the_initial_scales(gpu_ctx):  # test_io.cpp:94-110
    d = 0.3
    pos = np.array([[0, d, 2 * d], [0, 0, 0], [0, 0, 0]], np.float64)
    cloud, _ = check_against_oracle(gpu_ctx, pos)
    assert cloud.log_scales[0, 0] == pytest.approx(math.log(1.5 * d), rel=1e-12)
    assert cloud.log_scales[1, 1] == pytest.approx(math.log(d), rel=1e-12)
    assert cloud.log_scales[2, 2] == pytest.approx(math.log(1.5 * d), rel=1e-12)


def test_degenerate_clusters_floor_the_initial_scale(gpu_ctx):  # test_io.cpp:112-118
    cloud, scale = check_against_oracle(gpu_ctx, np.zeros((3, 4)))
    assert np.all(scale == 1e-7)
    assert cloud.log_scales[0, 0] == pytest.approx(math.log(1e-7), rel=1e-12)


def test_no_points_is_an_invalid_argument(gpu_ctx):  # io.cpp:260
    with pytest.raises(InvalidArgument, match="no points"):
        run(gpu_ctx, np.zeros((3, 0)))


@pytest.mark.parametrize("kind", ["uniform", "clustered", "planar", "duplicates", "nonfinite", "two", "wide"])
def test_matches_brute_force(gpu_ctx, kind):
    r = np.random.default_rng(hash(kind) % 2**32)
    n = 6000
    if kind == "uniform":
        pos = r.uniform(-5, 5, (3, n))
    elif kind == "clustered":  # dense blobs + sparse background (SfM-like)
        centres = r.uniform(-10, 10, (3, 12))
        pos = np.concatenate([centres[:, r.integers(0, 12, n - 300)] + r.normal(0, 0.02, (3, n - 300)),
                              r.uniform(-20, 20, (3, 300))], axis=1)
    elif kind == "planar":
        pos = np.stack([r.uniform(-3, 3, n), r.uniform(-3, 3, n), np.zeros(n)])
    elif kind == "duplicates":
        base = r.uniform(-1, 1, (3, n // 3))
        pos = np.concatenate([base, base, base[:, : n - 2 * (n // 3)]], axis=1)
    elif kind == "nonfinite":
        pos = r.uniform(-2, 2, (3, n))
        pos[0, 5] = np.nan
        pos[1, 77] = np.inf
        pos[2, 999] = -np.inf
    elif kind == "two":
        pos = r.uniform(-1, 1, (3, 2))
    else:  # widely spread scales: 1e-6 .. 1e6
        pos = r.standard_normal((3, n)) * 10.0 ** r.uniform(-6, 6, n)[None]
    check_against_oracle(gpu_ctx, pos)


def test_large_cloud_subset_is_exact(gpu_ctx):
    """2M points: every sampled point's scale equals a binary64 brute force over all points."""
    r = np.random.default_rng(4)
    n = 2_000_000
    pos = np.concatenate([r.uniform(-50, 50, (3, n // 2)),
                          r.normal(0, 0.5, (3, n // 2)) + r.uniform(-40, 40, (3, 1))], axis=1)
    _, scale = run(gpu_ctx, pos)
    for i in r.choice(n, 48, replace=False):
        d = pos - pos[:, i:i + 1]
        d2 = d[0] * d[0] + (d[1] * d[1] + d[2] * d[2])
        d2[i] = np.inf
        best = np.sort(np.partition(d2, 3)[:3])
        s = 0.0
        for v in best:
            s += math.sqrt(v)
        assert scale[i] == max(s / 3, 1e-7), i

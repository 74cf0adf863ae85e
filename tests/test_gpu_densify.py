"""GPU density control vs the oracle restatement (reference densify.hpp:81-166):
densify_and_prune and reset_opacity bit-exact against densify_and_prune<float,
PortableMath> on the same seeded inputs (stats, every parameter and moment row, the
generator's position afterwards), the reference's own test_densify.cpp cases, edge
cases (empty, nothing to do, everything pruned, bad configs, degenerate split
quaternion) and a 1M-Gaussian run with its row-count identity."""
import math

import numpy as np
import pytest
import torch

import oracle_lib as O
from paper_2410_20686_b200 import (DensifyConfig, GaussianCloud, InvalidArgument, Rng, TrainState,
                                   densify_and_prune, reset_opacity)
from paper_2410_20686_b200.densify import MOMENTS, PARAMS

pytestmark = pytest.mark.gpu
f32 = np.float32


def make_case(n, seed, extent_scale=1.0, low_frac=0.1, moments=True):
    rs = np.random.default_rng(seed)
    means, rot, ls, op, col = O.random_cloud(seed, n)
    op = op.copy()
    op[rs.random(n) < low_frac] = -6.0  # sigmoid(-6) = 0.0025 < 0.005
    params = {"means": means, "rotations": rot, "log_scales": ls, "raw_opacities": op, "colors": col}
    params = {k: v.astype(f32) for k, v in params.items()}
    mom = {k: (rs.standard_normal((w, n) if w > 1 else n).astype(f32) if moments else
               np.zeros((w, n) if w > 1 else n, f32)) for k, w in MOMENTS}
    count = rs.integers(0, 5, n).astype(np.int32)
    ga = (rs.random(n) * 2e-4 * count).astype(f32)
    ea = (rs.random(n) * count).astype(f32)
    return params, mom, ga, ea, count


def to_device(params, mom, ga, ea, count):
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    cloud = GaussianCloud(*[d(params[k]) for k, _ in PARAMS])
    st = TrainState(len(count), "cuda")
    for k, _ in MOMENTS:
        setattr(st, k, d(mom[k]))
    st.grad_accum, st.elev_accum, st.grad_count = d(ga), d(ea), d(count)
    return cloud, st


CFG_TUPLE = lambda c: (c.grad_threshold_min, c.grad_threshold_max, c.percent_dense, c.opacity_prune_floor,
                       c.split_scale_divisor)


def run_both(gpu_ctx, case, cfg, extent, seed):
    params, mom, ga, ea, count = case
    want_p, want_m, want_stats, want_next = O.densify(params, mom, ga, ea, count, CFG_TUPLE(cfg), extent, seed)
    cloud, st = to_device(*case)
    rng = Rng(seed)
    stats = densify_and_prune(gpu_ctx, cloud, st, cfg, extent, rng)
    return (want_p, want_m, want_stats, want_next), (cloud, st, stats, rng)


def assert_bit_exact(want, got):
    want_p, want_m, want_stats, want_next = want
    cloud, st, stats, rng = got
    assert (stats.cloned, stats.split, stats.pruned) == want_stats
    m = cloud.n
    assert m == want_p["raw_opacities"].shape[0]
    for k, _ in PARAMS:
        g = getattr(cloud, k).cpu().numpy()
        assert np.array_equal(g.view(np.uint32), want_p[k].astype(f32).view(np.uint32)), k
    for k, _ in MOMENTS:
        g = getattr(st, k).cpu().numpy()
        assert np.array_equal(g.view(np.uint32), want_m[k].astype(f32).view(np.uint32)), k
    assert int(st.grad_count.abs().sum()) == 0
    assert float(st.grad_accum.abs().sum()) == 0 and float(st.elev_accum.abs().sum()) == 0
    assert rng.next() == want_next


@pytest.mark.parametrize("seed,n,extent", [(1, 2000, 60.0), (2, 20000, 60.0), (3, 5000, 8.0), (4, 5000, 400.0)])
def test_densify_bit_exact_vs_oracle(gpu_ctx, seed, n, extent):
    case = make_case(n, seed)
    want, got = run_both(gpu_ctx, case, DensifyConfig(), extent, seed + 100)
    assert want[2][0] + want[2][1] > 0  # something densified
    assert_bit_exact(want, got)


def test_densify_custom_config_bit_exact(gpu_ctx):
    cfg = DensifyConfig(grad_threshold_min=1e-5, grad_threshold_max=5e-5, percent_dense=0.01,
                        opacity_prune_floor=0.02, split_scale_divisor=2.5)
    case = make_case(8000, 11, low_frac=0.2)
    want, got = run_both(gpu_ctx, case, cfg, 3.0, 7)
    assert_bit_exact(want, got)


def test_densify_one_million_rows(gpu_ctx):
    n = 1_000_000
    case = make_case(n, 21, moments=False)
    want, got = run_both(gpu_ctx, case, DensifyConfig(), 60.0, 5)
    cloned, split, pruned = got[2].cloned, got[2].split, got[2].pruned
    assert got[0].n == n + cloned + split - pruned  # +1 per clone, +2-1 per split
    assert_bit_exact(want, got)


def marker_case(n):  # test_densify.cpp:14-24 in float
    params = {"means": np.stack([np.arange(n), 0.5 * np.arange(n), 2.0 + np.arange(n)]).astype(f32),
              "rotations": np.vstack([np.ones(n), np.zeros((3, n))]).astype(f32),
              "log_scales": np.full((3, n), math.log(0.05), f32),
              "raw_opacities": np.zeros(n, f32),  # logit(0.5)
              "colors": np.tile(0.1 * (np.arange(n) + 1), (3, 1)).astype(f32)}
    mom = {k: np.zeros((w, n) if w > 1 else n, f32) for k, w in MOMENTS}
    return params, mom, np.zeros(n, f32), np.zeros(n, f32), np.zeros(n, np.int32)


def set_window(case, i, mean_grad, elevation, count=2):  # test_densify.cpp:28-34
    case[4][i] = count
    case[2][i] = f32(mean_grad * count)
    case[3][i] = f32((1.0 - math.cos(elevation)) * count)


def test_reference_cases(gpu_ctx):  # test_densify.cpp:76-195 on the GPU
    cfg, extent = DensifyConfig(), 100.0
    # zero gradients leave the cloud untouched
    case = marker_case(4)
    for i in range(4):
        set_window(case, i, 0.0, 0.3)
    cloud, st = to_device(*case)
    s = densify_and_prune(gpu_ctx, cloud, st, cfg, extent, Rng(41))
    assert (s.cloned, s.split, s.pruned) == (0, 0, 0) and cloud.n == 4
    assert np.array_equal(cloud.means.cpu().numpy(), case[0]["means"])
    # equatorial Gaussian over threshold and small: cloned, exact copy appended
    case = marker_case(3)
    set_window(case, 0, 5e-5, 0.0)
    cloud, st = to_device(*case)
    s = densify_and_prune(gpu_ctx, cloud, st, cfg, extent, Rng(41))
    assert s.cloned == 1 and cloud.n == 4
    for k, _ in PARAMS:
        a = getattr(cloud, k).cpu().numpy()
        assert np.array_equal(a[..., 3], a[..., 0]), k
    # the same gradient observed only near the pole: blocked
    case = marker_case(3)
    set_window(case, 0, 5e-5, math.pi / 2)
    cloud, st = to_device(*case)
    s = densify_and_prune(gpu_ctx, cloud, st, cfg, extent, Rng(41))
    assert (s.cloned, s.split) == (0, 0) and cloud.n == 3
    # large Gaussian: split into two shrunken children inside the parent's 1-sigma ellipsoid
    case = marker_case(2)
    case[0]["log_scales"][:, 0] = f32(math.log(0.5))
    q = np.array([0.8, 0.1, -0.3, 0.2], f32)
    case[0]["rotations"][:, 0] = q
    set_window(case, 0, 5e-5, 0.0)
    cloud, st = to_device(*case)
    s = densify_and_prune(gpu_ctx, cloud, st, cfg, extent, Rng(41))
    assert s.split == 1 and cloud.n == 3
    qn = q.astype(np.float64) / np.linalg.norm(q.astype(np.float64))
    w, x, y, z = qn
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    means = cloud.means.cpu().numpy().astype(np.float64)
    for child in (1, 2):
        assert cloud.raw_opacities[child].item() == case[0]["raw_opacities"][0]
        scale = np.exp(cloud.log_scales[:, child].cpu().numpy().astype(np.float64))
        assert np.abs(scale * 1.6 - 0.5).max() < 1e-6
        assert np.array_equal(cloud.rotations[:, child].cpu().numpy(), q)
        local = (R.T @ (means[:, child] - case[0]["means"][:, 0])) / 0.5
        assert np.linalg.norm(local) <= 1.0 + 1e-6
    # transparent Gaussians are pruned and moments follow the survivors
    case = marker_case(4)
    case[0]["raw_opacities"][1] = f32(math.log(0.004 / 0.996))
    case[1]["means_m"][:, 3] = 7.0
    cloud, st = to_device(*case)
    s = densify_and_prune(gpu_ctx, cloud, st, cfg, extent, Rng(41))
    assert s.pruned == 1 and cloud.n == 3
    assert cloud.colors[0, 1].item() == pytest.approx(0.3)
    assert st.means_m[0, 2].item() == 7.0 and st.n == 3


def test_lower_thresholds_densify_a_superset(gpu_ctx):  # test_densify.cpp:165-194
    n = 12
    elev = np.random.default_rng(43).uniform(0, math.pi / 2, n)

    def run(cfg):
        case = marker_case(n)
        for i in range(n):
            set_window(case, i, 4e-5, elev[i])
        cloud, st = to_device(*case)
        densify_and_prune(gpu_ctx, cloud, st, cfg, 100.0, Rng(47))
        return cloud.n

    strict = run(DensifyConfig())
    loose = run(DensifyConfig(grad_threshold_min=1e-5, grad_threshold_max=5e-5))
    assert loose >= strict and loose > n


def test_edge_cases(gpu_ctx):
    # empty cloud
    case = marker_case(0)
    cloud, st = to_device(*case)
    s = densify_and_prune(gpu_ctx, cloud, st, DensifyConfig(), 10.0, Rng(1))
    assert cloud.n == 0 and (s.cloned, s.split, s.pruned) == (0, 0, 0)
    # everything pruned (clones and split children too)
    case = make_case(3000, 5, low_frac=1.01)
    want, got = run_both(gpu_ctx, case, DensifyConfig(), 60.0, 3)
    assert got[0].n == 0
    assert_bit_exact(want, got)
    # invalid configuration / extent (densify.hpp:26-32, 87-88)
    case = marker_case(3)
    cloud, st = to_device(*case)
    with pytest.raises(InvalidArgument):
        densify_and_prune(gpu_ctx, cloud, st, DensifyConfig(grad_threshold_min=2e-4), 10.0, Rng(1))
    with pytest.raises(InvalidArgument):
        densify_and_prune(gpu_ctx, cloud, st, DensifyConfig(), 0.0, Rng(1))
    with pytest.raises(ValueError):  # the raw ABI performs the same check
        import ctypes as C
        from paper_2410_20686_b200 import _capi as capi
        from paper_2410_20686_b200.densify import params_of
        bad = capi.DensifyConfig(2e-5, 1e-4, 1.5, 0.005, 1.6)
        stats = capi.DensifyStats()
        gpu_ctx.check(gpu_ctx.lib.odgs_densify_plan(gpu_ctx.handle, C.byref(params_of(cloud)), C.byref(st.to_c()),
                                                    C.byref(bad), 10.0, C.byref(stats)))
    # a split parent with a zero quaternion: normalize_quaternion throws, cloud untouched
    case = marker_case(5)
    case[0]["log_scales"][:, 3] = f32(math.log(0.5))
    case[0]["rotations"][:, 3] = 0.0
    set_window(case, 3, 5e-5, 0.0)
    cloud, st = to_device(*case)
    with pytest.raises(InvalidArgument) as e:
        densify_and_prune(gpu_ctx, cloud, st, DensifyConfig(), 100.0, Rng(1))
    assert e.value.index == 3
    assert cloud.n == 5


def test_reset_opacity_bit_exact(gpu_ctx):
    rs = np.random.default_rng(3)
    raw = rs.uniform(-12, 12, 100_000).astype(f32)
    raw[:3] = [math.log(0.8 / 0.2), math.log(0.006 / 0.994), 0.0]
    want = O.reset_opacity(raw.astype(np.float64), 0.01)
    case = marker_case(raw.shape[0])
    case[0]["raw_opacities"][:] = raw
    case[1]["opac_m"][:] = 0.5
    case[1]["opac_v"][:] = 0.25
    cloud, st = to_device(*case)
    reset_opacity(gpu_ctx, cloud, st)
    got = cloud.raw_opacities.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.astype(f32).view(np.uint32))
    op = 1 / (1 + np.exp(-got[:3].astype(np.float64)))
    assert op[0] == pytest.approx(0.01, rel=1e-6) and op[1] == pytest.approx(0.006, rel=1e-6)
    assert float(st.opac_m.abs().sum()) == 0 and float(st.opac_v.abs().sum()) == 0
    # a custom ceiling
    want2 = O.reset_opacity(raw.astype(np.float64), 0.3)
    cloud2, st2 = to_device(*case)
    reset_opacity(gpu_ctx, cloud2, st2, 0.3)
    assert np.array_equal(cloud2.raw_opacities.cpu().numpy().view(np.uint32), want2.astype(f32).view(np.uint32))


def test_reset_opacity_throw_point(gpu_ctx):
    # sigmoid(-200) == 0 in float: logit(0) throws at row 5; rows before are rewritten,
    # later rows and the moments are untouched (the reference's sequential loop).
    raw = np.full(10, 2.0, f32)
    raw[5] = -200.0
    case = marker_case(10)
    case[0]["raw_opacities"][:] = raw
    case[1]["opac_m"][:] = 0.5
    cloud, st = to_device(*case)
    with pytest.raises(InvalidArgument) as e:
        reset_opacity(gpu_ctx, cloud, st)
    assert e.value.index == 5
    got = cloud.raw_opacities.cpu().numpy()
    want = O.reset_opacity(np.full(5, 2.0), 0.01).astype(f32)
    assert np.array_equal(got[:5], want)
    assert np.array_equal(got[5:], raw[5:])
    assert float(st.opac_m.min()) == 0.5
    with pytest.raises(O.OracleError):
        O.reset_opacity(raw.astype(np.float64))


def test_trainer_runs_the_density_schedule(gpu_ctx):
    """optimizer.hpp:144-153: densify every `densify_interval` steps up to
    `densify_until`, opacity reset every `opacity_reset_interval`; the trainer's
    gradient buffers follow the new row count and the window restarts."""
    from helpers import to_cloud32
    from paper_2410_20686_b200 import CameraPose, RenderSettings, render
    from paper_2410_20686_b200.train import TrainConfig, ViewShardedTrainer
    host = to_cloud32(O.random_cloud(301, 3000))
    cloud = GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(getattr(host, k))).cuda() for k, _ in PARAMS])
    W, H = 256, 128
    views = [CameraPose(W, H), CameraPose(W, H, np.eye(3), [0.1, 0.0, -0.2])]
    tgt = [torch.from_numpy(render(gpu_ctx, to_cloud32(O.random_cloud(302, 3000)), v, RenderSettings())
                            .image.ravel()).cuda() for v in views]
    d = DensifyConfig(grad_threshold_min=1e-9, grad_threshold_max=1e-8, densify_interval=2, densify_until=4,
                      opacity_reset_interval=4)
    tr = ViewShardedTrainer(gpu_ctx, cloud, views, tgt, RenderSettings(), TrainConfig(lambda_ssim=0.2, densify=d),
                            extent=10.0)
    sizes = []
    for step in range(1, 7):
        n_before = tr.cloud.n
        loss = tr.step()
        assert math.isfinite(loss)
        s = tr.last_densify
        if step in (2, 4):
            assert s is not None and s.cloned + s.split > 0
            assert tr.cloud.n == n_before + s.cloned + s.split - s.pruned
            assert tr.flat.numel() == 16 * tr.cloud.n and int(tr.state.grad_count.sum()) == 0
        else:
            assert s is None and tr.cloud.n == n_before
        sizes.append(tr.cloud.n)
    assert sizes[-1] > 3000
    # step 4 reset every opacity to <= 0.01 before steps 5-6 moved them again
    assert tr.state.opac_m.shape[0] == tr.cloud.n

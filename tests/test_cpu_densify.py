"""CPU checks of the host half of density control (densify.hpp): the library's
std::mt19937 unit-ball stream replays the oracle's (= the reference's) draws exactly,
dynamic_threshold matches, and the Python mirror validates configs like the reference.
No device work."""
import math

import numpy as np
import pytest

import oracle_lib as O
from paper_2410_20686_b200 import DensifyConfig, DomainError, InvalidArgument, Rng, dynamic_threshold
from paper_2410_20686_b200 import _capi as capi


@pytest.mark.parametrize("seed", [41, 47, 5489, 2024])
def test_unit_ball_stream_replays_the_reference_draws(seed):
    want, want_next = O.unit_ball(seed, 5000)
    r = Rng(seed)
    got = r.unit_ball(5000)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert r.next() == want_next  # same number of raw draws consumed
    n = np.sqrt(got[:, 0].astype(np.float64) ** 2 + got[:, 1] ** 2 + got[:, 2] ** 2)
    assert n.max() <= 1.0 + 1e-6


def test_unit_ball_chunks_concatenate():
    a = Rng(9)
    whole = a.unit_ball(300)
    b = Rng(9)
    parts = np.concatenate([b.unit_ball(k) for k in (1, 0, 99, 200)])
    assert np.array_equal(whole, parts)


def test_dynamic_threshold_matches_oracle_and_reference_cases():  # test_densify.cpp:37-74
    cfg = DensifyConfig()
    assert dynamic_threshold(0.0, cfg) == 2e-5
    assert dynamic_threshold(math.pi / 2, cfg) == 1e-4
    assert dynamic_threshold(-math.pi / 2, cfg) == 1e-4
    assert dynamic_threshold(math.pi / 3, cfg) == pytest.approx(6e-5, rel=1e-12)
    for k in range(0, 1000, 7):
        th = (math.pi / 2) * k / 999.0
        assert dynamic_threshold(th, cfg) == O.dynamic_threshold(th)
        assert dynamic_threshold(-th, cfg) == dynamic_threshold(th, cfg)
    with pytest.raises(DomainError):
        dynamic_threshold(1.8, cfg)


def test_config_validation():
    DensifyConfig().validate()
    with pytest.raises(InvalidArgument):
        DensifyConfig(grad_threshold_min=2e-4).validate()
    with pytest.raises(InvalidArgument):
        DensifyConfig(percent_dense=0.0).validate()
    c = capi.DensifyConfig()
    capi.load_library().odgs_default_densify_config(c)
    d = DensifyConfig()
    assert (c.grad_threshold_min, c.grad_threshold_max, c.percent_dense, c.opacity_prune_floor,
            c.split_scale_divisor) == (d.grad_threshold_min, d.grad_threshold_max, d.percent_dense,
                                       d.opacity_prune_floor, d.split_scale_divisor)

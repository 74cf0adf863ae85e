"""CPU checks of the checker itself: the oracle restatement passes the reference's
own hot-path tests (ported), the portable math agrees with libm, and the committed
golden fixtures still reproduce."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle_lib

GOLDEN = Path(__file__).resolve().parent / "golden"


def test_ported_reference_suites_pass_on_the_oracle():
    oracle_lib.build()
    r = subprocess.run([str(oracle_lib.REF_TESTS)], capture_output=True, text=True, timeout=600)
    tail = "\n".join(r.stdout.splitlines()[-15:])
    assert r.returncode == 0, r.stdout[-4000:]
    assert " 0 failures" in tail


@pytest.mark.parametrize("path", sorted(GOLDEN.glob("*.npz")), ids=lambda p: p.stem)
def test_golden_fixture_reproduces(path):
    g = np.load(path)
    cloud = tuple(g[k].astype(np.float64) for k in ("means", "rotations", "log_scales", "raw_opacities", "colors"))
    W, H = int(g["width"]), int(g["height"])
    s = oracle_lib.OracleSettings(*[float(x) for x in g["settings"]])
    s.tile = int(s.tile)
    for portable in (False, True):
        fr = oracle_lib.render(cloud, g["rotation"], g["translation"], W, H, s, portable=portable)
        tag = "portable" if portable else "std"
        assert np.array_equal(fr.get("walked"), g[f"walked_{tag}"])
        assert np.array_equal(fr.get("tile_offsets"), g[f"tile_offsets_{tag}"])
        assert np.array_equal(fr.get("tile_entries"), g[f"tile_entries_{tag}"])
        assert np.array_equal(fr.get("image").astype(np.float32), g[f"image_{tag}"])


def test_random_cloud_generator_matches_reference_bounds():
    means, rot, ls, op, col = oracle_lib.random_cloud(77, 1000)
    r = np.linalg.norm(means, axis=0)
    assert r.min() >= 0.5 - 1e-5 and r.max() <= 20 + 1e-4
    assert np.allclose(np.linalg.norm(rot, axis=0), 1, atol=1e-6)
    assert col.min() >= 0.05 - 1e-6 and col.max() <= 0.95 + 1e-6

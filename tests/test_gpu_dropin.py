"""The C++ drop-in header (include/odgs_b200.hpp) used with reference-shaped types."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
HERE = Path(__file__).resolve().parent / "cpp"


def test_cpp_dropin():
    subprocess.run(["make", "-C", str(HERE)], check=True, capture_output=True)
    r = subprocess.run([str(HERE / "dropin_test")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout

"""CPU checks of the drop-in boundary: the C-ABI library loads and exports every
symbol include/odgs_b200.h declares; host-side defaults mirror RenderSettings
(types.hpp:229-255). No compute calls (there is no GPU here)."""
import ctypes
import re
from pathlib import Path

import numpy as np

from paper_2410_20686_b200 import RenderSettings
from paper_2410_20686_b200 import _capi as capi

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "odgs_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(odgs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = capi.load_library()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(capi.SIGNATURES), set(syms) ^ set(capi.SIGNATURES)


def test_abi_version_and_defaults():
    lib = capi.load_library()
    assert lib.odgs_abi_version() == 1
    s = lib.odgs_default_settings()
    r = RenderSettings()
    assert s.tile_size == 16 == r.tile_size
    for k in ("near_radius", "far_radius", "alpha_clamp", "transmittance_floor", "cutoff_sigma",
              "lowpass_dilation", "max_elevation"):
        assert np.float32(getattr(s, k)) == np.float32(getattr(r, k)), k
    # max_elevation = 85 deg in float, as RenderSettings<float> computes it
    assert np.float32(s.max_elevation) == np.float32(np.float32(85) * np.float32(np.pi) / np.float32(180))


def test_struct_layouts_match_header():
    assert ctypes.sizeof(capi.Settings) == 36
    assert ctypes.sizeof(capi.Camera) == 56
    assert ctypes.sizeof(capi.Cloud) == 64
    assert ctypes.sizeof(capi.FrameInfo) == 56

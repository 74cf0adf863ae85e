"""Generates the golden fixtures in tests/golden/ from the CPU oracle.

Each fixture holds a small seeded scene (cloud in float32, camera, settings) and the
oracle's outputs for it with StdMath (literal libm) and PortableMath: walk lengths,
tile CSR, tile entries and the float image. They pin the oracle (tests/test_cpu_oracle.py)
and are the bit-exact targets of the GPU (tests/test_gpu_golden.py). Run:
    python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import oracle_lib  # noqa: E402

CASES = {
    # name: (seed, n, width, height, rotation, translation, settings)
    "ref77_100_256x128": (77, 100, 256, 128, np.eye(3), np.zeros(3), oracle_lib.OracleSettings()),
    "seed404_300_tile8_cutoff8": (404, 300, 256, 128, np.eye(3), np.zeros(3),
                                  oracle_lib.OracleSettings(tile=8, cutoff=8.0)),
    "seed505_500_pitched_512x256": (505, 500, 512, 256,
                                    np.array([[0.8775826, -0.4794255, 0.0], [0.4794255, 0.8775826, 0.0],
                                              [0.0, 0.0, 1.0]]),
                                    np.array([0.2, -0.1, 0.3]), oracle_lib.OracleSettings()),
}


def main():
    for name, (seed, n, W, H, R, t, s) in CASES.items():
        cloud = oracle_lib.random_cloud(seed, n)
        out = {"means": cloud[0].astype(np.float32), "rotations": cloud[1].astype(np.float32),
               "log_scales": cloud[2].astype(np.float32), "raw_opacities": cloud[3].astype(np.float32),
               "colors": cloud[4].astype(np.float32), "width": W, "height": H,
               "rotation": R.astype(np.float32).astype(np.float64), "translation": t.astype(np.float32).astype(np.float64),
               "settings": s.array()}
        for portable in (False, True):
            fr = oracle_lib.render(cloud, out["rotation"], out["translation"], W, H, s, portable=portable)
            tag = "portable" if portable else "std"
            out[f"walked_{tag}"] = fr.get("walked")
            out[f"tile_offsets_{tag}"] = fr.get("tile_offsets")
            out[f"tile_entries_{tag}"] = fr.get("tile_entries")
            out[f"image_{tag}"] = fr.get("image").astype(np.float32)
        np.savez_compressed(HERE / f"{name}.npz", **out)
        print(name, {k: v.shape for k, v in out.items() if hasattr(v, "shape")})


if __name__ == "__main__":
    main()

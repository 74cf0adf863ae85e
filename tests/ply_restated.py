"""TEST INFRASTRUCTURE: an independent numpy restatement of the reference's polygon
writers (src/io.cpp), used to check the library's output byte for byte.

    pointcloud_bytes   save_pointcloud  io.cpp:225-257
    checkpoint_bytes   save_checkpoint  io.cpp:299-332
"""
import numpy as np

KSH0 = 0.28209479177387814
FIELDS = ["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1", "scale_2",
          "rot_0", "rot_1", "rot_2", "rot_3"]


def _byte(v):
    # static_cast<unsigned char>(std::lround(std::clamp(v, 0.0, 1.0) * 255.0)), finite inputs
    x = np.clip(np.asarray(v, np.float64), 0.0, 1.0) * 255.0
    return (np.floor(x + 0.5)).astype(np.uint8)  # lround: halves away from zero (x >= 0 here)


def pointcloud_bytes(positions, colors) -> bytes:
    n = positions.shape[1]
    head = ("ply\nformat binary_little_endian 1.0\n"
            f"element vertex {n}\n"
            "property float x\nproperty float y\nproperty float z\n"
            "property uchar red\nproperty uchar green\nproperty uchar blue\n"
            "end_header\n").encode()
    rec = np.zeros(n, dtype=[("p", "<f4", 3), ("c", "u1", 3)])
    rec["p"] = positions.T.astype(np.float32)
    rec["c"] = _byte(colors.T)
    return head + rec.tobytes()


def checkpoint_bytes(means, rotations, log_scales, raw_opacities, colors) -> bytes:
    n = raw_opacities.shape[0]
    head = "ply\nformat binary_little_endian 1.0\ncomment odgs_checkpoint_version 1\n"
    head += f"element vertex {n}\n" + "".join(f"property float {f}\n" for f in FIELDS) + "end_header\n"
    f_dc = ((colors - 0.5) / KSH0).astype(np.float32)
    f_dc = np.where(np.abs(f_dc) < np.float32(2.0 ** -27), np.float32(0.0), f_dc)
    rows = np.concatenate([means.astype(np.float32), f_dc, raw_opacities[None].astype(np.float32),
                           log_scales.astype(np.float32), rotations.astype(np.float32)], axis=0)
    return head.encode() + np.ascontiguousarray(rows.T, dtype="<f4").tobytes()

"""Scene I/O: the library's polygon readers/writers against the
reference's own test_io.cpp cases and, byte for byte, against an independent
restatement of the writers (tests/ply_restated.py). Host code: runs without a GPU."""
import math

import numpy as np
import pytest

import ply_restated
from paper_2410_20686_b200 import io
from paper_2410_20686_b200.rasterizer import OdgsRuntimeError


def write_text(path, text):
    path.write_bytes(text.encode())


def random_cloud64(n, seed):  # test_io.cpp:32-47 (distribution shape; numpy generator)
    r = np.random.default_rng(seed)
    u = lambda *s: r.uniform(-1.0, 1.0, s)
    return io.GaussianCloud64(3.0 * u(3, n), u(4, n), -2.0 + u(3, n), 2.0 * u(n), 0.5 + 0.45 * u(3, n))


CKPT_FIELDS = ["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1", "scale_2",
               "rot_0", "rot_1", "rot_2", "rot_3"]


def checkpoint_header_14(extra_comment):  # test_io.cpp:57-67
    h = "ply\nformat ascii 1.0\n"
    if extra_comment:
        h += "comment " + extra_comment + "\n"
    h += "element vertex 1\n" + "".join(f"property float {f}\n" for f in CKPT_FIELDS) + "end_header\n"
    return h


def test_one_point_ascii_cloud_loads(tmp_path):  # test_io.cpp:71-92 (load half)
    p = tmp_path / "one_point.ply"
    write_text(p, "ply\nformat ascii 1.0\nelement vertex 1\n"
                  "property float x\nproperty float y\nproperty float z\n"
                  "property uchar red\nproperty uchar green\nproperty uchar blue\n"
                  "end_header\n0 0 0 255 255 255\n")
    pts = io.load_pointcloud(p)
    assert pts.positions.shape == (3, 1)
    assert np.linalg.norm(pts.positions[:, 0]) == 0.0
    assert np.array_equal(pts.colors[:, 0], [1.0, 1.0, 1.0])


def test_binary_and_ascii_point_clouds_load_identically(tmp_path):  # test_io.cpp:118-147
    r = np.random.default_rng(11)
    pos = r.uniform(-4, 4, (3, 23))
    col = np.abs(r.uniform(-4, 4, (3, 23))) / 4.0
    pts = io.PointCloud(pos, col)
    io.save_pointcloud(pts, tmp_path / "b.ply", binary=True)
    io.save_pointcloud(pts, tmp_path / "a.ply", binary=False)
    b = io.load_pointcloud(tmp_path / "b.ply")
    a = io.load_pointcloud(tmp_path / "a.ply")
    assert b.positions.shape == (3, 23)
    assert np.array_equal(a.positions, b.positions) and np.array_equal(a.colors, b.colors)
    assert np.array_equal(b.positions.astype(np.float32).astype(np.float64), b.positions)
    assert np.abs(b.positions - pos).max() < 1e-6
    assert np.abs(b.colors - np.minimum(col, 1.0)).max() < 0.5 / 255.0 + 1e-12
    # byte-exact against the restated writer
    assert (tmp_path / "b.ply").read_bytes() == ply_restated.pointcloud_bytes(pos, col)


def test_float_typed_colors_are_not_rescaled(tmp_path):  # test_io.cpp:149-159
    p = tmp_path / "float_colors.ply"
    write_text(p, "ply\nformat ascii 1.0\nelement vertex 1\n"
                  "property float x\nproperty float y\nproperty float z\n"
                  "property float red\nproperty float green\nproperty float blue\n"
                  "end_header\n1 2 3 0.25 0.5 0.75\n")
    pts = io.load_pointcloud(p)
    assert np.array_equal(pts.colors[:, 0], [0.25, 0.5, 0.75])
    assert np.array_equal(pts.positions[:, 0], [1, 2, 3])


def test_double_properties_and_trailing_elements(tmp_path):  # io.cpp:79-89, 163-166
    p = tmp_path / "mixed.ply"
    head = ("ply\nformat binary_little_endian 1.0\ncomment made by hand\nelement vertex 2\n"
            "property double x\nproperty float32 y\nproperty float64 z\nproperty uint8 red\n"
            "property uchar green\nproperty uchar blue\nelement face 0\nproperty list uchar int vertex_indices\n"
            "end_header\n").encode()
    rec = np.zeros(2, dtype=[("x", "<f8"), ("y", "<f4"), ("z", "<f8"), ("c", "u1", 3)])
    rec["x"] = [1.0 / 3.0, -2.5]
    rec["y"] = [0.1, 7.0]
    rec["z"] = [1e-300, 3.0]
    rec["c"] = [[0, 51, 255], [255, 255, 1]]
    p.write_bytes(head + rec.tobytes())
    pts = io.load_pointcloud(p)
    assert np.array_equal(pts.positions[0], [1.0 / 3.0, -2.5])
    assert np.array_equal(pts.positions[1], np.float32([0.1, 7.0]).astype(np.float64))
    assert np.array_equal(pts.positions[2], [1e-300, 3.0])
    assert np.array_equal(pts.colors[:, 0], [0.0, 51 / 255.0, 1.0])


def test_checkpoints_reload_to_the_values_they_stored(tmp_path):  # test_io.cpp:161-186
    original = random_cloud64(17, 5)
    io.save_checkpoint(original, tmp_path / "a.ply")
    assert (tmp_path / "a.ply").read_bytes() == ply_restated.checkpoint_bytes(
        original.means, original.rotations, original.log_scales, original.raw_opacities, original.colors)
    once = io.load_checkpoint(tmp_path / "a.ply")
    assert once.n == 17
    assert np.abs(once.means - original.means).max() < 1e-6
    assert np.array_equal(once.raw_opacities.astype(np.float32).astype(np.float64), once.raw_opacities)
    io.save_checkpoint(once, tmp_path / "b.ply")
    twice = io.load_checkpoint(tmp_path / "b.ply")
    for k in ("means", "rotations", "log_scales", "raw_opacities", "colors"):
        assert np.array_equal(getattr(once, k), getattr(twice, k)), k
    assert np.array_equal(once.means[:, 3], original.means[:, 3].astype(np.float32).astype(np.float64))
    assert once.raw_opacities[3] == float(np.float32(original.raw_opacities[3]))
    assert np.array_equal(once.rotations[:, 3], original.rotations[:, 3].astype(np.float32).astype(np.float64))


def test_checkpoint_colors_pass_through_the_degree_zero_basis(tmp_path):  # test_io.cpp:188-203
    c = io.GaussianCloud64.empty(1)
    c.means[:, 0] = [0, 0, 2]
    c.colors[:, 0] = [0.9, 0.5, 0.2]
    io.save_checkpoint(c, tmp_path / "c.ply")
    loaded = io.load_checkpoint(tmp_path / "c.ply")
    k = 0.28209479177387814
    assert loaded.colors[0, 0] == 0.5 + k * float(np.float32((0.9 - 0.5) / k))
    assert loaded.colors[1, 0] == 0.5
    assert loaded.colors[2, 0] == 0.5 + k * float(np.float32((0.2 - 0.5) / k))


def test_newer_versions_rejected_older_accepted(tmp_path):  # test_io.cpp:205-221
    row = "0 0 1 0 0 0 0 -1 -1 -1 1 0 0 0\n"
    write_text(tmp_path / "newer.ply", checkpoint_header_14("odgs_checkpoint_version 2") + row)
    with pytest.raises(OdgsRuntimeError, match="version 2"):
        io.load_checkpoint(tmp_path / "newer.ply")
    write_text(tmp_path / "unversioned.ply", checkpoint_header_14("") + row)
    c = io.load_checkpoint(tmp_path / "unversioned.ply")
    assert c.n == 1
    assert np.array_equal(c.means[:, 0], [0, 0, 1])
    assert np.array_equal(c.colors[:, 0], [0.5, 0.5, 0.5])
    assert np.array_equal(c.rotations[:, 0], [1, 0, 0, 0])


def test_missing_properties_and_truncated_data_name_the_problem(tmp_path):  # test_io.cpp:223-261
    write_text(tmp_path / "no_blue.ply", "ply\nformat ascii 1.0\nelement vertex 1\n"
                                         "property float x\nproperty float y\nproperty float z\n"
                                         "property uchar red\nproperty uchar green\nend_header\n0 0 0 10 20\n")
    with pytest.raises(OdgsRuntimeError, match="missing required property 'blue'"):
        io.load_pointcloud(tmp_path / "no_blue.ply")
    head = ("ply\nformat binary_little_endian 1.0\nelement vertex 2\n"
            "property float x\nproperty float y\nproperty float z\n"
            "property uchar red\nproperty uchar green\nproperty uchar blue\nend_header\n").encode()
    (tmp_path / "truncated.ply").write_bytes(head + np.zeros(3, "<f4").tobytes() + bytes([255, 255, 255]))
    with pytest.raises(OdgsRuntimeError, match=r"truncated vertex data \(byte %d\)" % (len(head) + 15)):
        io.load_pointcloud(tmp_path / "truncated.ply")
    write_text(tmp_path / "not_a.ply", "solid teapot\n")
    with pytest.raises(OdgsRuntimeError, match=r"missing 'ply' magic\) \(byte 0\)"):
        io.load_pointcloud(tmp_path / "not_a.ply")
    with pytest.raises(OdgsRuntimeError, match="cannot open file"):
        io.load_pointcloud(tmp_path / "does_not_exist.ply")


@pytest.mark.parametrize("text,needle", [
    ("ply\nformat binary_big_endian 1.0\nelement vertex 1\nproperty float x\nend_header\n",
     "unsupported format 'binary_big_endian' (byte 4)"),
    ("ply\nformat ascii 1.0\nelement face 1\nelement vertex 1\nproperty float x\nend_header\n",
     "element 'face' precedes the vertex element"),
    ("ply\nformat ascii 1.0\nelement vertex 1\nproperty list uchar int idx\nend_header\n",
     "list properties are not supported on vertices"),
    ("ply\nformat ascii 1.0\nelement vertex 1\nproperty short x\nend_header\n", "unsupported property type 'short'"),
    ("ply\nformat ascii 1.0\nelement vertex 1\nproperty float x\nbogus line\nend_header\n",
     "unrecognized header line 'bogus line'"),
    ("ply\nelement vertex 1\nproperty float x\nend_header\n", "header has no format line"),
    ("ply\nformat ascii 1.0\nelement vertex 1\nend_header\n", "no vertex properties declared"),
    ("ply\nformat ascii 1.0\nelement vertex 1\nproperty float x\n", "header ended before 'end_header'"),
    ("ply\nformat ascii 1.0\nelement vertex 1\nproperty float x\nproperty float y\nend_header\n1 zz\n",
     "malformed vertex line"),
    ("ply\nformat ascii 1.0\nelement vertex 0\nproperty float x\nend_header\n", "point cloud is empty"),
])
def test_header_grammar_errors(tmp_path, text, needle):  # parse_ply_header io.cpp:41-118, read_ply :141-199
    p = tmp_path / "bad.ply"
    write_text(p, text)
    with pytest.raises(OdgsRuntimeError) as e:
        io.load_pointcloud(p)
    assert needle in str(e.value)
    assert str(e.value).startswith(str(p) + ": ")


def test_checkpoint_missing_property(tmp_path):
    text = checkpoint_header_14("").replace("property float rot_3\n", "") + "0 0 1 0 0 0 0 -1 -1 -1 1 0 0\n"
    write_text(tmp_path / "c.ply", text)
    with pytest.raises(OdgsRuntimeError, match="missing required property 'rot_3'"):
        io.load_checkpoint(tmp_path / "c.ply")

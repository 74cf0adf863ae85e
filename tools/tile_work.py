"""Per-tile blend work distribution of the C3 render (list lengths, sum of walks)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_20686_b200 import Context, GaussianCloud, RenderSettings, render, scenes  # noqa: E402

ctx = Context(0)
c = scenes.cloud_c3(1_000_000)
fr = render(ctx, c, scenes.yaw_camera(0.0, 2048, 1024), RenderSettings())
offs = fr.tile_offsets.astype(np.int64)
L = np.diff(offs)
W, H = 2048, 1024
walked = fr.walked.reshape(W, H)  # [x][y]
tw = walked.reshape(128, 16, 64, 16).sum(axis=(1, 3))  # [tx][ty]
tw = tw.T.ravel()  # tile id = ty * 128 + tx
print("tiles", L.size, "entries", L.sum())
for name, v in (("list length", L), ("sum walked", tw)):
    q = np.percentile(v, [50, 90, 99, 99.9, 100])
    print(f"{name:12s} mean {v.mean():10.1f}  p50 {q[0]:9.0f} p90 {q[1]:9.0f} p99 {q[2]:9.0f} p99.9 {q[3]:9.0f} max {q[4]:9.0f}")
top = np.argsort(tw)[::-1][:10]
print("top tiles (ty, tx, list, sum_walked):", [(int(t // 128), int(t % 128), int(L[t]), int(tw[t])) for t in top])
print("share of walked work in top 1% tiles:", tw[np.argsort(tw)[::-1][: L.size // 100]].sum() / tw.sum())

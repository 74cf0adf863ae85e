"""Stage times of single row bands of the C5 render (10M Gaussians, 4096x2048, 8 bands)."""
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_20686_b200 import Context, GaussianCloud, RenderOutput, RenderSettings, render_band, scenes  # noqa

dev = torch.device("cuda", 0)
ctx = Context(0, stream=torch.cuda.current_stream().cuda_stream)
src = scenes.cloud_c5(10_000_000)
cloud = GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(getattr(src, k))).to(dev)
                        for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")])
W, H = 4096, 2048
fr = RenderOutput(ctx)
s = RenderSettings()
for b in (0, 3):
    r0, r1 = b * 256, (b + 1) * 256
    for k in range(2):
        render_band(ctx, cloud, scenes.yaw_camera(0.1 * k, W, H), s, r0, r1, out=fr)
    ctx.set_profiling(True)
    ctx.reset_stage_times()
    for k in range(3):
        render_band(ctx, cloud, scenes.yaw_camera(0.1 * k, W, H), s, r0, r1, out=fr)
    torch.cuda.synchronize()
    st = {k: round(v[0] / max(v[1], 1), 4) for k, v in ctx.stage_times().items() if v[1]}
    ctx.set_profiling(False)
    print("band", b, "entries", fr.info().n_entries, st, "sum", round(sum(st.values()), 3))

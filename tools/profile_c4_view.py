"""One C4 view (3M Gaussians, 2048x1024): render + L1 loss + backward, for ncu captures."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_20686_b200 import Context, GaussianCloud, RenderSettings, backward, render, scenes  # noqa: E402

dev = torch.device("cuda", 0)
ctx = Context(0, stream=torch.cuda.current_stream().cuda_stream)
src = scenes.cloud_c4(3_000_000, 4001)
cloud = GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(getattr(src, k))).to(dev)
                        for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")])
cam = scenes.c4_views()[1]
s = RenderSettings()
dl = torch.from_numpy(np.random.default_rng(0).uniform(-1e-7, 1e-7, (3, 2048, 1024)).astype(np.float32)).to(dev)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for _ in range(2):
    fr = render(ctx, cloud, cam, s)
    g = backward(ctx, cloud, cam, fr, dl, s)
ctx.set_profiling(True)
ctx.reset_stage_times()
for _ in range(iters):
    fr = render(ctx, cloud, cam, s)
    g = backward(ctx, cloud, cam, fr, dl, s)
from paper_2410_20686_b200 import _capi as capi  # noqa: E402
torch.cuda.synchronize()
stages = {k: round(v[0] / max(v[1], 1), 4) for k, v in ctx.stage_times().items() if v[1]}
ctx.lib.odgs_frame_set_flags(fr.handle, capi.FRAME_COUNT_WORK)
fr = render(ctx, cloud, cam, s, out=fr)
g = backward(ctx, cloud, cam, fr, dl, s)
torch.cuda.synchronize()
print("n_entries", fr.info().n_entries, "work", fr.work(), "bwd_work", fr.backward_work())
print(stages)

"""A/B of the C5 row-band render (10M Gaussians, 4096x2048, 8 bands) on one GPU:
mean ms per band over all 8 bands, device-timed (set ODGS_B200_LIB to pick a build)."""
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
s = RenderSettings()
frs = [RenderOutput(ctx) for _ in range(8)]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
for k in range(2):
    for b in range(8):
        render_band(ctx, cloud, scenes.yaw_camera(0.0, W, H), s, b * 256, (b + 1) * 256, out=frs[b])
torch.cuda.synchronize()
ms = []
for b in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(reps):
        render_band(ctx, cloud, scenes.yaw_camera(0.0, W, H), s, b * 256, (b + 1) * 256, out=frs[b])
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1) / reps)
print("splats per band", [frs[b].info().n_splats for b in range(8)])
print("bands ms", [round(v, 3) for v in ms], "mean", round(sum(ms) / 8, 4), "max", round(max(ms), 4))

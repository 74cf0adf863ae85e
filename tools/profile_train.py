"""C4 training steps (3M Gaussians, 8 views at 2048x1024, lambda_SSIM 0.2) for launch-list
captures: `python tools/profile_train.py STEPS` runs 2 warm-up steps then STEPS steps."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_20686_b200 import Context, GaussianCloud, RenderOutput, RenderSettings, render, scenes  # noqa: E402
from paper_2410_20686_b200.train import TrainConfig, ViewShardedTrainer  # noqa: E402

dev = torch.device("cuda", 0)
ctx = Context(0, stream=torch.cuda.current_stream().cuda_stream)
W, H, n = 2048, 1024, 3_000_000
views = scenes.c4_views(W, H, 8)
load = lambda seed: GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(getattr(scenes.cloud_c4(n, seed), k)))
                                    .to(dev) for k in ("means", "rotations", "log_scales", "raw_opacities",
                                                       "colors")])
cloud, tcloud = load(4001), load(4002)
s = RenderSettings()
fr = RenderOutput(ctx)
targets = []
for v in views:
    render(ctx, tcloud, v, s, out=fr)
    targets.append(torch.from_numpy(fr.image.ravel()).to(dev))
tr = ViewShardedTrainer(ctx, cloud, views, targets, s, TrainConfig(), 10.0)
for _ in range(2):
    tr.step()
torch.cuda.synchronize()
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(steps):
    tr.step()
ev[1].record()
torch.cuda.synchronize()
print("ms/step", ev[0].elapsed_time(ev[1]) / steps)

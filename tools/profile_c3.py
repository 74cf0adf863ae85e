"""C3 frames (1M Gaussians, 2048x1024): per-stage CUDA-event times and the frame time
(asynchronous renders, events around the queued frames) — for A/B builds
(ODGS_B200_LIB=...)."""
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_20686_b200 import Context, GaussianCloud, RenderOutput, RenderSettings, render, scenes  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream()
ctx = Context(0, stream=stream.cuda_stream)
ctx.set_async(True)
c = scenes.cloud_c3(1_000_000)
cloud = GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(getattr(c, k))).to(dev)
                        for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")])
s = RenderSettings()
fr = RenderOutput(ctx)
cam = lambda k: scenes.yaw_camera(2 * math.pi * (k % 64) / 64.0, 2048, 1024)
for k in range(5):
    render(ctx, cloud, cam(k), s, out=fr)
fr.check()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
torch.cuda.synchronize()
for k in range(steps):
    flush.zero_()
    ev[k][0].record(stream)
    render(ctx, cloud, cam(k), s, out=fr)
    ev[k][1].record(stream)
torch.cuda.synchronize()
fr.check()
ms = sorted(a.elapsed_time(b) for a, b in ev)
ctx.set_profiling(True)
ctx.reset_stage_times()
for k in range(10):
    flush.zero_()
    render(ctx, cloud, cam(k), s, out=fr)
torch.cuda.synchronize()
st = {k: round(v[0] / max(v[1], 1), 4) for k, v in ctx.stage_times().items() if v[1]}
print(f"frame median {ms[len(ms) // 2]:.4f} ms  mean {sum(ms) / len(ms):.4f}  stages {st}")

"""C3 throughput with S frames in flight: S contexts (own streams) render alternate frames
(asynchronous), an L2 flush before every frame on its stream; events around the whole
batch. `python tools/profile_c3_pipe.py FRAMES S [flush 0/1]`."""
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_20686_b200 import Context, GaussianCloud, RenderOutput, RenderSettings, render, scenes  # noqa: E402

dev = torch.device("cuda", 0)
frames = int(sys.argv[1]) if len(sys.argv) > 1 else 40
S = int(sys.argv[2]) if len(sys.argv) > 2 else 2
do_flush = int(sys.argv[3]) if len(sys.argv) > 3 else 1
streams = [torch.cuda.Stream(dev) for _ in range(S)]
ctxs = [Context(0, stream=st.cuda_stream) for st in streams]
for c in ctxs:
    c.set_async(True)
src = scenes.cloud_c3(1_000_000)
cloud = GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(getattr(src, k))).to(dev)
                        for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")])
s = RenderSettings()
frs = [RenderOutput(c) for c in ctxs]
flush = [torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev) for _ in range(S)]
cam = lambda k: scenes.yaw_camera(2 * math.pi * (k % 64) / 64.0, 2048, 1024)
torch.cuda.synchronize()
for k in range(2 * S):
    i = k % S
    with torch.cuda.stream(streams[i]):
        render(ctxs[i], cloud, cam(k), s, out=frs[i])
for f in frs:
    f.check()
torch.cuda.synchronize()
main = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(main)
for st in streams:
    st.wait_event(e0)
for k in range(frames):
    i = k % S
    with torch.cuda.stream(streams[i]):
        if do_flush:
            flush[i].zero_()
        render(ctxs[i], cloud, cam(k), s, out=frs[i])
for st in streams:
    main.wait_stream(st)
e1.record(main)
torch.cuda.synchronize()
for f in frs:
    assert not f.check()
ms = e0.elapsed_time(e1)
print(f"S={S} flush={do_flush}: {ms / frames:.4f} ms/frame  {1000 * frames / ms:.1f} fps")

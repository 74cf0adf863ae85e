"""Photometric loss (L1 + SSIM, lambda 0.2) on two 2048x1024 RGB images, for timing and ncu
captures of the loss kernels: prints the mean loss-call time (CUDA events)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_20686_b200 import Context  # noqa: E402

W, H = 2048, 1024
dev = torch.device("cuda", 0)
ctx = Context(0, stream=torch.cuda.current_stream().cuda_stream)
rng = np.random.default_rng(5)
a = torch.from_numpy(rng.random(3 * W * H, dtype=np.float32)).to(dev)
b = torch.from_numpy(np.clip(a.cpu().numpy() + rng.normal(0, 0.1, a.shape).astype(np.float32), 0, 1)).to(dev)
grad = torch.empty_like(a)
acc = torch.zeros(1, dtype=torch.float64, device=dev)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20


def call():
    ctx.check(ctx.lib.odgs_photometric_loss_async(ctx.handle, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), W, H,
                                                  0.2, C.c_void_p(grad.data_ptr()), C.c_void_p(acc.data_ptr())))


for _ in range(3):
    call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    call()
e1.record()
torch.cuda.synchronize()
print(f"loss call {e0.elapsed_time(e1) / iters:.4f} ms")

"""Row-band renders over several GPUs with the all-gather fused into the blend
(SURVEY.md §8e, config C5).

Every rank owns a full-image buffer; the buffers are exported and opened on every
other rank with CUDA IPC (odgs_ipc_get_handle / odgs_ipc_open — one process per GPU on
one node, NVLink / NVSwitch peer memory). The frame's blend then writes each pixel of
its band into all ranks' full images as it composites it (odgs_frame_set_image_peers),
so no collective moves image data: after one barrier (a tiny NCCL all-reduce, which
orders every rank's stream behind every other rank's render) each rank holds the whole
frame.
"""
from __future__ import annotations

import ctypes as C
from typing import List

from . import _capi as capi


def ipc_handle(lib, device_ptr: int) -> bytes:
    buf = C.create_string_buffer(capi.IPC_HANDLE_BYTES)
    st = lib.odgs_ipc_get_handle(C.c_void_p(device_ptr), buf)
    if st != capi.STATUS_OK:
        raise RuntimeError(f"odgs_ipc_get_handle failed ({st})")
    return buf.raw


def ipc_open(lib, handle: bytes) -> int:
    p = C.c_void_p()
    st = lib.odgs_ipc_open(C.create_string_buffer(handle, capi.IPC_HANDLE_BYTES), C.byref(p))
    if st != capi.STATUS_OK:
        raise RuntimeError(f"odgs_ipc_open failed ({st})")
    return int(p.value)


class BandGather:
    """Full-image buffers of all ranks, wired into `frame` as blend outputs."""

    def __init__(self, ctx, frame, width: int, height: int, device, group=None):
        import torch
        import torch.distributed as dist
        self.ctx, self.frame = ctx, frame
        self.full = torch.zeros(3 * width * height, dtype=torch.float32, device=device)
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.opened: List[int] = []
        ptrs = [self.full.data_ptr()]
        if world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, ipc_handle(ctx.lib, self.full.data_ptr()), group=group)
            for r, h in enumerate(handles):
                if r != rank:
                    p = ipc_open(ctx.lib, h)
                    self.opened.append(p)
                    ptrs.append(p)
        frame.set_image_peers(ptrs)
        self.world, self.group = world, group

    def sync(self, device_id: int) -> None:
        """After every rank's band render: all full images are complete. With NCCL the
        barrier's all-reduce is stream-ordered behind each rank's render; with other
        backends the device is synchronised first."""
        import torch
        import torch.distributed as dist
        if self.world > 1:
            if dist.get_backend(self.group) == "nccl":
                dist.barrier(group=self.group, device_ids=[device_id])
            else:
                torch.cuda.synchronize()
                dist.barrier(group=self.group)

    def close(self) -> None:
        self.frame.set_image_peers([])
        for p in self.opened:
            self.ctx.lib.odgs_ipc_close(C.c_void_p(p))
        self.opened = []

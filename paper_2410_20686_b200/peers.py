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
    """Full-image buffers of all ranks, wired into `frame` as blend outputs.

    Double-buffered: frame k's bands are written into every rank's buffer k % 2, so a
    rank may still read frame k's image (`full`) while the others already render frame
    k + 1 into the other buffer. The rule: read a frame's image before calling sync() of
    the next frame — that sync's barrier then orders the reads before any rank's frame
    k + 2 writes into the same buffer. Call begin() before each band render."""

    def __init__(self, ctx, frame, width: int, height: int, device, group=None):
        import torch
        import torch.distributed as dist
        self.ctx, self.frame = ctx, frame
        self.buffers = [torch.zeros(3 * width * height, dtype=torch.float32, device=device) for _ in range(2)]
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.opened: List[int] = []
        self.ptrs = [[b.data_ptr()] for b in self.buffers]  # per parity: own buffer first, then the peers'
        if world > 1:
            for par, b in enumerate(self.buffers):
                handles = [None] * world
                dist.all_gather_object(handles, ipc_handle(ctx.lib, b.data_ptr()), group=group)
                for r, h in enumerate(handles):
                    if r != rank:
                        p = ipc_open(ctx.lib, h)
                        self.opened.append(p)
                        self.ptrs[par].append(p)
        self.world, self.group = world, group
        self.parity = 1
        self._fresh = False
        self.begin()

    @property
    def full(self):
        """This rank's copy of the current frame (all bands after sync())."""
        return self.buffers[self.parity]

    def begin(self) -> None:
        """Starts the next frame: its bands go into the other buffer of every rank (a no-op
        until the current frame has been synced, so calling it before every render is safe)."""
        if self._fresh:
            return
        self.parity ^= 1
        self.frame.set_image_peers(self.ptrs[self.parity])
        self._fresh = True

    def sync(self, device_id: int) -> None:
        """After every rank's band render: all full images are complete. With NCCL the
        barrier's all-reduce is stream-ordered behind each rank's render; with other
        backends the device is synchronised first."""
        import torch
        import torch.distributed as dist
        self._fresh = False
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

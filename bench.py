#!/usr/bin/env python
"""Benchmark of the B200 ODGS rasterizer (BASELINE.json metric: ERP frames/sec for 1M
Gaussians at 2048x1024).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one forward render (preprocess -> depth sort -> emit -> tile sort -> tile
ranges -> blend) of the C3 workload — 1M synthetic Gaussians, 50% uniform, 25% near the
poles, 25% on the azimuth seam — into a 2048x1024 ERP frame, from a camera yawed by a
different angle every step. With N > 1 (torchrun, one process per GPU) every rank
renders its own views (weak scaling; the render path has no exchange step, so there
is no collective in it). Rank 0 prints one JSON line.

--impl reference times the reference algorithm's CPU implementation (the oracle
restatement, oracle/odgs_oracle.hpp, StdMath float — the reference itself cannot be
built in this image) on the host's cores, one full C3 frame per step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ERP frames/sec (1M Gaussians, 2048×1024)"
UNIT = "frames/s"
W_IMG, H_IMG = 2048, 1024
N_GAUSS = 1_000_000
E2E_LANES = int(os.environ.get("ODGS_E2E_LANES", "4"))  # frames in flight on the e2e path (contexts / streams / host threads)
WORKLOAD = ("C3: 1M synthetic Gaussians (50% uniform, 25% poles |elev| 75-89.5 deg, 25% azimuth seam), "
            "SH0, 2048x1024 ERP, camera yawed per step")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-train", action="store_true")
    ap.add_argument("--train-steps", type=int, default=5)
    ap.add_argument("--no-large", action="store_true")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock and throttle reasons sampled every 20 ms during the timed region, via
    NVML in-process (nvidia-smi as a fallback)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None
            self.thread = threading.Thread(target=self._poll_smi, daemon=True)
            self.thread.start()
            return self
        self.thread = threading.Thread(target=self._poll, daemon=True)
        self.thread.start()
        return self

    def _poll(self):
        n = self.nvml
        while not self.stop.is_set():
            try:
                sm = n.nvmlDeviceGetClockInfo(self.handle, n.NVML_CLOCK_SM)
                reasons = n.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
                self.rows.append((sm, reasons))
            except Exception:
                pass
            self.stop.wait(0.02)

    def _poll_smi(self):
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-i",
                                      str(self.gpu)], capture_output=True, text=True, timeout=5).stdout.strip()
                sm, smax, bits = [x.strip() for x in out.split(",")]
                self.max_mhz = float(smax)
                self.rows.append((float(sm), int(bits, 16)))
            except Exception:
                return
            self.stop.wait(0.05)

    def __exit__(self, *a):
        self.stop.set()
        if hasattr(self, "thread"):
            self.thread.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({name for _, bits in self.rows for name, m in self.REASONS.items() if bits & m})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": reasons,
                "samples": len(self.rows)}


def ncu_traffic(kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu capture
    summary (profiles/ncu_traffic.json), or None."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    return d.get(kernel)


def cloud_arrays():
    from paper_2410_20686_b200 import scenes
    c = scenes.cloud_c3(N_GAUSS)
    return [c.means, c.rotations, c.log_scales, c.raw_opacities, c.colors]


def camera(step: int, rank: int):
    from paper_2410_20686_b200 import scenes
    yaw = 2 * math.pi * ((rank * 7919 + step) % 64) / 64.0
    return scenes.yaw_camera(yaw, W_IMG, H_IMG)


# ------------------------------------------------------------------ CPU reference arm
def cpu_frames(arrs, max_frames: int, min_seconds: float):
    """Renders full C3 frames with the oracle (StdMath float, all host threads)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import numpy as np
    import oracle_lib  # the CPU restatement (only the baseline leg may run it)
    a64 = [np.asarray(a, dtype=np.float64) for a in arrs]
    cores = oracle_lib.lib().oracle_hardware_concurrency()
    times = []
    t_all = time.perf_counter()
    for k in range(max_frames):
        cam = camera(k, 0)
        t0 = time.perf_counter()
        oracle_lib.render(a64, cam.rotation, cam.translation, W_IMG, H_IMG, oracle_lib.OracleSettings())
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all >= min_seconds:
            break
    return times, cores


def run_reference(args, rank: int):
    if rank != 0:
        return
    arrs = cloud_arrays()
    cpu_frames(arrs, max_frames=max(args.warmup, 0), min_seconds=0.0) if args.warmup > 0 else None
    times, cores = cpu_frames(arrs, max_frames=args.steps, min_seconds=float("inf"))
    total = sum(times)
    value = len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(times), "warmup": args.warmup, "ms_per_step": 1000 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n_gaussians": N_GAUSS, "width": W_IMG, "height": H_IMG},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{len(times)} full C3 frames, oracle restatement (StdMath float), "
                                   f"threads = all {cores} host threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def pcie_peaks(torch, dev, h2d: int, d2h: int) -> dict:
    """Pinned-host copy bandwidth of this box, one frame's bytes per copy (best of 10,
    CUDA events): the ceiling of the e2e path, which moves h2d + d2h bytes per frame."""
    hs = torch.empty(h2d, dtype=torch.uint8).pin_memory()
    ds = torch.empty(h2d, dtype=torch.uint8, device=dev)
    hd = torch.empty(d2h, dtype=torch.uint8).pin_memory()
    dd = torch.empty(d2h, dtype=torch.uint8, device=dev)
    out = {}
    for key, dst, src, nbytes in (("h2d_gbs", ds, hs, h2d), ("d2h_gbs", hd, dd, d2h)):
        best = None
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dst.copy_(src, non_blocking=True)
            b.record()
            b.synchronize()
            ms = a.elapsed_time(b)
            best = ms if best is None else min(best, ms)
        out[key] = nbytes / (best * 1e-3) / 1e9
    # Both directions at once (as in the pipelined e2e frames): H2D rate while a D2H of
    # a frame's image runs on another stream, per frame (h2d bytes + d2h bytes in flight).
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    best = None
    for _ in range(10):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s1)
        s2.wait_event(a)
        with torch.cuda.stream(s1):
            ds.copy_(hs, non_blocking=True)
        with torch.cuda.stream(s2):
            for _ in range(max(1, h2d // d2h)):
                hd.copy_(dd, non_blocking=True)
        b.record(s1)
        b.synchronize()
        ms = a.elapsed_time(b)
        best = ms if best is None else min(best, ms)
    torch.cuda.synchronize()
    out["h2d_gbs_with_d2h"] = h2d / (best * 1e-3) / 1e9
    return out


# ------------------------------------------------------------------ GPU arm
def run_ours(args, rank: int, world: int, local_rank: int):
    import numpy as np
    import torch
    import torch.distributed as dist
    import ctypes as C

    from paper_2410_20686_b200 import Context, GaussianCloud, RenderOutput, RenderSettings, render
    from paper_2410_20686_b200 import _capi as capi

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream(dev)
    ctx = Context(local_rank, stream=stream.cuda_stream)
    # Asynchronous renders: no host round trip inside or between frames (errors and
    # entry-buffer overflows surface at frame.check()).
    ctx.set_async(True)
    settings = RenderSettings()
    arrs = cloud_arrays()
    dcloud = GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in arrs])
    frame = RenderOutput(ctx)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    # A second buffer read after the flush write evicts the flush's dirty lines, so a step
    # starts from a cold, clean L2 (no write-back of the flush inside the next step).
    flush_clean = torch.zeros(64 * 1024 * 1024, dtype=torch.int32, device=dev)

    def barrier():
        if world > 1:
            rank_barrier(local_rank)

    for k in range(args.warmup):
        render(ctx, dcloud, camera(k, rank), settings, out=frame)
    frame.check()
    torch.cuda.synchronize()

    # Timed region: K renders queued back to back on the stream (no host synchronisation),
    # L2 flushed between steps (outside the step events).
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = ctx.launch_count
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clocks:
        for k in range(args.steps):
            flush.zero_()
            flush_clean.sum()
            starts[k].record(stream)
            render(ctx, dcloud, camera(k, rank), settings, out=frame)
            ends[k].record(stream)
        torch.cuda.synchronize()
    if frame.check():  # an entry-buffer overflow would have re-rendered the last frame
        raise RuntimeError("bench: a timed frame overflowed its entry buffers")
    barrier()
    launches = ctx.launch_count - launches0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    # Per-stage times from a separate profiled pass (stage events and their per-frame
    # readback stay out of the timed region).
    ctx.set_profiling(True)
    ctx.reset_stage_times()
    for k in range(min(args.steps, 10)):
        flush.zero_()
        flush_clean.sum()
        render(ctx, dcloud, camera(k, rank), settings, out=frame)
    torch.cuda.synchronize()
    stages = ctx.stage_times()
    ctx.set_profiling(False)
    # Work counters of the same frames (a separate pass: each read synchronises; the
    # timed frames do not count).
    work = []
    ctx.lib.odgs_frame_set_flags(frame.handle, capi.FRAME_COUNT_WORK)
    for k in range(args.steps):
        render(ctx, dcloud, camera(k, rank), settings, out=frame)
        work.append(frame.work())
    ctx.lib.odgs_frame_set_flags(frame.handle, 0)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_total_ms = float(t.item())
    value = world * args.steps / (max_total_ms / 1000.0)

    # Roofline of the dominant stage.
    hbm_peak, hbm_src = peaks()
    fp32_peak = ctx.measure_fp32_tflops()
    e_exam = sum(w[0] for w in work) / len(work)
    e_contrib = sum(w[1] for w in work) / len(work)
    info = frame.info()
    K = info.n_entries
    stage_ms = {k: v[0] / max(v[1], 1) for k, v in stages.items() if v[1] > 0}
    dominant = max(stage_ms, key=stage_ms.get)
    # Algorithmic work per unit: blend 11 flops per examined entry
    # + 12 per composited entry; preprocess 104 B per Gaussian;
    # sorts 20 B per item per 8-bit pass.
    blend_flops = 11 * e_exam + 12 * e_contrib
    depth_passes = 4
    tile_bits = math.ceil(math.log2(info.tiles_x * info.tiles_y))
    tile_passes = math.ceil(tile_bits / 8)
    bytes_by_stage = {
        "preprocess": 104.0 * N_GAUSS,
        "depth_sort": 20.0 * N_GAUSS * depth_passes,
        "tile_sort": 20.0 * K * tile_passes,
        "emit": 8.0 * K + 44.0 * N_GAUSS,
    }
    stage_roof = {}
    for k, b in bytes_by_stage.items():
        if k in stage_ms:
            gbs = b / (stage_ms[k] * 1e-3) / 1e9
            stage_roof[k] = {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
                             "frac": gbs / hbm_peak, "ms": stage_ms[k]}
    # FP32 lane-op peak: SMs x 128 FP32 lanes x the SM clock sampled under
    # load in the timed region; the blend's ops are unfused (--fmad=false), one lane-op each.
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    clk = clocks.summary()
    sm_mhz = clk["sm_mhz"] or clk["sm_max_mhz"] or 1965.0
    lane_peak = sms * 128 * sm_mhz * 1e6 / 1e12
    if "blend" in stage_ms:
        tf = blend_flops / (stage_ms["blend"] * 1e-3) / 1e12
        stage_roof["blend"] = {"bound": "fp32 lane ops", "achieved": tf, "peak": lane_peak, "unit": "T lane-ops/s",
                               "frac": tf / lane_peak, "ms": stage_ms["blend"],
                               "peak_source": f"{sms} SMs x 128 lanes x {sm_mhz:.0f} MHz (median SM clock, timed region)",
                               "frac_fma_convention": tf / fp32_peak,
                               "fma_peak_tflops": fp32_peak,
                               "work_model": "11 ops per examined entry + 12 per composited (SURVEY.md §8d)"}
    roof = dict(stage_roof[dominant]) if dominant in stage_roof else {"bound": "unknown"}
    roof["kernel"] = dominant
    roof["traffic"] = ncu_traffic(dominant)
    roof.setdefault("peak_source", hbm_src)

    # End to end through the C ABI with host buffers: every frame uploads the cloud from
    # pinned host memory inside odgs_render (56 MB H2D) and downloads the image into
    # pinned memory (25 MB D2H); `pcie` reports this box's pinned copy rates and the frame-rate
    # bound they set. E2E_LANES contexts (own CUDA streams) driven by as many host
    # threads pipeline the frames, so one frame's copies overlap another's kernels (4 lanes: 833 fps vs
    # 762 with 3, 703 with 2; 6 lanes no better — the 56 MB H2D per frame is then ~47 GB/s of PCIe Gen5).
    import threading as _th
    hcloud = GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in arrs])
    h2d = sum(int(np.asarray(a).nbytes) for a in arrs)
    d2h = 3 * W_IMG * H_IMG * 4
    lanes = []
    for _ in range(E2E_LANES):
        c2 = Context(local_rank)  # private stream
        lanes.append((c2, RenderOutput(c2), torch.empty(3 * W_IMG * H_IMG, dtype=torch.float32).pin_memory()))

    def e2e_step(lane, k):
        c2, fr2, himg = lane
        render(c2, hcloud, camera(k, rank), settings, out=fr2)
        c2.check(c2.lib.odgs_frame_download(c2.handle, fr2.handle, capi.FRAME_IMAGE, C.c_void_p(himg.data_ptr()),
                                            d2h))

    def e2e_run(n_frames):
        errs = []

        def worker(li):
            try:
                for k in range(li, n_frames, len(lanes)):
                    e2e_step(lanes[li], k)
            except Exception as e:  # surfaced below
                errs.append(e)
        ths = [_th.Thread(target=worker, args=(li,)) for li in range(len(lanes))]
        for t_ in ths:
            t_.start()
        for t_ in ths:
            t_.join()
        if errs:
            raise errs[0]

    e2e_run(max(args.warmup, 2) * len(lanes))  # every lane allocates its buffers before timing
    barrier()
    torch.cuda.synchronize()
    e2e_launch0 = sum(l[0].launch_count for l in lanes)
    t0 = time.perf_counter()
    e2e_run(args.steps)
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * args.steps / float(te.item())
    for c2, fr2, _ in lanes:
        fr2.destroy()
        c2.close()
    pcie = pcie_peaks(torch, dev, h2d, d2h)

    aux = run_aux(args, ctx, dev, stream) if rank == 0 and not args.no_train else None
    train = None if args.no_train else run_train(args, ctx, rank, world, local_rank, dev, stream, lane_peak, hbm_peak)
    large = None if args.no_large else run_large(args, ctx, rank, world, local_rank, dev, stream)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        times, cores = cpu_frames(arrs, max_frames=5, min_seconds=10.0)
        cpu = {"value": len(times) / sum(times), "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{len(times)} full C3 frame(s) (1M Gaussians, 2048x1024), oracle restatement "
                         f"(StdMath float), threads = all {cores} host threads"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n_gaussians": N_GAUSS, "width": W_IMG, "height": H_IMG,
                       "tile_entries": K, "entries_examined": e_exam, "entries_composited": e_contrib,
                       "l2": "flushed between steps (256 MiB write, then a 256 MiB read that evicts its dirty lines; outside the step events)",
                       "parallelism": f"view-replicas x{world}"},
            "distributed": {"world_size": world, "backend": (__import__("torch.distributed").distributed.get_backend()
                                                             if world > 1 else None),
                            "shared_gpu": SHARE_GPU},
            "roofline": roof,
            "stages_ms": {k: round(v, 4) for k, v in stage_ms.items()},
            "stage_rooflines": stage_roof,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "path": f"odgs_render (host cloud, pinned) + odgs_frame_download (pinned), {E2E_LANES} "
                            f"contexts / streams / host threads pipelining frames",
                    "pcie": dict(pcie, h2d_gbs_achieved=e2e_value * h2d / 1e9,
                                 h2d_frac=e2e_value * h2d / 1e9 / pcie["h2d_gbs"],
                                 h2d_frac_vs_bidirectional=e2e_value * h2d / 1e9 / pcie["h2d_gbs_with_d2h"],
                                 fps_bound=pcie["h2d_gbs_with_d2h"] * 1e9 / h2d)},
            "cpu_baseline": cpu,
            "other_configs": aux,
            "train": train,
            "large_render": large,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "step_ms": {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)},
        }
        print(json.dumps(line), flush=True)
    frame.destroy()
    ctx.close()


def run_train(args, ctx, rank, world, local_rank, dev, stream, lane_peak_tops, hbm_peak):
    """BASELINE config 4: 3M Gaussians, a batch of 8 views at 2048x1024, views sharded
    over the ranks, NCCL all-reduce of the gradients, Adam. One step = the whole
    batch (8/G renders + photometric losses + backward passes per rank, all-reduce, Adam).
    Timed unprofiled (CUDA events on the stream, max over ranks); stage times, work
    counters and the all-reduce time come from separate passes."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2410_20686_b200 import GaussianCloud, RenderSettings, render, scenes
    from paper_2410_20686_b200.train import FLAT_WIDTH, TrainConfig, ViewShardedTrainer, allreduce_grads

    n = 3_000_000
    views = scenes.c4_views(W_IMG, H_IMG, 8)
    src = scenes.cloud_c4(n, 4001)
    cloud = GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(getattr(src, k))).to(dev)
                            for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")])
    tsrc = scenes.cloud_c4(n, 4002)
    tcloud = GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(getattr(tsrc, k))).to(dev)
                             for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")])
    settings = RenderSettings()
    targets = []
    from paper_2410_20686_b200 import RenderOutput
    tf = RenderOutput(ctx)
    for v in views:  # targets: renders of a second cloud
        render(ctx, tcloud, v, settings, out=tf)
        targets.append(torch.from_numpy(tf.image.ravel()).to(dev))
    tf.destroy()
    del tcloud
    extent = float(np.sqrt(((src.means - src.means.mean(axis=1, keepdims=True)) ** 2).sum(axis=0).max()))
    lanes = int(os.environ.get("ODGS_TRAIN_LANES", "2"))  # A/B knob: contexts in the view pipeline
    tr = ViewShardedTrainer(ctx, cloud, views, targets, settings, TrainConfig(), extent, rank, world, pipeline=lanes)

    def barrier():
        if world > 1:
            rank_barrier(local_rank)

    first_loss = tr.step()
    tr.step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.train_steps):
        tr.step(read_loss=False)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    barrier()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    last_loss = tr.step()

    # Separate passes: per-stage times (library CUDA events), then the work counters of
    # every view of one step (forward examined / composited, backward replayed /
    # contributing; the counting backward is a separate, slower instantiation).
    # (stage times summed over the trainer's contexts: its views alternate between two)
    for c in tr.contexts:
        c.set_profiling(True)
        c.reset_stage_times()
    tr.step(read_loss=False)
    torch.cuda.synchronize()
    stages = {}
    for c in tr.contexts:
        for k, v in c.stage_times().items():
            if v[1] > 0:
                stages[k] = stages.get(k, 0.0) + v[0]
        c.set_profiling(False)
    fwd_work, bwd_work = [0, 0], [0, 0, 0, 0]
    import paper_2410_20686_b200.train as train_mod
    real_backward = train_mod.backward

    def counting_backward(*a, **kw):
        out = real_backward(*a, **kw)
        fr = a[3]  # the view's frame
        w = fr.work()
        b = fr.backward_work()
        fwd_work[0] += w[0]; fwd_work[1] += w[1]
        for j in range(4):
            bwd_work[j] += b[j]
        return out
    train_mod.backward = counting_backward
    from paper_2410_20686_b200 import _capi as capi
    for ln in tr.lanes:
        ln.ctx.lib.odgs_frame_set_flags(ln.frame.handle, capi.FRAME_COUNT_WORK)
    try:
        tr.step(read_loss=False)
    finally:
        train_mod.backward = real_backward
        for ln in tr.lanes:
            ln.ctx.lib.odgs_frame_set_flags(ln.frame.handle, 0)
    torch.cuda.synchronize()
    nv = len(tr.mine)
    stage_view = {k: v / nv for k, v in stages.items()}

    # The all-reduce alone (the step's one exchange), and NCCL's bus bandwidth on a 1 GiB
    # buffer as its roofline denominator (measured in the same run).
    allreduce = None
    if world > 1:
        def time_ar(buf, obs, reps=5):
            allreduce_grads(buf, obs)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                allreduce_grads(buf, obs)
            b.record(stream)
            torch.cuda.synchronize()
            return a.elapsed_time(b) / reps
        ar_ms = time_ar(tr.flat, tr.observed)
        big = torch.zeros(256 * 1024 * 1024, dtype=torch.float32, device=dev)
        big_ms = time_ar(big, torch.zeros(1, dtype=torch.int32, device=dev), reps=3)
        del big
        factor = 2.0 * (world - 1) / world
        grad_bytes = 4.0 * (FLAT_WIDTH + 1) * n
        ar_busbw = factor * grad_bytes / (ar_ms * 1e-3) / 1e9
        peak_busbw = factor * 4.0 * 256 * 1024 * 1024 / (big_ms * 1e-3) / 1e9
        allreduce = {"bound": "nvlink", "ms": ar_ms, "bytes": grad_bytes, "achieved": ar_busbw,
                     "peak": peak_busbw, "unit": "GB/s (bus bandwidth, 2(G-1)/G x bytes / time)",
                     "frac": ar_busbw / peak_busbw,
                     "peak_source": "NCCL all-reduce of a 1 GiB fp32 buffer, same run",
                     "frac_vs_nominal_900": ar_busbw / 900.0}

    # Rooflines of the training kernels, per view.
    roof = {}
    if "bwd_raster" in stage_view:
        e_rep, e_con = bwd_work[0] / nv, bwd_work[1] / nv
        ops = 11.0 * e_rep + 45.0 * e_con  # replay: the forward's d2 test; + ~45 ops per contribution
        tops = ops / (stage_view["bwd_raster"] * 1e-3) / 1e12
        roof["bwd_raster"] = {"bound": "fp32 lane ops", "ms_per_view": stage_view["bwd_raster"],
                              "entries_replayed": e_rep, "contributions": e_con, "ops": ops,
                              "achieved": tops, "peak": lane_peak_tops, "unit": "T lane-ops/s",
                              "frac": tops / lane_peak_tops,
                              "work_model": "11 ops per replayed entry + 45 per contribution (SURVEY.md §8d)"}
    if "bwd_splat" in stage_view:
        K = tr.frame.info().n_entries
        byts = 56.0 * n + 36.0 * K + 4.0 * 14 * n + 12.0 * n
        gbs = byts / (stage_view["bwd_splat"] * 1e-3) / 1e9
        roof["fold_and_splat"] = {"bound": "hbm", "ms_per_view": stage_view["bwd_splat"], "bytes": byts,
                                  "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                                  "work_model": "N (56 B cloud + 4x14 B grads + 12 B stats) + 36 B per tile entry "
                                                "(SURVEY.md §8d)"}
    for k in ("bwd_raster", "fold_and_splat"):
        if k in roof:
            roof[k]["traffic"] = ncu_traffic(k)
            roof[k]["traffic_source"] = "profiles/ncu_traffic.json (one ncu --set full capture of a C4 view)"
    if allreduce:
        roof["allreduce"] = allreduce

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = train_cpu_baseline(src, tsrc, views[0])
    return {"metric": "train iters/sec (C4: 3M Gaussians, batch of 8 ERP views at 2048x1024)",
            "value": args.train_steps / (ms_max / 1000.0), "unit": "iters/s", "ms_per_step": ms_max / args.train_steps,
            "steps": args.train_steps, "warmup": 2, "views_per_gpu": nv, "n_gpus": world,
            "view_pipeline": f"{len(tr.lanes)} contexts (view k + 1 renders while view k back-propagates)",
            "scaling": "strong", "loss": "photometric_loss, lambda_ssim = 0.2 (L1 + SSIM on the GPU)",
            "timing": "CUDA events around the unprofiled steps (no host loss readback), max over ranks",
            "collective": (f"{dist.get_backend().upper()} all-reduce (sum) of 16n floats + n int32" if world > 1
                           else "none (1 rank)"),
            "stage_ms_per_step": {k: round(v, 4) for k, v in stages.items()},
            "work_per_view": {"fwd_examined": fwd_work[0] / nv, "fwd_composited": fwd_work[1] / nv,
                              "bwd_replayed": bwd_work[0] / nv, "bwd_contributions": bwd_work[1] / nv,
                              "bwd_warp_entries": bwd_work[2] / nv, "bwd_warp_entries_live": bwd_work[3] / nv},
            "roofline": roof, "cpu_baseline": cpu, "first_loss": first_loss, "last_loss": last_loss}


def train_cpu_baseline(src, tsrc, cam):
    """The reference algorithm on the host (oracle restatement, StdMath double — the
    reference CLI trains in double, tools/odgs.cpp:242; its float isZero() would skip
    every pixel of a photometric gradient — all host threads): render + photometric
    loss + backward of one C4 view, timed; iters/s = 1 / (8 x that) — the CPU's step is
    8 such views (Adam is negligible next to them)."""
    import numpy as np
    sys.path.insert(0, str(ROOT / "tests"))
    import ctypes as C
    import oracle_lib  # the CPU restatement (only the baseline leg may run it)
    L = oracle_lib.lib()
    cores = L.oracle_hardware_concurrency()
    arrs = [np.asarray(getattr(src, k), dtype=np.float64) for k in ("means", "rotations", "log_scales",
                                                                    "raw_opacities", "colors")]
    tarrs = [np.asarray(getattr(tsrc, k), dtype=np.float64) for k in ("means", "rotations", "log_scales",
                                                                      "raw_opacities", "colors")]
    r, t = np.asarray(cam.rotation, np.float32).astype(np.float64), np.asarray(cam.translation, np.float32).astype(
        np.float64)
    target = oracle_lib.render(tarrs, r, t, W_IMG, H_IMG, dbl=True).get("image")
    t0 = time.perf_counter()
    fr = oracle_lib.render(arrs, r, t, W_IMG, H_IMG, dbl=True)
    t1 = time.perf_counter()
    img = fr.get("image")
    g = np.empty_like(img)
    dp = C.POINTER(C.c_double)
    L.oracle_photometric_loss(img.ctypes.data_as(dp), target.ctypes.data_as(dp), H_IMG, W_IMG, 0.2,
                              g.ctypes.data_as(dp))
    t2 = time.perf_counter()
    fr.backward(g)
    t3 = time.perf_counter()
    view_s = t3 - t0
    return {"value": 1.0 / (8.0 * view_s), "unit": "iters/s", "cores": cores, "kind": "port",
            "render_s": t1 - t0, "loss_s": t2 - t1, "backward_s": t3 - t2,
            "sample": f"1 of the 8 C4 views (3M Gaussians, 2048x1024): oracle render + photometric loss "
                      f"(lambda 0.2) + backward, StdMath double, threads = all {cores} host threads; "
                      f"iters/s = 1 / (8 x view time)"}


def run_aux(args, ctx, dev, stream):
    """The other BASELINE configs on this GPU (device-resident, CUDA events): C1 render
    throughput (the reference's own test workload, 100K Gaussians at 1024x512) and the C2
    forward + backward step (500K Gaussians, SH degree 3, 2048x1024)."""
    import numpy as np
    import torch
    from paper_2410_20686_b200 import GaussianCloud, RenderOutput, RenderSettings, backward, render, scenes

    def on_dev(c):
        d = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        return GaussianCloud(d(c.means), d(c.rotations), d(c.log_scales), d(c.raw_opacities), d(c.colors),
                             c.sh_degree, d(c.sh_rest))

    def timed(fn, reps):
        for k in range(2):
            fn(k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for k in range(reps):
            fn(k)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    s = RenderSettings()
    fr = RenderOutput(ctx)
    c1 = on_dev(scenes.cloud_c1())
    ms1 = timed(lambda k: render(ctx, c1, scenes.yaw_camera(0.1 * k, 1024, 512), s, out=fr), 20)
    c2 = on_dev(scenes.cloud_c2())
    dl = torch.from_numpy(np.random.default_rng(2004).uniform(-1, 1, 3 * 2048 * 1024).astype(np.float32)).to(dev)
    from paper_2410_20686_b200 import GradBuffers
    n2 = c2.n
    z = lambda *sh: torch.zeros(sh, dtype=torch.float32, device=dev)
    g2 = GradBuffers(z(3, n2), z(4, n2), z(3, n2), z(n2), z(3, n2), z(n2), z(n2),
                     torch.zeros(n2, dtype=torch.int32, device=dev), z(15, 3, n2))

    def step2(k):
        cam = scenes.yaw_camera(0.1 * k, 2048, 1024)
        render(ctx, c2, cam, s, out=fr)
        backward(ctx, c2, cam, fr, dl, s, grads=g2)

    ms2 = timed(step2, 5)
    fr.check()
    fr.destroy()
    return {"C1_render": {"workload": "100K Gaussians (default bounds), SH0, 1024x512", "ms": ms1,
                          "frames_per_s": 1000.0 / ms1},
            "C2_fwd_bwd": {"workload": "500K Gaussians, SH degree 3, 2048x1024, render + backward", "ms": ms2,
                           "steps_per_s": 1000.0 / ms2}}


def run_large(args, ctx, rank, world, local_rank, dev, stream):
    """BASELINE config 5: 10M Gaussians at 4096x2048, rank r renders ERP rows
    [r*H/G, (r+1)*H/G) (odgs_render_band; each band is bit-identical to the full render's
    rows) and the bands are all-gathered over NCCL into the full image."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2410_20686_b200 import GaussianCloud, RenderOutput, RenderSettings, render_band, scenes
    from paper_2410_20686_b200 import _capi as capi

    W, H, n = 4096, 2048, 10_000_000
    src = scenes.cloud_c5(n)
    cloud = GaussianCloud(*[torch.from_numpy(np.ascontiguousarray(getattr(src, k))).to(dev)
                            for k in ("means", "rotations", "log_scales", "raw_opacities", "colors")])
    del src
    rows = H // world
    r0, r1 = rank * rows, (rank + 1) * rows
    settings = RenderSettings()
    fr = RenderOutput(ctx)
    # The all-gather of the bands is fused into the blend: each rank's blend writes its
    # rows straight into every rank's full-image buffer over NVLink (CUDA IPC peer
    # pointers, paper_2410_20686_b200/peers.py); one barrier then completes the frame.
    # Should the peer set-up fail, NCCL's all_gather is the fallback.
    gather, gathered, collective = None, None, "none"
    if world > 1:
        failure = None
        try:
            from paper_2410_20686_b200.peers import BandGather
            gather = BandGather(ctx, fr, W, H, dev)
        except Exception as e:  # noqa: BLE001 — reported in the JSON line
            failure = type(e).__name__
        # Every rank must take the same path: the fused gather only if it set up everywhere.
        ok = torch.tensor([0 if failure else 1], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 1:
            collective = "fused: blend writes its band into every rank's image over NVLink (CUDA IPC), 1 barrier"
        else:
            if gather is not None:
                gather.close()
                gather = None
            gathered = torch.empty((world, 3, W, rows), dtype=torch.float32, device=dev)
            collective = f"NCCL all_gather of the band images (peer set-up failed: {failure or 'on another rank'})"

    def frame(k):
        if gather is not None:
            gather.begin()  # this frame's bands go to the other image buffer of every rank
        render_band(ctx, cloud, scenes.yaw_camera(2 * math.pi * k / 16, W, H), settings, r0, r1, out=fr)
        if gather is not None:
            gather.sync(local_rank)
        elif gathered is not None:
            band = _device_view(fr.device_ptr(capi.FRAME_IMAGE), 3 * W * H, dev).view(3, W, H)[:, :, r0:r1]
            dist.all_gather_into_tensor(gathered, band.contiguous())

    for k in range(2):
        frame(k)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier(device_ids=[local_rank])
    steps = max(3, min(args.steps, 10))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for k in range(steps):
        frame(k)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if fr.check():
        raise RuntimeError("bench: a C5 frame overflowed its entry buffers")
    # stage times from a separate profiled pass (its event readbacks stay out of the timing)
    ctx.set_profiling(True)
    ctx.reset_stage_times()
    for k in range(2):
        frame(k)
    torch.cuda.synchronize()
    stages = {k: round(v[0] / 2, 4) for k, v in ctx.stage_times().items() if v[1] > 0}
    ctx.set_profiling(False)
    info = fr.info()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    out = {"metric": "ERP frames/sec (C5: 10M Gaussians, 4096x2048, row bands over the GPUs)",
           "value": steps / (ms_max / 1000.0), "unit": "frames/s", "ms_per_frame": ms_max / steps,
           "bands": world, "rows_per_band": rows, "n_gpus": world, "scaling": "strong",
           "collective": collective,
           "band_tile_entries_rank0": info.n_entries, "stage_ms_per_frame_rank0": stages}
    if world == 1:
        # Each of the 8 bands an 8-GPU run would give one rank, rendered alone on this GPU
        # (CUDA events, same frames): the per-rank work of the row-band split, without
        # the all-gather (8 x 12.6 MB over NVLink).
        band_ms = []
        for b in range(8):
            b0, b1 = b * (H // 8), (b + 1) * (H // 8)
            for k in range(2):
                render_band(ctx, cloud, scenes.yaw_camera(2 * math.pi * k / 16, W, H), settings, b0, b1, out=fr)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for k in range(3):
                render_band(ctx, cloud, scenes.yaw_camera(2 * math.pi * k / 16, W, H), settings, b0, b1, out=fr)
            e1.record(stream)
            torch.cuda.synchronize()
            band_ms.append(e0.elapsed_time(e1) / 3)
        out["bands8_single_gpu_ms"] = [round(v, 4) for v in band_ms]
        out["bands8_slowest_band_fps"] = 1000.0 / max(band_ms)
    if gather is not None:
        gather.close()
    fr.destroy()
    return out


def _device_view(ptr: int, numel: int, dev):
    """A float32 torch view of device memory owned by the library (no copy)."""
    import torch

    class _Holder:
        pass

    h = _Holder()
    h.__cuda_array_interface__ = {"shape": (numel,), "typestr": "<f4", "data": (ptr, False), "version": 2}
    return torch.as_tensor(h, device=dev)


SHARE_GPU = os.environ.get("ODGS_BENCH_SHARE_GPU") == "1"  # test mode: every rank on GPU 0, gloo


def rank_barrier(local_rank: int) -> None:
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        dist.barrier(device_ids=[local_rank])
    else:
        dist.barrier()


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` started without a launcher: re-executes itself under
    torch.distributed.run with N ranks (one process per GPU) on 127.0.0.1."""
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = 0 if SHARE_GPU else int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}")
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if SHARE_GPU:  # NCCL refuses two ranks on one GPU; gloo moves the CUDA tensors
            dist.init_process_group("gloo")
        else:
            if torch.cuda.device_count() < world:
                raise SystemExit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} visible GPUs")
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (nRanks) on stderr
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        assert dist.get_world_size() == world
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Multi-process (world_size 2, gloo, CPU) checks of the view-sharded training step's
host logic (paper_2410_20686_b200/train.py): every view is assigned exactly once, and
the all-reduced flat gradient buffer equals the single-process sum over all views
(GradBuffers::accumulate semantics, backward.hpp:364-373; test_backward.cpp:536-556).
Per-view gradients come from the fp64 oracle, so this runs without a GPU."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_lib
from paper_2410_20686_b200.train import FLAT_LAYOUT, FLAT_WIDTH, allreduce_grads, assign_views, flat_views

N_VIEWS, W, H = 4, 64, 32
FD_BOUNDS = (0.8, 10.0, 75.0 * math.pi / 180.0, 0.1, 0.7, 0.02, 0.12)


def test_assign_views_partitions_every_view_once():
    for world in range(1, 9):
        for n in (1, 3, 8, 13):
            got = sorted(v for r in range(world) for v in assign_views(n, r, world))
            assert got == list(range(n))


def view_grads(arrs, v):
    """(flat float64 16n, observed int32 n) for view v from the fp64 oracle."""
    a = 2 * math.pi * v / N_VIEWS
    R = np.array([[math.cos(a), 0, -math.sin(a)], [0, 1, 0], [math.sin(a), 0, math.cos(a)]])
    t = np.array([0.05 * math.cos(a), 0.02 * (v % 2), 0.05 * math.sin(a)])
    s = oracle_lib.OracleSettings(cutoff=8.0)
    fr = oracle_lib.render(arrs, R, t, W, H, s, dbl=True)
    dl = np.random.default_rng(100 + v).uniform(-1, 1, 3 * W * H)
    fr.backward(dl)
    n = arrs[3].shape[0]
    flat = np.concatenate([fr.get("g_" + name) for name, _ in FLAT_LAYOUT])
    assert flat.size == FLAT_WIDTH * n
    return flat, fr.get("g_observed")


def _worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    arrs = oracle_lib.random_cloud(211, 12, FD_BOUNDS)
    n = arrs[3].shape[0]
    flat = torch.zeros(FLAT_WIDTH * n, dtype=torch.float64)
    obs = torch.zeros(n, dtype=torch.int32)
    for v in assign_views(N_VIEWS, rank, world):
        f, o = view_grads(arrs, v)
        flat += torch.from_numpy(f)
        obs += torch.from_numpy(o)
    allreduce_grads(flat, obs)
    if rank == 0:
        result_q.put((flat.numpy().copy(), obs.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_allreduce_equals_single_process_sum():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    flat, obs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    arrs = oracle_lib.random_cloud(211, 12, FD_BOUNDS)
    ref_flat = np.zeros_like(flat)
    ref_obs = np.zeros_like(obs)
    for v in range(N_VIEWS):
        f, o = view_grads(arrs, v)
        ref_flat += f
        ref_obs += o
    assert np.array_equal(obs, ref_obs)
    assert np.allclose(flat, ref_flat, rtol=1e-12, atol=1e-15)
    views = flat_views(torch.from_numpy(flat), 12)
    assert views["means"].shape == (3, 12) and views["one_minus_cos"].shape == (12,)

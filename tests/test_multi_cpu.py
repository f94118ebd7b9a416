"""Multi-process host logic of the sharded paths, world_size 2 over gloo on CPU."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2201_10887_b200 import multi


def test_shard_views_cover_exactly_once():
    for world in (1, 2, 3, 8):
        seen = sorted(v for r in range(world) for v in multi.shard_views(64, world, r))
        assert seen == list(range(64))


def test_screen_strips_partition_and_balance():
    for world in (1, 2, 4, 8):
        s = multi.screen_strips(3840, world)
        assert s[0][0] == 0 and s[-1][1] == 3840
        assert all(a[1] == b[0] for a, b in zip(s, s[1:]))
        assert all(x0 % multi.TILE_W == 0 for x0, _ in s)
    # a cost map concentrated on the right half pushes the cuts right
    tw, th = multi.TILE_W, multi.TILE_H
    cost = np.zeros((1080 // th) * (1920 // tw))
    cost.reshape(1080 // th, 1920 // tw)[:, 960 // tw:] = 10.0
    s = multi.balance_strips(cost, 1920, 1080, 4)
    assert s[0][1] > 960 and s[-1][1] == 1920


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    H, W = 6, 37
    rects = multi.screen_strips(W, world)
    full = (np.arange(H * W * 3) % 251).astype(np.uint8).reshape(H, W, 3)
    x0, x1 = rects[rank]
    strip = torch.from_numpy(full[:, x0:x1].copy())
    out = multi.gather_strips(strip, rects, rank, world)
    # weak-scaling timing reduction used by bench.py: max over ranks
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((bool(np.array_equal(out.numpy(), full)), float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gather_strips_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    ok, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert ok and tmax == float(world)

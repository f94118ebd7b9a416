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
    # the sharded frame's exchange: each rank's computed entries, -inf elsewhere; the
    # MAX all-reduce must leave every rank with every entry
    rng = np.random.default_rng(5)
    truth = rng.normal(size=4096).astype(np.float32)
    truth[::7] = -np.float32(rng.normal(size=truth[::7].size)) ** 2   # negated minima
    owner = rng.integers(0, world, truth.size)
    extra = rng.random(truth.size) < 0.3                    # blocks computed by two ranks
    mine = (owner == rank) | (extra & (owner == (rank + 1) % world))
    xchg = torch.from_numpy(np.where(mine, truth, -np.inf).astype(np.float32))
    multi.all_reduce_max(xchg)
    xchg_ok = bool(np.array_equal(xchg.numpy(), truth))
    # C4 view batch: 5 views over the ranks, gathered to rank 0 in view order
    n_views = 5
    mine = multi.shard_views(n_views, world, rank)
    frames = [torch.full((3, 4, 3), v, dtype=torch.uint8) for v in mine]
    views = multi.gather_views(frames, n_views, rank, world)
    views_ok = views is None if rank else [int(f[0, 0, 0]) for f in views] == list(range(n_views))
    # weak-scaling timing reduction used by bench.py: max over ranks
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put((bool(np.array_equal(out.numpy(), full)) and xchg_ok and views_ok, float(t.item())))
    else:
        assert out is None and xchg_ok and views_ok
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


def _block_selected(fp_args, s, x0, y0, x1, y1, blk_id):
    """Host twin of hc_discretize.cu block_selected for strip s."""
    apex, wedges = fp_args
    meets = lambda r: wedges[r][0] or multi.square_meets_wedge(x0, y0, x1, y1, apex, wedges[r][1], wedges[r][2])
    if meets(s):
        return True
    if any(meets(r) for r in range(len(wedges)) if r != s):
        return False
    return blk_id % len(wedges) == s


def _cameras():
    from paper_2201_10887_b200.cascade import CameraView
    from paper_2201_10887_b200.configs import CONFIGS
    cams = [CONFIGS[n].path_camera(i) for n in ("C2", "C5") for i in (0, 30, 60)]
    rng = np.random.default_rng(11)
    for _ in range(6):
        eye = (float(rng.uniform(-300, 2300)), float(rng.uniform(-300, 2300)), float(rng.uniform(20, 900)))
        tgt = (float(rng.uniform(200, 1800)), float(rng.uniform(200, 1800)), 0.0)
        cams.append(CameraView(eye=eye, look_dir=tuple(b - a for a, b in zip(eye, tgt)), up=(0.0, 0.0, 1.0),
                               fov_y=float(rng.uniform(30, 100)), aspect=16 / 9, near_clip=1.0, far_clip=6000.0))
    # straight down: every strip may reach the whole plane
    cams.append(CameraView(eye=(1000.0, 1000.0, 500.0), look_dir=(1e-9, 0.0, -1.0), up=(0.0, 1.0, 0.0),
                           fov_y=60.0, aspect=16 / 9, near_clip=1.0, far_clip=6000.0))
    return cams


def test_strip_wedges_contain_every_ray_and_blocks_are_covered():
    """Every pixel ray of a strip stays inside its wedge (sampled along the ray on the
    ground), so the blocks it crosses are selected by its rank; and every block of a
    cascade is selected by at least one rank (block_selected's host twin)."""
    from paper_2201_10887_b200.render import camera_ray_dirs
    W, H = 384, 216
    for cam in _cameras():
        dirs = camera_ray_dirs(cam, W, H)
        for world in (2, 3, 8):
            rects = multi.screen_strips(W, world)
            wedges = multi.strip_wedges(cam, W, H, rects)
            apex = (float(cam.eye[0]), float(cam.eye[1]))
            for s, ((x0, x1), (whole, d0, d1)) in enumerate(zip(rects, wedges)):
                if whole:
                    continue
                d = dirs[::9, x0:x1:3].reshape(-1, 3)
                for tt in (1.0, 37.0, 400.0, 5000.0):
                    px = apex[0] + tt * d[:, 0]
                    py = apex[1] + tt * d[:, 1]
                    # a point on the ray: a degenerate square must meet the wedge
                    for x, y in zip(px[::17], py[::17]):
                        assert multi.square_meets_wedge(x - 1e-6, y - 1e-6, x + 1e-6, y + 1e-6, apex, d0, d1)
            # coverage of a synthetic 512^2 cascade (16 x 16 blocks of 32 texels, 2 m texels)
            org, tex = (apex[0] - 400.0, apex[1] - 300.0), 2.0
            fp = (apex, wedges)
            for by in range(16):
                for bx in range(16):
                    sq = (org[0] + (32 * bx - 2.5) * tex, org[1] + (32 * by - 2.5) * tex,
                          org[0] + (32 * bx + 34.5) * tex, org[1] + (32 * by + 34.5) * tex)
                    assert any(_block_selected(fp, r, *sq, by * 16 + bx) for r in range(world))


def test_strip_wedge_of_full_width_view_is_the_view():
    """One strip = the whole image: the wedge is the horizontal field of view."""
    import math
    from paper_2201_10887_b200.cascade import CameraView
    cam = CameraView(eye=(0.0, 0.0, 100.0), look_dir=(1.0, 0.0, -0.2), up=(0.0, 0.0, 1.0), fov_y=60.0,
                     aspect=2.0, near_clip=1.0, far_clip=6000.0)
    (whole, d0, d1), = multi.strip_wedges(cam, 1000, 500, [(0, 1000)])
    assert not whole
    a0, a1 = math.atan2(d0[1], d0[0]), math.atan2(d1[1], d1[0])
    assert a0 < 0 < a1 and abs(a0 + a1) < 1e-6


def test_strip_balancer_converges_on_uneven_cost():
    """Strips cut from measured per-rank times converge to equal cost on a cost
    profile with a heavy band (the horizon's long rays), cuts snapped to tiles and at
    least min_width apart, identical for identical inputs (every rank computes them)."""
    W, world = 3840, 8
    x = np.arange(W) + 0.5
    density = 1.0 + 30.0 * np.exp(-((x - 2100.0) / 250.0) ** 2)
    bal = multi.StripBalancer(W, world)
    cost = lambda rects: np.array([density[a:b].sum() for a, b in rects])
    first = cost(bal.rects)
    for _ in range(12):
        bal.update(cost(bal.rects))
    last = cost(bal.rects)
    assert last.max() / last.mean() < 0.6 * (first.max() / first.mean())
    assert last.max() / last.mean() < 1.35
    xs = [a for a, _ in bal.rects] + [W]
    assert xs[0] == 0 and xs[-1] == W
    assert all(b - a >= bal.min_width for a, b in bal.rects)
    assert all(a % multi.TILE_W == 0 for a, _ in bal.rects)
    twin = multi.StripBalancer(W, world)
    for _ in range(12):
        twin.update(cost(twin.rects))
    assert twin.rects == bal.rects
    # missing / invalid measurements leave the cuts alone
    before = list(bal.rects)
    assert bal.update([0.0] * world) == before and bal.update([1.0] * (world - 1)) == before

"""Multi-GPU partitioning of the frame path (SURVEY.md §8 e), one process per GPU.

* camera batches (C4): views are independent; rank r renders views
  r, r+N, r+2N, ... of a batch against the grid resident in its own HBM.
  `shard_views` assigns them; no data-path collective, weak scaling;
  `gather_views` collects a batch's frames on one rank when the caller wants
  them there (one gather per round of views).
* screen strips (C5): every rank plans the SAME full-view cascades (the host
  planner is deterministic) and traces only its vertical strip of pixels
  (`HcRenderArgs.x0..x1`).  Each rank builds its own cascades: it discretizes
  only the 32x32-texel blocks its strip's rays can reach -- the blocks that meet
  the strip's ground wedge (`strip_footprint`), dilated by 2.5 texels -- plus a
  round-robin share of the blocks no strip reaches.  The traversal's slab clip
  needs the global valid range (render.py:127,144, _kernels.py:105-115) and its
  upper mip levels need every block, so stage 1 of the frame writes each block's
  level-5 max-mip nodes and valid-height partials to an exchange buffer and ONE
  NCCL all-reduce (MAX, ~0.3 MB at C5) combines the ranks' buffers; stage 2
  builds mip levels >= 6 and the valid ranges from it and traces the strip.
  Every node and texel a strip ray reads then holds its single-GPU value, so
  strips are bit-identical to the full frame (heightcast.h HcFootprint).  The
  image is gathered to rank 0 (`gather_strips`, NCCL over NVLink; gloo on CPU).
  Strip widths can be rebalanced from per-tile costs (`balance_strips`).
"""

from __future__ import annotations

import numpy as np

TILE_W, TILE_H = 8, 4          # render-kernel pixel tile (hc_render.cu TILE_W/TILE_H)


def shard_views(n_views: int, world: int, rank: int) -> list[int]:
    """Round-robin view assignment for camera batches."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return list(range(rank, n_views, world))


def gather_views(frames, n_views: int, rank: int, world: int, group=None, dst: int = 0):
    """Collect a view batch on `dst`: rank r holds the (H, W, 3) uint8 frames of views
    shard_views(n_views, world, r), in that order.  One gather per round of views
    (round i: view i*world + r from every rank; ranks without a view that round send
    a zero frame); returns the list of n_views frames on `dst`, None elsewhere."""
    import torch
    import torch.distributed as dist
    mine = shard_views(n_views, world, rank)
    if len(frames) != len(mine):
        raise ValueError(f"rank {rank} holds {len(frames)} frames for {len(mine)} views")
    if not frames:
        raise ValueError("every rank needs at least one view (n_views >= world)")
    like = frames[0]
    out = [None] * n_views if rank == dst else None
    rounds = (n_views + world - 1) // world
    for i in range(rounds):
        send = frames[i] if i < len(frames) else torch.zeros_like(like)
        parts = [torch.empty_like(like) for _ in range(world)] if rank == dst else None
        dist.gather(send.contiguous(), parts, dst=dst, group=group)
        if rank == dst:
            for r, p in enumerate(parts):
                v = i * world + r
                if v < n_views:
                    out[v] = p
    return out


def screen_strips(width: int, world: int, weights=None) -> list[tuple[int, int]]:
    """Contiguous vertical strips [x0, x1) covering [0, width), one per rank.

    With `weights` (a per-column cost estimate, e.g. the previous frame's
    per-tile costs summed over rows) strips are cut at equal cumulative cost;
    cuts are snapped to multiples of 8 pixels (the render kernel's tile width)."""
    if world < 1 or width < 1:
        raise ValueError("bad width/world")
    if weights is None:
        cuts = [round(width * r / world) for r in range(world + 1)]
    else:
        w = np.asarray(weights, dtype=np.float64)
        if len(w) != width:
            raise ValueError("weights must have one entry per pixel column")
        c = np.concatenate([[0.0], np.cumsum(np.maximum(w, 0.0) + 1e-12)])
        cuts = [int(np.searchsorted(c, c[-1] * r / world)) for r in range(world + 1)]
    cuts = [min(width, max(0, TILE_W * round(x / TILE_W))) for x in cuts]
    cuts[0], cuts[-1] = 0, width
    for i in range(1, len(cuts)):
        cuts[i] = max(cuts[i], cuts[i - 1])
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def balance_strips(tile_cost, width: int, height: int, world: int, tile_w: int = None, tile_h: int = None):
    """Strip cuts from a per-tile cost map (row-major tiles of tile_w x tile_h pixels)."""
    tile_w = TILE_W if tile_w is None else tile_w
    tile_h = TILE_H if tile_h is None else tile_h
    tx = (width + tile_w - 1) // tile_w
    ty = (height + tile_h - 1) // tile_h
    cost = np.asarray(tile_cost, dtype=np.float64)[:tx * ty].reshape(ty, tx).sum(axis=0)
    cols = np.repeat(cost / tile_w, tile_w)[:width]
    return screen_strips(width, world, cols)


def gather_strips(strip: "torch.Tensor", rects, rank: int, world: int, group=None, dst: int = 0):
    """Assemble per-rank (H, x1-x0, 3) uint8 strips into one (H, W, 3) image on `dst`.

    A gather to `dst` only (the other ranks send their strip once) of equally padded
    strips; works with NCCL device tensors and gloo host tensors.  Returns the image
    on `dst`, None elsewhere."""
    import torch
    import torch.distributed as dist
    H = strip.shape[0]
    wmax = max(x1 - x0 for x0, x1 in rects)
    padded = torch.zeros((H, wmax, 3), dtype=strip.dtype, device=strip.device)
    padded[:, :strip.shape[1]] = strip
    parts = [torch.empty_like(padded) for _ in range(world)] if rank == dst else None
    dist.gather(padded, parts, dst=dst, group=group)
    if rank != dst:
        return None
    W = rects[-1][1]
    out = torch.empty((H, W, 3), dtype=strip.dtype, device=strip.device)
    for (x0, x1), p in zip(rects, parts):
        out[:, x0:x1] = p[:, :x1 - x0]
    return out


class StripBalancer:
    """Cost-balanced screen strips from measured per-rank frame times.

    A strip's cost is modelled as uniform over its columns (its time / its width);
    the next cuts split the image at equal modelled cost (`screen_strips` with
    per-column weights), moved only `damping` of the way from the old cuts so they
    do not oscillate while the view moves, and kept at least `min_width` pixels
    apart.  Every rank feeds the same times (exchanged in the frame's all-reduce, see
    `StripFrame.times_slot`), so every rank computes the same cuts."""

    def __init__(self, width: int, world: int, damping: float = 0.7, min_width: int = 4 * TILE_W):
        self.width, self.world, self.damping = width, world, damping
        self.min_width = min(min_width, max(TILE_W, width // max(world, 1) // TILE_W * TILE_W))
        self.rects = screen_strips(width, world)

    def update(self, times):
        t = np.asarray(times, dtype=np.float64)
        if self.world < 2 or len(t) != self.world or not np.all(np.isfinite(t)) or np.any(t <= 0):
            return self.rects
        cols = np.empty(self.width)
        for (x0, x1), ti in zip(self.rects, t):
            cols[x0:x1] = ti / max(x1 - x0, 1)
        target = screen_strips(self.width, self.world, cols)
        old = [x0 for x0, _ in self.rects] + [self.width]
        new = [x0 for x0, _ in target] + [self.width]
        cuts = [0]
        for r in range(1, self.world):
            c = (1.0 - self.damping) * old[r] + self.damping * new[r]
            c = TILE_W * int(round(c / TILE_W))
            lo = cuts[-1] + self.min_width
            hi = self.width - (self.world - r) * self.min_width
            cuts.append(min(max(c, lo), hi))
        cuts.append(self.width)
        self.rects = [(cuts[r], cuts[r + 1]) for r in range(self.world)]
        return self.rects


FOOTPRINT_MARGIN = 2.5        # texels of dilation of a block's square (SURVEY.md §8 e)
_WIDEN = 1e-9                  # radians: each wedge boundary turned outward


def strip_wedges(camera, width: int, height: int, rects):
    """Ground wedges of screen strips: for strip [x0, x1) the 2D directions of all its
    pixel rays (render.py:100-110: d = look + xs right + ys up, any ys of the image)
    lie between two boundary directions.  Returns [(all_plane, d0, d1)] per strip:
    the image of the strip's (xs, ys) rectangle under d -> d_xy is a parallelogram
    whose cone from the origin is spanned by its corners; if the corners do not fit
    in an open half-plane (the view looks nearly straight down, or the strip spans
    >= 180 degrees) the strip may reach the whole plane."""
    import math
    right, up, look = camera.basis()
    th = math.tan(math.radians(camera.fov_y) / 2.0)
    ys = ((1.0 - (0.5 / height) * 2.0) * th, (1.0 - ((height - 0.5) / height) * 2.0) * th)
    out = []
    for x0, x1 in rects:
        if x1 <= x0:
            out.append((True, (1.0, 0.0), (0.0, 1.0)))
            continue
        xs = ((((x0 + 0.5) / width) * 2.0 - 1.0) * th * camera.aspect,
              (((x1 - 0.5) / width) * 2.0 - 1.0) * th * camera.aspect)
        c = [np.asarray(look, dtype=np.float64) + x * right + y * up for x in xs for y in ys]
        c2 = np.array([v[:2] for v in c])
        scale = max(float(np.linalg.norm(v)) for v in c)
        n2 = np.linalg.norm(c2, axis=1)
        if np.any(n2 <= 1e-6 * scale):
            out.append((True, (1.0, 0.0), (0.0, 1.0)))
            continue
        base = c2[0] / n2[0]
        ang = [math.atan2(base[0] * v[1] - base[1] * v[0], base[0] * v[0] + base[1] * v[1]) for v in c2]
        lo, hi = min(ang) - _WIDEN, max(ang) + _WIDEN
        if hi - lo >= math.pi - 1e-6:
            out.append((True, (1.0, 0.0), (0.0, 1.0)))
            continue
        rot = lambda a: (base[0] * math.cos(a) - base[1] * math.sin(a), base[0] * math.sin(a) + base[1] * math.cos(a))
        out.append((False, rot(lo), rot(hi)))
    return out


def strip_footprint(camera, width: int, height: int, rects, rank: int, margin: float = FOOTPRINT_MARGIN):
    """HcFootprint of `rank` among the strips `rects` (the C struct of heightcast.h)."""
    from . import _cuda
    if not 0 <= rank < len(rects) or len(rects) > _cuda.HC_MAX_STRIPS:
        raise ValueError(f"rank {rank} of {len(rects)} strips (max {_cuda.HC_MAX_STRIPS})")
    fp = _cuda.HcFootprint()
    fp.n_strips, fp.rank, fp.margin = len(rects), rank, float(margin)
    fp.apex[0], fp.apex[1] = float(camera.eye[0]), float(camera.eye[1])
    for s, (whole, d0, d1) in enumerate(strip_wedges(camera, width, height, rects)):
        fp.all[s] = 1 if whole else 0
        fp.dir[s][0][0], fp.dir[s][0][1] = d0
        fp.dir[s][1][0], fp.dir[s][1][1] = d1
    return fp


def square_meets_wedge(x0, y0, x1, y1, apex, d0, d1) -> bool:
    """Host twin of the kernel's block test (hc_discretize.cu square_meets_wedge)."""
    D = (d0, d1)
    cs = ((x0, y0), (x1, y0), (x0, y1), (x1, y1))
    for e in range(2):
        nx, ny = -D[e][1], D[e][0]
        if nx * D[1 - e][0] + ny * D[1 - e][1] > 0.0:
            nx, ny = -nx, -ny
        if all(nx * (cx - apex[0]) + ny * (cy - apex[1]) > 0.0 for cx, cy in cs):
            return False
    inf = float("inf")
    xlo = -inf if (d0[0] < 0 or d1[0] < 0) else apex[0]
    xhi = inf if (d0[0] > 0 or d1[0] > 0) else apex[0]
    ylo = -inf if (d0[1] < 0 or d1[1] < 0) else apex[1]
    yhi = inf if (d0[1] > 0 or d1[1] > 0) else apex[1]
    return not (x1 < xlo or x0 > xhi or y1 < ylo or y0 > yhi)


def exchange_floats(settings) -> int:
    from . import _cuda
    return int(_cuda.lib().hc_frame_xchg_floats(settings.count, settings.resolution))


def all_reduce_max(xchg, group=None):
    """The sharded frame's one collective: elementwise MAX of the ranks' exchange buffers."""
    import torch.distributed as dist
    dist.all_reduce(xchg, op=dist.ReduceOp.MAX, group=group)


class StripFrame:
    """One rank's screen strip of a frame, in two stages around the exchange
    (heightcast.h hc_frame_stage).  `stage1()` plans and enqueues the footprint
    discretization; the caller MAX-reduces `xchg` across ranks; `stage2()` enqueues
    the upper mips, valid ranges and the strip's rays.  Pixels land in the frame
    buffers' `rgb[:, x0:x1]`."""

    def __init__(self, config, grid, table, settings, rects, rank, slot=0, debug=False, events=None,
                 staged=None):
        import torch
        from .render import prepare_frame
        self.rects, self.rank = rects, rank
        self.rect = (rects[rank][0], 0, rects[rank][1], config.height)
        self.events = events
        self.prep = prepare_frame(config, grid, table, settings, debug, slot)
        self.visible = self.prep is not None
        self.world = len(rects)
        # one strip renders as a plain frame unless `staged` forces the exchange stages
        self.staged = self.world > 1 if staged is None else bool(staged)
        if not self.visible:
            return
        self.buf, self.plan, self.plan_ms, self._launch = self.prep
        n = exchange_floats(settings)
        if self.staged and n == 0:
            raise ValueError("screen-strip sharding needs cascades of at least 34 texels (7 mip levels)")
        # the exchange buffer, plus one float per rank after it: each rank's last
        # measured frame time rides in the same MAX all-reduce (StripBalancer input)
        total = n + _cuda_max_strips()
        xb = getattr(self.buf, "_xchg", None)
        if xb is None or xb.numel() != total:
            xb = self.buf._xchg = torch.zeros(total, dtype=torch.float32, device=self.buf.rgb.device)
        self.xchg = xb
        self.times_slot = xb[n:n + self.world]
        self.footprint = strip_footprint(config.camera, config.width, config.height, rects, rank)

    def stage1(self):
        if not self.staged:          # a whole frame: no exchange
            self._launch(rect=self.rect, events=self.events)
        else:
            self._launch(rect=self.rect, events=self.events, stage=1, footprint=self.footprint, xchg=self.xchg)

    def stage2(self):
        if self.staged:
            self._launch(rect=self.rect, events=self.events, stage=2, footprint=self.footprint, xchg=self.xchg)

    def strip(self):
        x0, _, x1, _ = self.rect
        return self.buf.rgb[:, x0:x1]


class StripSequence:
    """This rank's screen strips of a sequence of frames (a camera path), with the
    strips rebalanced from the ranks' measured frame times.

    Each rank writes the time of its newest completed frame into the exchange
    buffer's time slots, which ride in the frame's one MAX all-reduce; step i cuts
    the image with the times exchanged at step i - LAG, so every rank changes its
    cuts at the same step and none waits on a frame still in flight.  With one rank
    the frame is a plain full frame."""

    LAG = 2

    def __init__(self, width: int, world: int, rank: int, balance: bool = True):
        self.world, self.rank, self.balance = world, rank, balance and world > 1
        self.balancer = StripBalancer(width, world)
        self._pending = {}
        self._own = []
        self._last_ms = 0.0
        self._step = 0

    @property
    def rects(self):
        return self.balancer.rects

    def frame(self, config, grid, table, settings, events=None, reduce=all_reduce_max):
        """Enqueue this rank's strip of `config` (both stages and the exchange);
        returns the StripFrame (pixels in `frame.strip()` once the stream gets there)."""
        import torch
        i = self._step
        self._step += 1
        if self.balance and (i - self.LAG) in self._pending:
            ev, host = self._pending.pop(i - self.LAG)
            ev.synchronize()
            self.balancer.update(host.numpy())
        while self._own and self._own[0][1].query():
            e0, e1 = self._own.pop(0)
            self._last_ms = e0.elapsed_time(e1)
        f = StripFrame(config, grid, table, settings, self.balancer.rects, self.rank, events=events)
        if not f.visible:
            return f
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        f.stage1()
        if f.staged:
            f.times_slot.zero_()
            f.times_slot[self.rank:self.rank + 1].fill_(self._last_ms)
            reduce(f.xchg)
            if self.balance:
                host = torch.empty(self.world, dtype=torch.float32, pin_memory=True)
                host.copy_(f.times_slot, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record()
                self._pending[i] = (ev, host)
        f.stage2()
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        self._own.append((e0, e1))
        return f


def _cuda_max_strips() -> int:
    from . import _cuda
    return _cuda.HC_MAX_STRIPS


def render_strip(config, grid, table, params, settings, rect, rects=None, rank=None, reduce=all_reduce_max):
    """Render pixel columns rect=(x0, x1) of the full frame on this rank's GPU.

    With `rects` (every rank's strip) and `rank`, the frame is sharded: this rank
    discretizes only its strip's footprint and `reduce(xchg)` (default: NCCL/gloo
    all-reduce MAX over the default group) combines the ranks' mip exchange
    buffers.  Without them the rank computes the full cascades (no collective).
    Returns the (H, x1-x0, 3) uint8 device tensor (a copy), or None if nothing is
    visible (the same on every rank: the plan is deterministic)."""
    if table.sigma != params.sigma:
        raise ValueError("influence table was built for a different sigma")
    if rects is None:
        rects, rank = [tuple(rect)], 0
    elif tuple(rects[rank]) != tuple(rect):
        raise ValueError("rect is not rects[rank]")
    f = StripFrame(config, grid, table, settings, rects, rank)
    if not f.visible:
        return None
    f.stage1()
    if f.staged:
        reduce(f.xchg)
    f.stage2()
    return f.strip().clone()


def render_strips_one_gpu(config, grid, table, params, settings, world: int, rects=None):
    """All `world` ranks of a sharded frame emulated on this GPU one after the other
    (stage 1 of every rank, the MAX reduction as torch.maximum, stage 2 of every
    rank): the (H, W, 3) image assembled from the strips, and each rank's frame
    counters (HC_CNT_*: its texels, pairs, rays).  For parity tests; nothing waits on another rank."""
    import torch
    rects = rects or screen_strips(config.width, world)
    frames = [StripFrame(config, grid, table, settings, rects, r, slot=r) for r in range(world)]
    if not frames[0].visible:
        return None, None
    for f in frames:
        f.stage1()
    if frames[0].staged:
        red = frames[0].xchg.clone()
        for f in frames[1:]:
            torch.maximum(red, f.xchg, out=red)
        for f in frames:
            f.xchg.copy_(red)
    for f in frames:
        f.stage2()
    img = torch.cat([f.strip() for f in frames], dim=1).cpu().numpy()
    counters = [f.buf.counters.cpu().numpy().copy() for f in frames]
    return img, counters

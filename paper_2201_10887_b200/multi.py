"""Multi-GPU partitioning of the frame path (SURVEY.md §8 e), one process per GPU.

Two decompositions, both without a data-path collective:

* camera batches (C4): views are independent; rank r renders views
  r, r+N, r+2N, ... of a batch against the grid resident in its own HBM.
  `shard_views` assigns them; throughput scales weakly.
* screen strips (C5): every rank plans the SAME full-view cascades (the host
  planner is deterministic) and discretizes the full cascades, so its rasters,
  pyramids and valid ranges equal the single-GPU ones bit for bit -- the
  traversal's slab clip needs the global valid range (render.py:127,144), which
  this gets without any all-reduce -- then traces only its vertical strip of
  pixels (`HcRenderArgs.x0..x1`).  Strip widths can be rebalanced from per-strip
  costs (`balance_strips`).  The only collective is the optional image gather to
  rank 0 at the end of the frame (`gather_strips`, NCCL over NVLink on GPUs,
  gloo in the CPU tests).

Pixels of a strip are identical to the same pixels of a full frame
(tests/test_gpu_parity.py::test_screen_strips_equal_full_frame), so sharded
frames are bit-identical to single-GPU frames at any GPU count.
"""

from __future__ import annotations

import numpy as np

TILE_W, TILE_H = 8, 4          # render-kernel pixel tile (hc_render.cu TILE_W/TILE_H)


def shard_views(n_views: int, world: int, rank: int) -> list[int]:
    """Round-robin view assignment for camera batches."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return list(range(rank, n_views, world))


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

    Uses all_gather on equally padded strips (works with NCCL device tensors and
    gloo host tensors); returns the image on `dst`, None elsewhere."""
    import torch
    import torch.distributed as dist
    H = strip.shape[0]
    wmax = max(x1 - x0 for x0, x1 in rects)
    padded = torch.zeros((H, wmax, 3), dtype=strip.dtype, device=strip.device)
    padded[:, :strip.shape[1]] = strip
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    if rank != dst:
        return None
    W = rects[-1][1]
    out = torch.empty((H, W, 3), dtype=strip.dtype, device=strip.device)
    for (x0, x1), p in zip(rects, parts):
        out[:, x0:x1] = p[:, :x1 - x0]
    return out


def render_strip(config, grid, table, params, settings, rect):
    """Render pixel columns rect=(x0, x1) of the full frame on this rank's GPU.

    Returns the (H, x1-x0, 3) uint8 device tensor (a copy), or None if nothing is visible."""
    from .render import enqueue_frame
    x0, x1 = rect
    if table.sigma != params.sigma:
        raise ValueError("influence table was built for a different sigma")
    queued = enqueue_frame(config, grid, table, settings, rect=(x0, 0, x1, config.height))
    if queued is None:
        return None
    buf = queued[0]
    return buf.rgb[:, x0:x1].clone()

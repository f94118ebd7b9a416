"""HBM residency of the grid and its influence table.

Uploaded once per (grid, device) and per (influence table, device): the reference
treats the grid and `build_influence_table` as startup precompute
(cli.py:48-54); here that precompute also includes the anchored influence
records the discretization kernel streams (hc_build_records).

Layout in HBM:
  cx, cy, size, terrain, depth   float64 [N]       cell SoA (grid.py:96-99)
  tile_index                     int32 [nty, ntx]  min-cell lookup (grid.py:154-177)
  offsets                        int32 [N+1]       CSR (grid.py:350-376)
  indices                        int32 [N*L]
  pair_offsets                   int32 [N+1]       prefix of ceil(list length / 2), each rounded up to x4
  rec                            float32 [pairs/4, 40] quads of record pairs (pairs of consecutive
                                                   list entries): {x0,x1,y0,y1} x4, {s0,s1,t0,t1} x4,
                                                   {d0,d1} x4
  anchor_t, anchor_d             float32 [N]       list-head terrain / depth
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _cuda


class InfluenceDevice:
    def __init__(self, gdev: "GridDevice", table):
        import torch
        dev = gdev.device
        if len(table.indices) >= 2 ** 31:
            raise ValueError("influence table too large for int32 device indexing")
        self.table = table
        self.sigma = float(table.sigma)
        cached = getattr(table, "_device_csr", {}).get(str(dev))
        if cached is not None:        # built on this GPU: no re-upload
            self.offsets, self.indices = cached
        else:
            self.offsets = torch.from_numpy(table.offsets.astype(np.int32)).to(dev)
            self.indices = torch.from_numpy(table.indices.astype(np.int32)).to(dev)
        n = gdev.n_cells
        lens = np.diff(np.asarray(table.offsets, dtype=np.int64))
        # pairs of list entries, padded to a multiple of 4 pairs: every list is a run
        # of whole 160-byte quads (one TMA bulk copy, 16-byte aligned)
        pair_off = np.zeros(n + 1, dtype=np.int64)
        np.cumsum((((lens + 1) // 2) + 3) & ~3, out=pair_off[1:])
        if pair_off[-1] >= 2 ** 31:
            raise ValueError("influence table too large for int32 device indexing")
        self.pair_offsets = torch.from_numpy(pair_off.astype(np.int32)).to(dev)
        n_pairs = max(int(pair_off[-1]), 1)
        self.rec = torch.empty((max(n_pairs // 4, 1), 40), dtype=torch.float32, device=dev)
        self.anchor_t = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
        self.anchor_d = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
        self.view = gdev.hc_grid(self)
        with torch.cuda.device(dev):
            _cuda.check(_cuda.lib().hc_build_records(C.byref(self.view), self.rec.data_ptr(),
                                                     self.anchor_t.data_ptr(),
                                                     self.anchor_d.data_ptr(),
                                                     _cuda.stream_ptr()), "hc_build_records")
        self.mean_list = float(len(table.indices)) / max(n, 1)


def _size_class_bins(grid, sigma):
    """Host counting sort of cells into one uniform bin grid per size class."""
    sizes = grid.sizes
    d = grid.domain
    classes = np.unique(sizes)
    if len(classes) > _cuda.HC_MAX_SIZE_CLASSES:
        raise ValueError(f"{len(classes)} cell size classes (max {_cuda.HC_MAX_SIZE_CLASSES})")
    cells, starts = [], []
    base_cells = 0
    base_bins = 0
    B = _cuda.HcInfluenceBins()
    B.n_classes = len(classes)
    B.xmin, B.ymin = float(d.xmin), float(d.ymin)
    for s, c in enumerate(classes.tolist()):
        idx = np.flatnonzero(sizes == c)
        bs = 3.5 * sigma * c + c                     # the reach spans ~3 bins per axis
        nbx = int(math.floor(d.width / bs)) + 1
        nby = int(math.floor(d.height / bs)) + 1
        bx = np.clip(np.floor((grid.centers[idx, 0] - d.xmin) / bs).astype(np.int64), 0, nbx - 1)
        by = np.clip(np.floor((grid.centers[idx, 1] - d.ymin) / bs).astype(np.int64), 0, nby - 1)
        key = by * nbx + bx
        order = np.argsort(key, kind="stable")
        cells.append(idx[order].astype(np.int32))
        counts = np.bincount(key, minlength=nby * nbx)
        st = np.zeros(nby * nbx + 1, dtype=np.int64)
        np.cumsum(counts, out=st[1:])
        starts.append((st + base_cells).astype(np.int32))
        B.class_size[s], B.bin_size[s], B.nbx[s], B.nby[s] = c, bs, nbx, nby
        B.class_bin_base[s] = base_bins
        base_cells += len(idx)
        base_bins += nby * nbx + 1
    return B, np.concatenate(cells), np.concatenate(starts)


def build_influence_gpu(grid, sigma, device=None):
    """grid.build_influence_table on the GPU (hc_influence_build); returns an
    InfluenceTable with host CSR arrays and caches the device copy for the frame path."""
    import torch
    from .grid import InfluenceTable
    gdev = grid.device_view(device)
    dev = gdev.device
    B, cells, starts = _size_class_bins(grid, sigma)
    cells_d = torch.from_numpy(cells).to(dev)
    starts_d = torch.from_numpy(starts).to(dev)
    B.cells, B.bin_start = cells_d.data_ptr(), starts_d.data_ptr()
    n = grid.n_cells
    L = _cuda.lib()
    ws = torch.empty(max(L.hc_influence_workspace_bytes(n), 16), dtype=torch.uint8, device=dev)
    offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
    total = torch.zeros(1, dtype=torch.int64, pin_memory=True)
    view = gdev.hc_grid()
    with torch.cuda.device(dev):
        s = _cuda.stream_ptr()
        _cuda.check(L.hc_influence_build(C.byref(view), C.byref(B), sigma, offsets.data_ptr(), None, 0,
                                         ws.data_ptr(), ws.numel(), total.data_ptr(), s), "hc_influence_build")
        torch.cuda.current_stream().synchronize()
        nnz = int(total.item())
        indices = torch.empty(max(nnz, 1), dtype=torch.int64, device=dev)
        flag = torch.zeros(1, dtype=torch.int64, pin_memory=True)
        _cuda.check(L.hc_influence_build(C.byref(view), C.byref(B), sigma, offsets.data_ptr(), indices.data_ptr(),
                                         nnz, ws.data_ptr(), ws.numel(), flag.data_ptr(), s), "hc_influence_build")
        torch.cuda.current_stream().synchronize()
    over, short = (int(x) for x in flag.numpy().view(np.int32)[:2])
    if short:
        raise _cuda.HeightcastCudaError(f"influence index buffer of {nnz} entries is too small")
    if over:
        raise _cuda.HeightcastCudaError(f"influence list of {over} entries exceeds the GPU sort capacity")
    table = InfluenceTable(offsets.cpu().numpy(), indices[:nnz].cpu().numpy(), sigma)
    table._device_csr = {str(dev): (offsets.to(torch.int32), indices[:nnz].to(torch.int32))}
    return table


class GridDevice:
    def __init__(self, grid, device):
        import torch
        _cuda.require_cuda()
        self.grid = grid
        self.device = device
        self.n_cells = grid.n_cells
        f64 = lambda a: torch.from_numpy(np.array(a, dtype=np.float64, copy=True)).to(device)
        self.cx = f64(grid.centers[:, 0])
        self.cy = f64(grid.centers[:, 1])
        self.size = f64(grid.sizes)
        self.terrain = f64(grid.terrain)
        self.depth = f64(grid.water_depth)
        painted = grid.device_tile_index(device)        # painted in this GPU's HBM: no upload
        self.tile_index = painted if painted is not None else \
            torch.from_numpy(np.array(grid.tile_index, copy=True)).to(device)
        self._influence = {}

    def influence(self, table) -> InfluenceDevice:
        key = id(table)
        hit = self._influence.get(key)
        if hit is None or hit.table is not table:
            hit = InfluenceDevice(self, table)
            self._influence[key] = hit
        return hit

    def hc_grid(self, inf: InfluenceDevice | None = None) -> _cuda.HcGrid:
        g = _cuda.HcGrid()
        g.cx, g.cy, g.size = self.cx.data_ptr(), self.cy.data_ptr(), self.size.data_ptr()
        g.terrain, g.depth = self.terrain.data_ptr(), self.depth.data_ptr()
        g.tile_index = self.tile_index.data_ptr()
        nty, ntx = self.tile_index.shape
        g.ntx, g.nty = ntx, nty
        d = self.grid.domain
        g.xmin, g.ymin, g.min_cell = d.xmin, d.ymin, self.grid.min_cell_size
        g.n_cells = self.n_cells
        if inf is not None:
            g.offsets, g.indices = inf.offsets.data_ptr(), inf.indices.data_ptr()
            g.pair_offsets = inf.pair_offsets.data_ptr()
            g.rec = inf.rec.data_ptr()
            g.anchor_t, g.anchor_d = inf.anchor_t.data_ptr(), inf.anchor_d.data_ptr()
            g.sigma = inf.sigma
        return g

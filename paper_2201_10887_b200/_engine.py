"""Per-frame GPU pipeline: descriptor packing, buffer reuse, launches, timing.

A frame is three kernel launch groups on one stream (plus one memset and the
pixel read-back):

  hc_discretize  mask + cell lookup + Eq. 1/2, all K cascades, both layers
  hc_maxmip      2K max pyramids + valid ranges + patch validity (2 launches)
  hc_render      rays + per-layer traversal/resolve + shading + pixel select

Buffers for a given (K, R, W, H) shape are allocated once and reused, so a
steady-state frame performs no device allocation.  Everything here is host
orchestration; the arithmetic lives in csrc/.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _cuda

_L = np.array([-0.45, -0.35, 0.82])
LIGHT_DIR = _L / np.linalg.norm(_L)               # render.py:35-36
COLOR_STOPS = np.array([(0.0, 0.0, 128.0), (0.0, 180.0, 220.0), (240.0, 248.0, 255.0)])


def mip_shape(R: int):
    """Level offsets and widths of the max pyramid of an R x R raster (raycast.py:71-87)."""
    off, w = [], []
    o, cw = 0, R - 1
    while True:
        off.append(o)
        w.append(cw)
        o += cw * cw
        if cw <= 1:
            break
        cw = (cw + 1) // 2
    return off, w, o


def fill_cascade_raster(desc: _cuda.HcCascadeRaster, layout, terrain, water, valid, mask=None):
    edges = layout.edge_table()
    desc.origin_x = float(layout.world_origin[0])
    desc.origin_y = float(layout.world_origin[1])
    desc.texel = float(layout.texel_size)
    desc.resolution = int(layout.resolution)
    desc.n_edges = len(edges)
    flat = np.zeros(_cuda.HC_MAX_EDGES * 5)
    flat[:edges.size] = edges.ravel()
    desc.edges[:] = flat.tolist()
    desc.terrain = _cuda.ptr(terrain)
    desc.water = _cuda.ptr(water)
    desc.valid = _cuda.ptr(valid)
    desc.mask = _cuda.ptr(mask)


def fill_mip_job(job: _cuda.HcMipJob, R, heights, valid, mip, vrange_key, patch_ok=None):
    off, w, _ = mip_shape(R)
    if len(off) > _cuda.HC_MAX_LEVELS:
        raise ValueError(f"raster resolution {R} needs {len(off)} mip levels (max {_cuda.HC_MAX_LEVELS})")
    job.heights = _cuda.ptr(heights)
    job.valid = _cuda.ptr(valid)
    job.mip = _cuda.ptr(mip)
    job.patch_ok = _cuda.ptr(patch_ok)
    job.vrange_key = _cuda.ptr(vrange_key)
    job.resolution = R
    job.n_levels = len(off)
    for L in range(len(off)):
        job.level_off[L] = off[L]
        job.level_w[L] = w[L]


def key_to_float(k: int) -> float:
    b = k if k >= 0 else (k ^ 0x7FFFFFFF)
    return float(np.array([b], dtype=np.int32).view(np.float32)[0])


class FrameBuffers:
    """Device buffers for frames of one shape (K cascades of R^2, W x H pixels)."""

    def __init__(self, device, K, R, W, H, debug=False):
        import torch
        self.K, self.R, self.W, self.H = K, R, W, H
        dev = device
        self.terrain = torch.empty((K, R, R), dtype=torch.float32, device=dev)
        self.water = torch.empty((K, R, R), dtype=torch.float32, device=dev)
        self.valid = torch.empty((K, R, R), dtype=torch.uint8, device=dev)
        self.mask = torch.empty((K, R, R), dtype=torch.uint8, device=dev)
        self.patch_ok = torch.empty((K, (R - 1) * (R - 1)), dtype=torch.uint8, device=dev)
        _, _, nodes = mip_shape(R)
        self.n_nodes = nodes
        self.mip = torch.empty((K, 2, nodes), dtype=torch.float32, device=dev)
        self.vrange = torch.empty((K, 2, 2), dtype=torch.int32, device=dev)
        ws = _cuda.lib().hc_maxmip_workspace_bytes(2 * K, R)
        self.mip_ws = torch.empty(max(ws, 16), dtype=torch.uint8, device=dev)
        # frame counters (HC_CNT_*): visible, valid, zero-weight flag, rays hit, pairs,
        # node visits, patch tests
        self.counters = torch.zeros(_cuda.N_COUNTERS, dtype=torch.int64, device=dev)
        self.rgb = torch.empty((H, W, 3), dtype=torch.uint8, device=dev)
        n_tiles = _cuda.lib().hc_render_tiles(0, 0, W, H)
        self.tile_cost = torch.zeros(max(n_tiles, 1), dtype=torch.int32, device=dev)
        self.tile_order = torch.empty(max(n_tiles, 1), dtype=torch.int32, device=dev)
        self.tile_counter = torch.zeros(1, dtype=torch.int32, device=dev)
        self.rgb_host = torch.empty((H, W, 3), dtype=torch.uint8, pin_memory=True)
        self.counters_host = torch.empty(_cuda.N_COUNTERS, dtype=torch.int64, pin_memory=True)
        self.dbg = None
        if debug:
            self.alloc_debug()
        # events: 0 frame start, 1 after discretize, 2 after render, 3 read-back done, 4 after maxmip
        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]

    def alloc_debug(self):
        import torch
        P = self.W * self.H
        dev = self.rgb.device
        self.dbg = {
            "hit": torch.empty((2, P), dtype=torch.uint8, device=dev),
            "t": torch.empty((2, P), dtype=torch.float64, device=dev),
            "near_k": torch.empty((2, P), dtype=torch.int8, device=dev),
            "far_k": torch.empty((2, P), dtype=torch.int8, device=dev),
            "w": torch.empty((2, P), dtype=torch.float64, device=dev),
            "raw_t": torch.empty((2, 2, P), dtype=torch.float64, device=dev),
            "raw_ix": torch.empty((2, 2, P), dtype=torch.int32, device=dev),
            "raw_iy": torch.empty((2, 2, P), dtype=torch.int32, device=dev),
            "raw_u": torch.empty((2, 2, P), dtype=torch.float64, device=dev),
            "raw_v": torch.empty((2, 2, P), dtype=torch.float64, device=dev),
            "water_depth": torch.empty(P, dtype=torch.float64, device=dev),
            "dirs": torch.empty((P, 3), dtype=torch.float64, device=dev),
        }


@dataclass
class FrameDescriptors:
    rasters: object
    jobs: object
    render: _cuda.HcRenderArgs
    K: int


def camera_constants(camera):
    right, true_up, look = camera.basis()
    tan_half = math.tan(math.radians(camera.fov_y) / 2.0)
    return right, true_up, look, tan_half


def pack_frame(buf: FrameBuffers, layouts, camera, grid, width, height, colormap_range, background,
               rect=None) -> FrameDescriptors:
    """Host-side descriptors for one frame (all float64 scalars evaluated as the reference does)."""
    K = len(layouts)
    rasters = (_cuda.HcCascadeRaster * max(K, 1))()
    jobs = (_cuda.HcMipJob * max(2 * K, 1))()
    A = _cuda.HcRenderArgs()
    eye = np.asarray(camera.eye, dtype=np.float64)
    right, up, look, tan_half = camera_constants(camera)
    A.width, A.height, A.n_cascades = width, height, K
    x0, y0, x1, y1 = rect if rect is not None else (0, 0, width, height)
    A.x0, A.y0, A.x1, A.y1 = x0, y0, x1, y1
    A.eye[:] = eye.tolist()
    A.look[:] = look.tolist()
    A.right[:] = right.tolist()
    A.up[:] = up.tolist()
    A.tan_half, A.aspect = tan_half, float(camera.aspect)
    if K:
        ax = layouts[0].polygon.axis
        A.axis_anchor[:] = [float(ax.anchor[0]), float(ax.anchor[1])]
        A.axis_dir[:] = [float(ax.direction[0]), float(ax.direction[1])]
    A.h_lo, A.h_hi = float(grid.height_range[0]), float(grid.height_range[1])
    A.light[:] = LIGHT_DIR.tolist()
    A.cm_lo, A.cm_hi = float(colormap_range[0]), float(colormap_range[1])
    A.stops[:] = COLOR_STOPS.ravel().tolist()
    A.background[:] = [int(background[0]), int(background[1]), int(background[2]), 0]
    off, w, _ = mip_shape(buf.R)
    for k, lay in enumerate(layouts):
        fill_cascade_raster(rasters[k], lay, buf.terrain[k], buf.water[k], buf.valid[k], buf.mask[k])
        for layer, hh in enumerate((buf.terrain[k], buf.water[k])):
            fill_mip_job(jobs[2 * k + layer], buf.R, hh, buf.valid[k], buf.mip[k, layer],
                         buf.vrange[k, layer], buf.patch_ok[k] if layer == 0 else None)
        c = A.c[k]
        s = lay.texel_size
        c.origin_x, c.origin_y, c.texel = float(lay.world_origin[0]), float(lay.world_origin[1]), s
        # render.py:135-136: (origin - world_origin) / s in float64
        c.rx = float((eye[0] - lay.world_origin[0]) / s)
        c.ry = float((eye[1] - lay.world_origin[1]) / s)
        c.near_offset = float(lay.polygon.near_offset)
        c.far_offset = float(lay.polygon.far_offset)
        c.resolution, c.n_levels = buf.R, len(off)
        c.heights[0], c.heights[1] = buf.terrain[k].data_ptr(), buf.water[k].data_ptr()
        c.valid = buf.valid[k].data_ptr()
        c.patch_ok = buf.patch_ok[k].data_ptr()
        c.mip[0], c.mip[1] = buf.mip[k, 0].data_ptr(), buf.mip[k, 1].data_ptr()
        c.vrange_key = buf.vrange[k].data_ptr()
        for L in range(len(off)):
            c.level_off[L] = off[L]
            c.level_w[L] = w[L]
    A.rgb = buf.rgb.data_ptr()
    A.counters = buf.counters.data_ptr()
    A.tile_counter = buf.tile_counter.data_ptr()
    if rect is None:       # costs/order are per full-frame tile grid
        A.tile_cost = buf.tile_cost.data_ptr()
        A.tile_order = buf.tile_order.data_ptr()
    if buf.dbg is not None:
        for name, t in buf.dbg.items():
            setattr(A.dbg, name, t.data_ptr())
    return FrameDescriptors(rasters, jobs, A, K)


LAUNCHES_PER_FRAME = 5   # hc_discretize (1) + hc_maxmip (2) + hc_render (2: tile order, render)


def launch_frame(buf: FrameBuffers, fd: FrameDescriptors, ginf, sentinel: float, stream=None,
                 timing: bool = True):
    """Enqueue discretize -> maxmip -> render on `stream` (no host sync)."""
    L = _cuda.lib()
    s = _cuda.stream_ptr(stream)
    buf.counters.zero_()
    if timing:
        buf.ev[0].record()
    if fd.K:
        _cuda.check(L.hc_discretize(fd.rasters, fd.K, C.byref(ginf.view), C.c_float(sentinel),
                                    buf.counters.data_ptr(), s), "hc_discretize")
    if timing:
        buf.ev[1].record()
    if fd.K:
        _cuda.check(L.hc_maxmip(fd.jobs, 2 * fd.K, buf.mip_ws.data_ptr(), buf.mip_ws.numel(), s),
                    "hc_maxmip")
    if timing:
        buf.ev[4].record()
    _cuda.check(L.hc_render(C.byref(fd.render), s), "hc_render")
    if timing:
        buf.ev[2].record()

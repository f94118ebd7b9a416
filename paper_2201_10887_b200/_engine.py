"""Per-frame GPU pipeline: buffer reuse, native planning + launch, timing.

A frame is one host call into the library after planning:

  hc_plan_cascades   host C++, float64 (bit-identical to the reference planner)
  hc_frame_launch    packs the kernel descriptors and enqueues on one stream:
    hc_discretize    mask + cell lookup + Eq. 1/2, all K cascades, both layers
    hc_maxmip        2K max pyramids + valid ranges + patch validity (2 launches)
    hc_render        tile order + rays/traversal/resolve/shading (2 launches)

Buffers for a given (K, R, W, H) shape are allocated once and reused, so a
steady-state frame performs no device allocation and ~30 us of host work.
Everything here is orchestration; the arithmetic lives in csrc/.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _cuda

_L = np.array([-0.45, -0.35, 0.82])
LIGHT_DIR = _L / np.linalg.norm(_L)               # render.py:35-36
COLOR_STOPS = np.array([(0.0, 0.0, 128.0), (0.0, 180.0, 220.0), (240.0, 248.0, 255.0)])

# hc_frame_launch: discretize with fused mip levels 0..5 (1) + mip levels >= 6 and
# valid ranges (1) -- both also compute the render's tile order in extra CTAs -- +
# render (1)
LAUNCHES_PER_FRAME = 3


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


def fill_mip_job(job: _cuda.HcMipJob, R, heights, valid, mip, vrange_key, patch_ok=None, heights_other=None):
    off, w, _ = mip_shape(R)
    if len(off) > _cuda.HC_MAX_LEVELS:
        raise ValueError(f"raster resolution {R} needs {len(off)} mip levels (max {_cuda.HC_MAX_LEVELS})")
    job.heights = _cuda.ptr(heights)
    job.valid = _cuda.ptr(valid)
    job.mip = _cuda.ptr(mip)
    job.patch_ok = _cuda.ptr(patch_ok)
    job.heights_other = _cuda.ptr(heights_other)
    job.vrange_key = _cuda.ptr(vrange_key)
    job.resolution = R
    job.n_levels = len(off)
    for L in range(len(off)):
        job.level_off[L] = off[L]
        job.level_w[L] = w[L]


def key_to_float(k: int) -> float:
    b = k if k >= 0 else (k ^ 0x7FFFFFFF)
    return float(np.array([b], dtype=np.int32).view(np.float32)[0])


def shading(colormap_range, background) -> _cuda.HcShading:
    s = _cuda.HcShading()
    s.cm_lo, s.cm_hi = float(colormap_range[0]), float(colormap_range[1])
    s.light[:] = LIGHT_DIR.tolist()
    s.stops[:] = COLOR_STOPS.ravel().tolist()
    s.background[:] = [int(background[0]), int(background[1]), int(background[2]), 0]
    return s


class FrameBuffers:
    """Device buffers for frames of one shape (up to K cascades of R^2, W x H pixels)."""

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
        n_order = _cuda.lib().hc_render_order_words(0, 0, W, H)
        self.tile_order = torch.empty(max(n_order, 1), dtype=torch.int32, device=dev)
        self.tile_counter = torch.zeros(1, dtype=torch.int32, device=dev)
        self.counters_host = torch.empty(_cuda.N_COUNTERS, dtype=torch.int64, pin_memory=True)
        self.dbg = None
        self.dbg_native = None
        if debug:
            self.alloc_debug()
        # events: 0 before discretize, 1 after discretize, 2 after render, 3 read-back done, 4 after maxmip
        self.ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        for e in self.ev:
            e.record()                       # materialise the CUDA event handles
        self.ev_handles = (C.c_void_p * 4)(self.ev[0].cuda_event, self.ev[1].cuda_event,
                                            self.ev[4].cuda_event, self.ev[2].cuda_event)
        nb = _cuda.HcFrameBuffers()
        nb.terrain, nb.water = self.terrain.data_ptr(), self.water.data_ptr()
        nb.valid, nb.mask, nb.patch_ok = self.valid.data_ptr(), self.mask.data_ptr(), self.patch_ok.data_ptr()
        nb.mip, nb.vrange = self.mip.data_ptr(), self.vrange.data_ptr()
        nb.mip_ws, nb.mip_ws_bytes = self.mip_ws.data_ptr(), self.mip_ws.numel()
        nb.rgb, nb.counters = self.rgb.data_ptr(), self.counters.data_ptr()
        nb.tile_counter = self.tile_counter.data_ptr()
        nb.tile_cost, nb.tile_order = self.tile_cost.data_ptr(), self.tile_order.data_ptr()
        nb.capacity, nb.resolution, nb.width, nb.height = K, R, W, H
        self.native = nb

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
            "visits": torch.empty((2, P), dtype=torch.int32, device=dev),
        }
        d = _cuda.HcRenderDebug()
        for name, t in self.dbg.items():
            setattr(d, name, t.data_ptr())
        self.dbg_native = d


def event_handles(events):
    """hc_frame_launch event array from 4 torch events: before discretize, after
    discretize, after maxmip (= before render), after render."""
    return (C.c_void_p * 4)(*[e.cuda_event for e in events])


def launch_planned(buf: FrameBuffers, plan, camera_native, domain_native, ginf, shade, rect=None, stream=None,
                   events=None, stage=None, footprint=None, xchg=None):
    """Enqueue one planned frame on `stream` (no host sync).  `events`: optional
    event_handles() array recorded instead of the buffers' own events.  With
    `stage` (1 or 2), `footprint` (HcFootprint) and `xchg` (float32 device tensor of
    hc_frame_xchg_floats): one stage of a sharded screen-strip frame."""
    r = None if rect is None else (C.c_int32 * 4)(*rect)
    args = (C.byref(plan), C.byref(camera_native), C.byref(domain_native), C.byref(ginf.view), C.byref(buf.native),
            C.byref(shade), C.byref(buf.dbg_native) if buf.dbg_native is not None else None,
            C.cast(r, C.c_void_p) if r is not None else None,
            C.cast(buf.ev_handles if events is None else events, C.c_void_p))
    if stage is None:
        _cuda.check(_cuda.lib().hc_frame_launch(*args, _cuda.stream_ptr(stream)), "hc_frame_launch")
    else:
        _cuda.check(_cuda.lib().hc_frame_stage(stage, *args, C.byref(footprint), _cuda.ptr(xchg),
                                               _cuda.stream_ptr(stream)), "hc_frame_stage")

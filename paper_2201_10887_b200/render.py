"""Per-frame orchestration on the GPU: plan cascades, fill rasters, cast rays, shade.

Drop-in for `heightcast.render` (pkg/src/heightcast/render.py).  `render_frame`
keeps the reference signature and result type.  Cascade planning is host
float64 geometry (cascade.py, bit-identical to the reference); everything per
texel and per pixel runs on the B200 in three launch groups (see _engine.py):

  approximation  hc_discretize            discretize.py:52-108 for all K cascades
  ray casting    hc_maxmip + hc_render    raycast.py:61-88, render.py:100-341

`Frame.approximation_ms` / `raycast_ms` keep the reference's two phase
categories (render.py:233-258) but are CUDA-event device times; `plan_ms` is
the host planning time the reference leaves untimed.  `CascadeSettings.count`
(default 3, the reference's fixed value) selects K cascades.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _cuda, _engine
from .cascade import CameraView, NothingVisibleError, layouts_from_plan, plan_native
from .cascade import _domain as _cascade_domain
from .discretize import CascadeRaster
from .grid import AdaptiveGrid, InfluenceTable
from .rbf import RbfParams

_COLOR_STOPS = _engine.COLOR_STOPS
_LIGHT_DIR = _engine.LIGHT_DIR


@dataclass(frozen=True)
class FrameConfig:
    width: int
    height: int
    camera: CameraView
    colormap_range: tuple[float, float] = (0.0, 5.0)
    background: tuple[int, int, int] = (30, 40, 60)

    def __post_init__(self):
        if self.width < 1 or self.height < 1:
            raise ValueError("image size must be at least 1x1")
        if not self.colormap_range[0] < self.colormap_range[1]:
            raise ValueError("colormap range min must be below max")


@dataclass(frozen=True)
class CascadeSettings:
    resolution: int = 1024
    overlap: float | str = "auto"
    count: int = 3

    def __post_init__(self):
        if not 1 <= self.count <= _cuda.HC_MAX_CASCADES:
            raise ValueError(f"cascade count must be in 1..{_cuda.HC_MAX_CASCADES}")


@dataclass
class Frame:
    pixels: np.ndarray                  # (height, width, 3) uint8, row 0 at the top
    approximation_ms: float
    raycast_ms: float
    visible_texels: int = 0
    rays_hit: int = 0
    visible: bool = True
    debug: dict | None = field(default=None, repr=False)
    plan_ms: float = 0.0
    valid_texels: int = 0


def depth_colormap(depth, colormap_range, background=(0, 0, 0)):
    """Blue-cyan-white depth gradient (render.py:71-97); host helper for scalar/array use."""
    lo, hi = colormap_range

    def cmap(d):
        t = np.clip((d - lo) / (hi - lo), 0.0, 1.0)
        out = np.empty(t.shape + (3,))
        for ch in range(3):
            s0, s1, s2 = _COLOR_STOPS[:, ch]
            out[..., ch] = np.where(t <= 0.5, s0 + (s1 - s0) * (2.0 * t), s1 + (s2 - s1) * (2.0 * t - 1.0))
        return np.clip(np.rint(out), 0, 255).astype(np.uint8)

    if isinstance(depth, np.ndarray):
        rgb = cmap(depth)
        bad = ~np.isfinite(depth)
        if bad.any():
            rgb[bad] = background
        return rgb
    if not math.isfinite(depth):
        return tuple(int(c) for c in background)
    r = cmap(np.array([float(depth)]))[0]
    return int(r[0]), int(r[1]), int(r[2])


def camera_ray_dirs(camera: CameraView, width: int, height: int) -> np.ndarray:
    """Per-pixel unit ray directions (render.py:100-110); host helper, the render
    kernel evaluates the same float64 expression per pixel on the GPU."""
    right, up, look = camera.basis()
    th = math.tan(math.radians(camera.fov_y) / 2.0)
    xs = ((np.arange(width) + 0.5) / width * 2.0 - 1.0) * th * camera.aspect
    ys = (1.0 - (np.arange(height) + 0.5) / height * 2.0) * th
    d = look[None, None, :] + xs[None, :, None] * right + ys[:, None, None] * up
    return d / np.linalg.norm(d, axis=2, keepdims=True)


class LayerResolve:
    """Per-pixel outcome of one layer (render.py:113-122), device tensors.

    `near`/`far` are cascade list indices (-1 = none); `raw[k]` holds
    (hit, t, ix, iy, u, v) for the pixels whose near or blend cascade is k (the
    GPU traverses only those; other entries are -1 / 0)."""

    def __init__(self, dbg, layer, K):
        import torch
        self.hit = dbg["hit"][layer].bool()
        self.t = dbg["t"][layer]
        self.near = dbg["near_k"][layer].to(torch.int32)
        self.far = dbg["far_k"][layer].to(torch.int32)
        self.w = dbg["w"][layer]
        self.raw_slots = {name: dbg["raw_" + name][layer] for name in ("t", "ix", "iy", "u", "v")}
        self.raw = {}
        for k in range(K):
            sel0 = self.hit & (self.near == k)
            sel1 = self.hit & (self.far == k)
            vals = []
            for name, fill in (("t", 0.0), ("ix", -1), ("iy", -1), ("u", 0.0), ("v", 0.0)):
                s = self.raw_slots[name]
                base = torch.full_like(s[0], fill)
                base = torch.where(sel0, s[0], base)
                vals.append(torch.where(sel1, s[1], base))
            self.raw[k] = (sel0 | sel1, *vals)


_BUFFERS: dict = {}
_SIDE_STREAMS: dict = {}       # per device: render_frames' read-back stream and side compute streams


def _frame_buffers(device, K, R, W, H, debug, slot=0):
    import torch
    key = (str(device), K, R, W, H, bool(debug), int(slot))
    buf = _BUFFERS.get(key)
    if buf is None:
        if len(_BUFFERS) > 8:
            # buffers may still be in use by queued frames (render_frames runs them
            # on side streams): let the device finish before releasing them
            torch.cuda.synchronize()
            _BUFFERS.clear()
        buf = _engine.FrameBuffers(torch.device(device), K, R, W, H, debug=debug)
        _BUFFERS[key] = buf
    return buf


def _background_frame(config, debug):
    px = np.empty((config.height, config.width, 3), dtype=np.uint8)
    px[:] = np.asarray(config.background, dtype=np.uint8)
    return Frame(px, 0.0, 0.0, 0, 0, visible=False, debug={"visible": False} if debug else None)


_SHADING: dict = {}


def _shading(config):
    key = (tuple(config.colormap_range), tuple(config.background))
    s = _SHADING.get(key)
    if s is None:
        s = _SHADING[key] = _engine.shading(config.colormap_range, config.background)
    return s


def enqueue_frame(config: FrameConfig, grid: AdaptiveGrid, table: InfluenceTable,
                  settings: CascadeSettings = CascadeSettings(), debug: bool = False, rect=None, events=None,
                  slot: int = 0, throughput: bool = False):
    """Plan natively on the host and enqueue one frame's kernels on the current stream.

    Returns (buffers, plan, plan_ms) without waiting for the GPU, or None when
    nothing is visible.  The device-resident half of `render_frame`; pixels stay
    in `buffers.rgb` until read back."""
    prep = prepare_frame(config, grid, table, settings, debug, slot, throughput)
    if prep is None:
        return None
    buf, plan, plan_ms, launch = prep
    launch(rect=rect, events=events)
    return buf, plan, plan_ms


def prepare_frame(config: FrameConfig, grid: AdaptiveGrid, table: InfluenceTable,
                  settings: CascadeSettings = CascadeSettings(), debug: bool = False, slot: int = 0,
                  throughput: bool = False):
    """Plan one frame on the host and bind its buffer set: (buffers, plan, plan_ms,
    launch) or None when nothing is visible; `launch(**kw)` enqueues the frame (or
    one stage of a sharded frame, see multi.py) via _engine.launch_planned.
    `throughput`: the frame overlaps other frames on the GPU (render_frames), so the
    render uses its high-occupancy instantiation (hc_render.cu)."""
    tp = time.perf_counter()
    plan = plan_native(config.camera, grid, settings.resolution, settings.overlap, settings.count)
    if plan.status != 0:
        return None
    plan_ms = (time.perf_counter() - tp) * 1e3
    gdev = grid.device_view()
    ginf = gdev.influence(table)
    buf = _frame_buffers(gdev.device, settings.count, settings.resolution, config.width, config.height, debug,
                         slot)
    buf.native.throughput = 1 if throughput else 0
    dom = getattr(grid, "_hc_domain", None)
    if dom is None:
        dom = grid._hc_domain = _cascade_domain(grid)
    cam = config.camera.native()
    shade = _shading(config)

    def launch(**kw):
        _engine.launch_planned(buf, plan, cam, dom, ginf, shade, **kw)

    return buf, plan, plan_ms, launch


def render_frame(config: FrameConfig, grid: AdaptiveGrid, table: InfluenceTable, params: RbfParams,
                 settings: CascadeSettings = CascadeSettings(), debug: bool = False) -> Frame:
    """Render one frame on the GPU; same inputs/outputs as the reference."""
    import torch
    if table.sigma != params.sigma:
        raise ValueError("influence table was built for a different sigma")
    _cuda.require_cuda()
    dev = grid.device_view().device
    with torch.cuda.device(dev):
        queued = enqueue_frame(config, grid, table, settings, debug)
        if queued is None:
            return _background_frame(config, debug)
        buf, plan, plan_ms = queued
        pixels = torch.empty((config.height, config.width, 3), dtype=torch.uint8, pin_memory=True)
        pixels.copy_(buf.rgb, non_blocking=True)
        buf.counters_host.copy_(buf.counters, non_blocking=True)
        buf.ev[3].record()
        buf.ev[3].synchronize()
    return _finish_frame(buf, plan, plan_ms, pixels, buf.counters_host, grid, params, debug)


def render_frames(configs, grid: AdaptiveGrid, table: InfluenceTable, params: RbfParams,
                  settings: CascadeSettings = CascadeSettings(), before_frame=None, depth: int = 4):
    """Render a sequence of frames (a camera path or a batch of views), yielding
    one `Frame` per config, identical to `render_frame`'s.

    Up to `depth` (default 4) frames are in flight, each with its own device buffer set and
    compute stream (the caller's and depth-1 side streams): a frame's planning,
    discretization and mips run while earlier frames' ray casting finishes (whose
    last long rays leave most SMs idle), and pixels are read back on a copy stream
    meanwhile.  `before_frame(i)`, if given, is called on frame i's stream before
    it is enqueued (e.g. to enqueue an L2 flush); with depth > 1 it runs while
    earlier frames are still in flight, not between frames.

    Per-frame `approximation_ms` / `raycast_ms` are event intervals on the frame's
    own stream: with depth > 1 other frames share the SMs during them, so they
    overlap and are not the times of a frame rendered alone (use depth=1 for
    per-phase timing, as `render_frame` does)."""
    import collections
    import torch
    if table.sigma != params.sigma:
        raise ValueError("influence table was built for a different sigma")
    if depth < 1:
        raise ValueError("depth must be at least 1")
    _cuda.require_cuda()
    dev = grid.device_view().device
    with torch.cuda.device(dev):
        caller = torch.cuda.current_stream()
        grid.device_view().influence(table)    # upload / build records now, before the side streams fork
        side = _SIDE_STREAMS.setdefault(str(dev), [])
        while len(side) < depth:           # side[0]: read-back stream, side[1:]: compute streams
            side.append(torch.cuda.Stream())
        copy = side[0]
        streams = [caller] + side[1:depth]
        for st in streams[1:]:
            st.wait_stream(caller)         # side streams start after the caller's prior work
        read_done = [None] * depth         # per buffer slot: its last read-back
        pending = collections.deque()
        try:
            for i, config in enumerate(configs):
                slot = i % depth
                compute = streams[slot]
                with torch.cuda.stream(compute):
                    if before_frame is not None:
                        before_frame(i)
                    if read_done[slot] is not None:
                        compute.wait_event(read_done[slot])  # slot's previous pixels copied out
                    queued = enqueue_frame(config, grid, table, settings, slot=slot, throughput=depth > 1)
                if queued is None:
                    pending.append(("background", config))
                else:
                    buf, plan, plan_ms = queued
                    done = torch.cuda.Event()
                    done.record(compute)
                    pixels = torch.empty((config.height, config.width, 3), dtype=torch.uint8, pin_memory=True)
                    counters = torch.empty(_cuda.N_COUNTERS, dtype=torch.int64, pin_memory=True)
                    with torch.cuda.stream(copy):
                        copy.wait_event(done)
                        pixels.copy_(buf.rgb, non_blocking=True)
                        counters.copy_(buf.counters, non_blocking=True)
                        read_done[slot] = torch.cuda.Event()
                        read_done[slot].record(copy)
                    pending.append(("frame", buf, plan, plan_ms, pixels, counters, read_done[slot]))
                if len(pending) >= depth:
                    yield _finish_pending(pending.popleft(), grid, params)
            while pending:
                yield _finish_pending(pending.popleft(), grid, params)
        finally:
            # also when the consumer stops early (GeneratorExit at a yield): later work
            # on the caller's stream -- including the caching allocator's reuse of memory
            # freed there -- must see every side-stream frame and read-back
            for st in streams[1:]:
                caller.wait_stream(st)
            caller.wait_stream(copy)


def _finish_pending(item, grid, params):
    if item[0] == "background":
        return _background_frame(item[1], False)
    _, buf, plan, plan_ms, pixels, counters, ev = item
    ev.synchronize()
    return _finish_frame(buf, plan, plan_ms, pixels, counters, grid, params, False)


def _finish_frame(buf, plan, plan_ms, pixels, counters, grid, params, debug):
    cnt = counters.tolist()
    if cnt[_cuda.CNT_ZERO_WEIGHT]:
        raise ValueError(f"zero weight sum while discretizing: influence table inconsistent "
                         f"with sigma={params.sigma}")
    frame = Frame(pixels.numpy(), buf.ev[0].elapsed_time(buf.ev[1]), buf.ev[1].elapsed_time(buf.ev[2]),
                  visible_texels=int(cnt[_cuda.CNT_VISIBLE]), rays_hit=int(cnt[_cuda.CNT_RAYS_HIT]),
                  plan_ms=plan_ms, valid_texels=int(cnt[_cuda.CNT_VALID]))
    frame.work = {"pairs": int(cnt[_cuda.CNT_PAIRS]), "node_visits": int(cnt[_cuda.CNT_NODE_VISITS]),
                  "patch_tests": int(cnt[_cuda.CNT_PATCH_TESTS])}
    if debug:
        hull, polygons, layouts = layouts_from_plan(plan)
        active = [lay for lay in layouts if lay is not None]
        for k, lay in enumerate(active):
            lay.mask = buf.mask[k].clone().bool()
        rasters = [CascadeRaster(lay, buf.terrain[k].clone(), buf.water[k].clone(),
                                 buf.valid[k].bool(), grid.height_range[0] - 1.0)
                   for k, lay in enumerate(active)]
        rasters += [None] * (len(layouts) - len(active))
        d = buf.dbg
        frame.debug = {"visible": True, "layouts": layouts, "rasters": rasters,
                       "terrain": LayerResolve(d, 0, len(active)),
                       "water": LayerResolve(d, 1, len(active)),
                       "dirs": d["dirs"].clone(), "water_depth": d["water_depth"].clone(),
                       "visits": d["visits"].clone(),
                       "polygons": polygons, "hull": hull,
                       "mips": {"terrain": [buf.mip[k, 0].clone() for k in range(len(active))],
                                "water": [buf.mip[k, 1].clone() for k in range(len(active))]},
                       "vrange_keys": buf.vrange.clone()}
    return frame


def write_ppm(pixels, target) -> None:
    """Binary PPM (P6, maxval 255) of an (H, W, 3) uint8 image (render.py:344-354)."""
    arr = pixels.detach().cpu().numpy() if hasattr(pixels, "detach") else np.asarray(pixels)
    h, w = arr.shape[:2]
    header = f"P6\n{w} {h}\n255\n".encode("ascii")
    if hasattr(target, "write"):
        target.write(header)
        target.write(arr.astype(np.uint8).tobytes())
    else:
        with open(target, "wb") as fh:
            fh.write(header)
            fh.write(arr.astype(np.uint8).tobytes())

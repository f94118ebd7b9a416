"""Max-mipmap construction and ray traversal (GPU), plus the scalar ray API.

Drop-in for `heightcast.raycast` (pkg/src/heightcast/raycast.py):

* `build_max_mipmap(raster, layer)` -> `MaxMipmap` runs `hc_maxmip` (levels,
  valid range and patch validity in two launches); `levels` are CUDA tensor
  views into one flat float32 pyramid (raycast.py:40-88).
* `traverse_cascade` / `cast_through_cascades` trace single rays through
  `hc_traverse_batch`, the sm_100a twin of the reference Numba kernel
  (_kernels.py:75-232), float64 and bit-identical on identical rasters.
* `intersect_bilinear_patch` is the reference's scalar closed form for one patch
  (raycast.py:95-179); it is host arithmetic on Python floats by design.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _cuda
from ._engine import fill_mip_job, key_to_float, mip_shape
from .discretize import CascadeRaster


@dataclass(frozen=True)
class HitRecord:
    t: float
    world_pos: tuple[float, float, float]
    layer: str
    cascade: int
    uv: tuple[float, float]
    patch: tuple[int, int]
    blend: tuple[int, float] | None = None


class MaxMipmap:
    """Pyramid of patch maxima of one raster layer, resident in HBM."""

    def __init__(self, flat, R: int, layer: str, vrange=None, patch_ok=None):
        import torch
        off, w, _ = mip_shape(R)
        self.layer = layer
        self.resolution = R
        self._flat = flat
        self._off = torch.tensor(off, dtype=torch.int64, device=flat.device)
        self._w = torch.tensor(w, dtype=torch.int64, device=flat.device)
        self._h = self._w
        self.levels = [flat[o:o + n * n].view(n, n) for o, n in zip(off, w)]
        self._vrange = vrange
        self.patch_ok = patch_ok

    @property
    def n_levels(self) -> int:
        return len(self.levels)

    def node_max(self, level: int, nx: int, ny: int) -> float:
        return float(self.levels[level][ny, nx])

    def valid_range(self):
        """(min, max) of valid heights computed by the mip kernel, or None."""
        k = self._vrange.cpu().tolist()
        if k[0] > k[1]:
            return None
        return key_to_float(k[0]), key_to_float(k[1])


def build_max_mipmap(raster: CascadeRaster, layer: str) -> MaxMipmap:
    import torch
    heights = raster.layer(layer)
    R = int(heights.shape[0])
    if R < 2:
        raise ValueError("raster resolution must be at least 2")
    _cuda.require_cuda()
    dev = heights.device
    _, _, nodes = mip_shape(R)
    flat = torch.empty(nodes, dtype=torch.float32, device=dev)
    vrange = torch.empty(2, dtype=torch.int32, device=dev)
    patch_ok = torch.empty((R - 1) * (R - 1), dtype=torch.uint8, device=dev)
    valid = raster.valid.to(torch.uint8).contiguous()
    hh = heights.contiguous()
    jobs = (_cuda.HcMipJob * 1)()
    fill_mip_job(jobs[0], R, hh, valid, flat, vrange, patch_ok)
    L = _cuda.lib()
    ws = torch.empty(max(L.hc_maxmip_workspace_bytes(1, R), 16), dtype=torch.uint8, device=dev)
    _cuda.check(L.hc_maxmip(jobs, 1, ws.data_ptr(), ws.numel(), _cuda.stream_ptr()), "hc_maxmip")
    return MaxMipmap(flat, R, layer, vrange, patch_ok)


# ---------------------------------------------------------------------------
# scalar patch intersection (raycast.py:95-179)


def _patch_roots(h00, h10, h01, h11, u0, v0, du, dv, z0, dz, seg_len):
    e10, e01 = h10 - h00, h01 - h00
    kk = h11 - h10 - h01 + h00
    a = du * dv * kk
    b = du * e10 + dv * e01 + kk * (u0 * dv + v0 * du) - dz
    c = h00 + u0 * e10 + v0 * e01 + kk * u0 * v0 - z0
    roots = [1e300, 1e300]
    if abs(a) < 1e-12 * abs(b):
        if b != 0.0:
            roots[0] = -c / b
    else:
        disc = b * b - 4.0 * a * c
        if disc >= 0.0:
            sq = math.sqrt(disc)
            q = -0.5 * (b + sq) if b >= 0.0 else -0.5 * (b - sq)
            roots = [q / a, c / q] if q != 0.0 else [0.0, -b / a]
            if roots[1] < roots[0]:
                roots.reverse()
    for tau in roots:
        if 0.0 <= tau <= seg_len:
            return tau, min(max(u0 + tau * du, 0.0), 1.0), min(max(v0 + tau * dv, 0.0), 1.0)
    return None


def intersect_bilinear_patch(origin, direction, corner_heights, patch_min, patch_size: float,
                             t_range=None):
    """Nearest hit (t, (u, v)) of a ray with one bilinear patch, or None."""
    ox, oy, oz = (float(v) for v in origin)
    dx, dy, dz = (float(v) for v in direction)
    h00, h10, h01, h11 = (float(v) for v in corner_heights)
    s = float(patch_size)
    uo = (ox - float(patch_min[0])) / s
    vo = (oy - float(patch_min[1])) / s
    du, dv = dx / s, dy / s
    if t_range is None:
        lo, hi = 0.0, 1e300
        for pos, dd in ((uo, du), (vo, dv)):
            if dd != 0.0:
                ta, tb = (0.0 - pos) / dd, (1.0 - pos) / dd
                if ta > tb:
                    ta, tb = tb, ta
                lo, hi = max(lo, ta), min(hi, tb)
            elif pos < 0.0 or pos > 1.0:
                return None
        if lo > hi:
            return None
    else:
        lo, hi = float(t_range[0]), float(t_range[1])
        if lo > hi:
            return None
    hit = _patch_roots(h00, h10, h01, h11, uo + lo * du, vo + lo * dv, du, dv, oz + lo * dz, dz,
                       hi - lo)
    if hit is None:
        return None
    return lo + hit[0], (hit[1], hit[2])


# ---------------------------------------------------------------------------
# single-ray traversal through the GPU kernel


def traverse_batch(heights, valid, mipmap: MaxMipmap, rx, ry, rz, dx, dy, dz, hmin, hmax):
    """`_kernels.traverse_batch` on device tensors (float64 rays, per-lane outputs)."""
    import torch
    dev = heights.device
    f64 = lambda a: torch.as_tensor(a, dtype=torch.float64, device=dev).reshape(-1).contiguous()
    dxt = f64(dx)
    n = dxt.numel()
    full = lambda a: f64(a).expand(n).contiguous() if f64(a).numel() == 1 else f64(a)
    ins = [full(rx), full(ry), full(rz), dxt, full(dy), full(dz)]
    out = (torch.zeros(n, dtype=torch.uint8, device=dev), torch.zeros(n, dtype=torch.float64, device=dev),
           torch.full((n,), -1, dtype=torch.int32, device=dev),
           torch.full((n,), -1, dtype=torch.int32, device=dev),
           torch.zeros(n, dtype=torch.float64, device=dev), torch.zeros(n, dtype=torch.float64, device=dev))
    R = int(heights.shape[0])
    v8 = valid.to(torch.uint8).contiguous()
    _cuda.check(_cuda.lib().hc_traverse_batch(
        heights.contiguous().data_ptr(), v8.data_ptr(), mipmap._flat.data_ptr(), mipmap._off.data_ptr(),
        mipmap._w.data_ptr(), mipmap.n_levels, R - 1, *[t.data_ptr() for t in ins], n,
        C.c_double(hmin), C.c_double(hmax), *[o.data_ptr() for o in out], _cuda.stream_ptr()),
        "hc_traverse_batch")
    return out


def _raster_ray(layout, origin, direction):
    s = layout.texel_size
    return ((float(origin[0]) - layout.world_origin[0]) / s, (float(origin[1]) - layout.world_origin[1]) / s,
            float(origin[2]), float(direction[0]) / s, float(direction[1]) / s, float(direction[2]))


def traverse_cascade(origin, direction, raster: CascadeRaster, mipmap: MaxMipmap) -> HitRecord | None:
    vr = raster.valid_range(mipmap.layer)
    if vr is None:
        return None
    rx, ry, rz, dx, dy, dz = _raster_ray(raster.layout, origin, direction)
    out = traverse_batch(raster.layer(mipmap.layer), raster.valid, mipmap, rx, ry, rz, dx, dy, dz,
                         vr[0], vr[1])
    hit, t, ix, iy, u, v = (o.cpu().numpy()[0] for o in out)
    if not hit:
        return None
    o = np.asarray(origin, dtype=np.float64)
    d = np.asarray(direction, dtype=np.float64)
    pos = o + t * d
    return HitRecord(t=float(t), world_pos=(pos[0], pos[1], pos[2]), layer=mipmap.layer,
                     cascade=raster.layout.index, uv=(float(u), float(v)), patch=(int(ix), int(iy)))


def cast_through_cascades(origin, direction, rasters, mipmaps, layouts) -> HitRecord | None:
    """Nearest-first cascade walk with overlap blending (raycast.py:217-256)."""
    n = len(layouts)
    usable = lambda k: layouts[k] is not None and rasters[k] is not None and mipmaps[k] is not None
    for k in range(n):
        if not usable(k):
            continue
        hit = traverse_cascade(origin, direction, rasters[k], mipmaps[k])
        if hit is None:
            continue
        nk = k + 1
        if nk < n and usable(nk):
            lo, hi = layouts[nk].polygon.near_offset, layouts[k].polygon.far_offset
            if hi > lo:
                off = layouts[k].polygon.axis.offset_of(hit.world_pos[:2])
                if lo <= off <= hi:
                    other = traverse_cascade(origin, direction, rasters[nk], mipmaps[nk])
                    if other is not None:
                        w = (off - lo) / (hi - lo)
                        t = (1.0 - w) * hit.t + w * other.t
                        pos = np.asarray(origin, dtype=np.float64) + t * np.asarray(direction, dtype=np.float64)
                        return HitRecord(t=float(t), world_pos=(pos[0], pos[1], pos[2]), layer=hit.layer,
                                         cascade=hit.cascade, uv=hit.uv, patch=hit.patch,
                                         blend=(layouts[nk].index, float(w)))
        return hit
    return None

"""Cascade raster fill on the GPU (the paper's approximation pass).

Drop-in for `heightcast.discretize` (pkg/src/heightcast/discretize.py):
`discretize_cascade(layout, grid, table, params) -> CascadeRaster` with the
same semantics — every visible texel inside the gridded domain gets both
smoothed layers (terrain, water surface) and `valid`; all other texels hold the
sentinel `height_range.min - 1` (discretize.py:52-108) — computed by the sm_100a
kernel `hc_discretize` (mask, cell lookup and Eq. 1/2 fused, one thread per
texel).  Arrays are CUDA tensors: terrain / water float32 [R, R], valid bool.
Heights agree with the float64 reference within the float32 tolerance stated
in DESIGN.md; `valid` and the mask are bit-exact.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _cuda
from ._engine import fill_cascade_raster
from .cascade import CascadeLayout
from .grid import AdaptiveGrid, InfluenceTable
from .rbf import RbfParams


@dataclass
class CascadeRaster:
    """Discretized heights of one cascade, both layers (discretize.py:27-49)."""

    layout: CascadeLayout
    terrain: object              # torch.float32 [R, R] (CUDA), [iy, ix]
    water: object                # water surface elevation
    valid: object                # torch.bool [R, R]: visible AND inside the grid
    sentinel: float

    def layer(self, name: str):
        if name == "terrain":
            return self.terrain
        if name == "water":
            return self.water
        raise ValueError(f"unknown layer {name!r}")

    def valid_range(self, name: str):
        """(min, max) of a layer over valid texels, or None if nothing is valid."""
        vals = self.layer(name)[self.valid]
        if vals.numel() == 0:
            return None
        return float(vals.min()), float(vals.max())


def compute_visibility_mask(layout: CascadeLayout):
    """layout.mask on the GPU (cascade.py:507-521), bool [R, R] CUDA tensor."""
    import torch
    _cuda.require_cuda()
    R = layout.resolution
    mask = torch.empty((R, R), dtype=torch.uint8, device="cuda")
    desc = _cuda.HcCascadeRaster()
    fill_cascade_raster(desc, layout, None, None, None, mask)
    _cuda.check(_cuda.lib().hc_visibility_mask(C.byref(desc), _cuda.stream_ptr()),
                "hc_visibility_mask")
    return mask.bool()


def discretize_cascade(layout: CascadeLayout, grid: AdaptiveGrid, table: InfluenceTable,
                       params: RbfParams) -> CascadeRaster:
    """Evaluate both smoothing layers at every visible texel of a layout."""
    import torch
    if table.sigma != params.sigma:
        raise ValueError("influence table was built for a different sigma")
    _cuda.require_cuda()
    gdev = grid.device_view()
    inf = gdev.influence(table)
    R = layout.resolution
    dev = gdev.device
    terrain = torch.empty((R, R), dtype=torch.float32, device=dev)
    water = torch.empty((R, R), dtype=torch.float32, device=dev)
    valid = torch.empty((R, R), dtype=torch.uint8, device=dev)
    mask = torch.empty((R, R), dtype=torch.uint8, device=dev)
    counters = torch.zeros(_cuda.N_COUNTERS, dtype=torch.int64, device=dev)
    desc = (_cuda.HcCascadeRaster * 1)()
    fill_cascade_raster(desc[0], layout, terrain, water, valid, mask)
    sentinel = grid.height_range[0] - 1.0
    _cuda.check(_cuda.lib().hc_discretize(desc, 1, C.byref(inf.view), C.c_float(sentinel),
                                          counters.data_ptr(), _cuda.stream_ptr()), "hc_discretize")
    if int(counters[_cuda.CNT_ZERO_WEIGHT].item()):
        raise ValueError(f"zero weight sum in cascade {layout.index}: influence table "
                         f"inconsistent with sigma={params.sigma}")
    layout.mask = mask.bool()
    return CascadeRaster(layout, terrain, water, valid.bool(), sentinel)


def write_pgm(values, lo: float, hi: float, target) -> None:
    """16-bit PGM of a height array, rows top-to-bottom (discretize.py:122-140)."""
    v = values.detach().cpu().numpy() if hasattr(values, "detach") else np.asarray(values)
    v = v.astype(np.float64)
    if hi <= lo:
        hi = lo + 1.0
    pix = np.clip(np.rint((v - lo) / (hi - lo) * 65535.0), 0, 65535).astype(">u2")[::-1, :]
    header = f"P5\n{pix.shape[1]} {pix.shape[0]}\n65535\n".encode("ascii")
    if hasattr(target, "write"):
        target.write(header)
        target.write(pix.tobytes())
    else:
        with open(target, "wb") as fh:
            fh.write(header)
            fh.write(pix.tobytes())

"""Truncated-Gaussian RBF kernel (Eq. 1) and single-point approximation (Eq. 2).

Drop-in for `heightcast.rbf` (pkg/src/heightcast/rbf.py).  `weight` /
`weights_vec` are the scalar/vector host forms of Eq. 1 (rbf.py:64-84), kept as
host arithmetic because they are API helpers, not the per-frame path.
`approximate` (rbf.py:133-156) evaluates Eq. 2 for one point on the GPU in
float64 (`hc_eval_points`), anchored at the first listed influencer like the
reference, so it matches the reference to ~1e-15 relative.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _cuda
from .grid import TRUNCATION, AdaptiveGrid, InfluenceTable, OutsideDomainError

_CUT_SQ = TRUNCATION * TRUNCATION          # 12.25
_REMAINDER = math.exp(-_CUT_SQ / 2.0)      # exp(-6.125)
_CUT_EDGE = _CUT_SQ * (1.0 - 1e-12)

LAYERS = ("terrain", "water")


@dataclass(frozen=True)
class RbfParams:
    sigma: float = 1.0
    truncation: float = TRUNCATION

    def __post_init__(self):
        if self.sigma <= 0:
            raise ValueError("sigma must be positive")
        if self.truncation != TRUNCATION:
            raise ValueError("truncation is a fixed kernel constant")


@dataclass(frozen=True)
class SampleValue:
    value: float
    weight_sum: float
    influencer_count: int

    @property
    def defined(self) -> bool:
        return self.weight_sum > 0.0


def weight(center, cell_size: float, point, params: RbfParams) -> float:
    """Eq. 1: exp(-(d/c)^2 / (2 sigma^2)) - exp(-3.5^2/2), exactly 0 beyond 3.5 sigma c."""
    if cell_size <= 0:
        raise ValueError("cell_size must be positive")
    dx = center[0] - point[0]
    dy = center[1] - point[1]
    cs = cell_size * params.sigma
    r2 = (dx * dx + dy * dy) / (cs * cs)
    if r2 >= _CUT_EDGE:
        return 0.0
    return max(0.0, math.exp(-r2 / 2.0) - _REMAINDER)


def weights_vec(dx, dy, cell_sizes, sigma):
    cs = np.asarray(cell_sizes) * sigma
    r2 = (dx * dx + dy * dy) / (cs * cs)
    w = np.maximum(np.exp(-0.5 * r2) - _REMAINDER, 0.0)
    w[r2 >= _CUT_EDGE] = 0.0
    return w


def approximate(point, layer: str, grid: AdaptiveGrid, table: InfluenceTable,
                params: RbfParams) -> SampleValue:
    """Smoothed value of one layer at a world position (GPU, float64)."""
    import torch
    if layer not in LAYERS:
        raise ValueError(f"unknown layer {layer!r}")
    if table.sigma != params.sigma:
        raise ValueError("influence table was built for a different sigma")
    cell = grid.cell_at(float(point[0]), float(point[1]))
    if cell < 0:
        raise OutsideDomainError(f"position {tuple(point)} is outside the gridded domain")
    gdev = grid.device_view()
    inf = gdev.influence(table)
    dev = gdev.device
    px = torch.tensor([float(point[0])], dtype=torch.float64, device=dev)
    py = torch.tensor([float(point[1])], dtype=torch.float64, device=dev)
    cells = torch.tensor([cell], dtype=torch.int32, device=dev)
    out = [torch.empty(1, dtype=torch.float64, device=dev) for _ in range(3)]
    cnt = torch.empty(1, dtype=torch.int64, device=dev)
    _cuda.check(_cuda.lib().hc_eval_points(C.byref(inf.view), px.data_ptr(), py.data_ptr(),
                                           cells.data_ptr(), 1, out[0].data_ptr(), out[1].data_ptr(),
                                           out[2].data_ptr(), cnt.data_ptr(), _cuda.stream_ptr()),
                "hc_eval_points")
    t, w, ws = (float(o.item()) for o in out)
    if ws <= 0.0:
        raise ValueError(f"zero weight sum at {tuple(point)}: influence table inconsistent "
                         f"with sigma={params.sigma}")
    return SampleValue(value=t if layer == "terrain" else w, weight_sum=ws,
                       influencer_count=int(cnt.item()))

"""Deterministic inputs shared by tests/golden/make_golden.py and the tests.

Inputs are regenerated from seeds (numpy PCG64 streams are stable), so the
golden files only need to hold the reference's outputs.
"""

from __future__ import annotations

import numpy as np

# synthetic grids whose arrays (and influence tables) are pinned against the reference
GRID_SPECS = [
    {"name": "flat100", "kind": "flat", "seed": 0, "cells": 100, "max_depth": None, "sigmas": [1.0]},
    {"name": "ramp4096", "kind": "ramp", "seed": 0, "cells": 4096, "max_depth": None, "sigmas": [1.0]},
    {"name": "hill3000", "kind": "hill", "seed": 42, "cells": 3000, "max_depth": None, "sigmas": [1.0, 2.0]},
    {"name": "pond3000", "kind": "pond", "seed": 42, "cells": 3000, "max_depth": None, "sigmas": [1.0, 0.5]},
    {"name": "pond20k_d7", "kind": "pond", "seed": 7, "cells": 20000, "max_depth": 7, "sigmas": [1.0]},
]

PLAN_GRIDS = {
    "pond3000": {"kind": "pond", "seed": 42, "cells": 3000},
    "ramp4096": {"kind": "ramp", "seed": 0, "cells": 4096},
}


def plan_poses(grid_name: str, n: int = 40):
    """Random camera poses (including looking-away and steep-down views)."""
    rng = np.random.default_rng(1000 + sum(map(ord, grid_name)))
    ext = 2048.0 if grid_name.startswith("pond") else 256.0
    poses = []
    for i in range(n):
        eye = (float(rng.uniform(-0.3, 1.3) * ext), float(rng.uniform(-0.3, 1.3) * ext),
               float(rng.uniform(10.0, 0.4 * ext + 50.0)))
        if i % 10 == 7:      # nearly straight down
            la = (eye[0] + 1e-7 * eye[2], eye[1], 0.0)
        else:
            la = (float(rng.uniform(0, ext)), float(rng.uniform(0, ext)), float(rng.uniform(0, 60)))
        look = tuple(b - a for a, b in zip(eye, la))
        cam = dict(eye=eye, look_dir=look, up=(0.0, 0.0, 1.0), fov_y=float(rng.uniform(30, 90)),
                   aspect=float(rng.uniform(0.6, 2.2)), near_clip=1.0,
                   far_clip=float(rng.choice([0.8 * ext, 3.0 * ext])))
        res = int(rng.choice([64, 128, 256, 1024]))
        ov = "auto" if rng.random() < 0.7 else float(rng.uniform(0.0, 0.02 * ext))
        poses.append({"id": i, "camera": cam, "res": res, "overlap": ov})
    return poses


def _raster(rng, n, kind):
    y, x = np.mgrid[0:n, 0:n].astype(np.float64)
    if kind == "flat":
        h = np.full((n, n), 12.5)
    elif kind == "ramp":
        h = 3.0 + 0.37 * x - 0.11 * y
    elif kind == "saddle":
        h = 20.0 + 0.02 * (x - n / 2) * (y - n / 2)
    else:
        h = 15.0 + np.zeros((n, n))
        for _ in range(4):
            kx, ky = rng.uniform(0.02, 0.3, 2)
            h += rng.uniform(1, 8) * np.sin(kx * x + rng.uniform(0, 6)) * np.cos(ky * y + rng.uniform(0, 6))
        h += rng.normal(0, 0.6, (n, n))
    h = h.astype(np.float32).astype(np.float64)       # float32-representable, like HBM rasters
    valid = np.ones((n, n), dtype=bool)
    if kind == "holes":
        for _ in range(5):
            cx, cy, r = rng.uniform(0, n, 3)
            valid &= (x - cx) ** 2 + (y - cy) ** 2 > (r / 4) ** 2
    return np.ascontiguousarray(h), valid


def _rays(rng, n_rays, n, hmin, hmax):
    m = n_rays
    rx = rng.uniform(-0.4 * n, 1.4 * n, m)
    ry = rng.uniform(-0.4 * n, 1.4 * n, m)
    rz = rng.uniform(hmin - 5.0, hmax + 0.8 * n, m)
    tx = rng.uniform(0, n, m)
    ty = rng.uniform(0, n, m)
    tz = rng.uniform(hmin - 3.0, hmax + 1.0, m)
    d = np.stack([tx - rx, ty - ry, tz - rz], axis=1)
    # special directions: vertical, axis-parallel, grazing, upward
    k = m // 10
    d[:k, 0] = 0.0
    d[:k, 1] = 0.0
    d[:k, 2] = -1.0
    d[k:2 * k, 1] = 0.0
    d[2 * k:3 * k, 0] = 0.0
    d[3 * k:4 * k, 2] = rng.uniform(-1e-3, 1e-3, k)
    d[4 * k:4 * k + k // 2, 2] = np.abs(d[4 * k:4 * k + k // 2, 2]) + 0.1
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    s = rng.uniform(0.5, 4.0)           # texel size: raster-space ray dx = d / s
    return (rx, ry, rz, d[:, 0] / s, d[:, 1] / s, d[:, 2].copy())


def traversal_cases(n_rasters: int = 24, n_rays: int = 500, size: int = 64):
    kinds = ["flat", "ramp", "saddle", "holes"] + ["smooth"] * (n_rasters - 4)
    out = []
    for i, kind in enumerate(kinds):
        rng = np.random.default_rng(5000 + i)
        if kind == "smooth" and i % 3 == 0:
            kind = "holes"
        n = size if i % 5 else size + 1 + i % 7          # some non-power-of-two sizes
        h, valid = _raster(rng, n, kind)
        vals = h[valid]
        rays = _rays(rng, n_rays, n, float(vals.min()), float(vals.max()))
        out.append({"name": f"r{i:02d}_{kind}", "heights": h, "valid": valid, "rays": rays})
    return out


def rbf_cases(n: int = 20, n_points: int = 100):
    out = []
    for i in range(n):
        kind = ("pond", "hill", "ramp", "pond")[i % 4]
        out.append({"name": f"g{i:02d}", "kind": kind, "seed": 300 + i,
                    "cells": int(80 + 21 * i) if kind != "ramp" else 144, "max_depth": 6,
                    "sigma": (1.0, 2.0, 0.5, 1.0)[i % 4], "n_points": n_points})
    return out


def rbf_points(domain, seed: int, n: int):
    rng = np.random.default_rng(9000 + seed)
    x = rng.uniform(domain.xmin, domain.xmax, n)
    y = rng.uniform(domain.ymin, domain.ymax, n)
    # keep points strictly inside the domain
    x = np.clip(x, domain.xmin + 1e-6, domain.xmax - 1e-6)
    y = np.clip(y, domain.ymin + 1e-6, domain.ymax - 1e-6)
    return np.stack([x, y], axis=1)


# ---- scalar twins (traverse_cascade / cast_through_cascades, raycast.py:195-256)

TWIN_GRID = {"kind": "pond", "seed": 42, "cells": 3000}
TWIN_POSES = [
    {"eye": (150.0, 120.0, 160.0), "look_at": (1100.0, 1150.0, 20.0), "fov_y": 55.0, "res": 128},
    {"eye": (1900.0, 300.0, 90.0), "look_at": (900.0, 1300.0, 10.0), "fov_y": 70.0, "res": 256},
    {"eye": (1024.0, -150.0, 300.0), "look_at": (1024.0, 1024.0, 0.0), "fov_y": 40.0, "res": 64},
]
TWIN_W, TWIN_H = 48, 32          # image whose every pixel's ray is cast


def twin_camera_args(pose):
    eye, la = pose["eye"], pose["look_at"]
    return dict(eye=eye, look_dir=tuple(b - a for a, b in zip(eye, la)), up=(0.0, 0.0, 1.0),
                fov_y=pose["fov_y"], aspect=TWIN_W / TWIN_H, near_clip=1.0, far_clip=6000.0)


def twin_raster(origin, texel, R, mask):
    """Deterministic float32-representable (terrain, water, valid) for a cascade layout.

    A smooth polynomial of the texel centre plus integer-hash noise, built from
    + and * only (no libm), so every host computes the same bits.  Water lies
    above the terrain inside a disc, equals it elsewhere."""
    i = np.arange(R, dtype=np.float64)
    x = origin[0] + i * texel
    y = origin[1] + i * texel
    X, Y = np.meshgrid(x, y)
    u, v = (X - 1024.0) / 1024.0, (Y - 1024.0) / 1024.0
    h = 25.0 + 18.0 * u * v - 9.0 * u * u * u + 6.0 * v * v
    iy, ix = np.meshgrid(np.arange(R, dtype=np.int64), np.arange(R, dtype=np.int64), indexing="ij")
    kx = np.floor(X / 7.0).astype(np.int64)
    ky = np.floor(Y / 7.0).astype(np.int64)
    hsh = ((kx * 73856093) ^ (ky * 19349663)) % 1009
    h = h + hsh.astype(np.float64) * (4.0 / 1009.0)
    terrain = h.astype(np.float32).astype(np.float64)
    pond = (X - 1000.0) ** 2 + (Y - 1100.0) ** 2 < 350.0 ** 2
    water = np.where(pond, np.maximum(terrain, 31.25), terrain).astype(np.float32).astype(np.float64)
    valid = np.ascontiguousarray(mask, dtype=bool).copy()
    valid[(ix * 7 + iy * 3) % 97 == 0] = False          # scattered invalid texels
    return np.ascontiguousarray(terrain), np.ascontiguousarray(water), valid

"""Shared helpers for the parity tests."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(str(a.dtype).encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def unhex(s) -> float:
    return float.fromhex(s)


def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        return json.load(fh)


def npz(name):
    return np.load(os.path.join(GOLDEN, name))


def demo_setup():
    """Demo scene (scene.py:181-196) built with this package's host code."""
    import heightcast_oracle as O
    from paper_2201_10887_b200 import scene
    sc = scene.demo_scene()
    g = scene.scene_grid(sc)
    t = O.build_influence_table(g, sc.sigma)
    cfg = scene.scene_frame_config(sc)
    st = scene.scene_settings(sc)
    return sc, g, t, cfg, st


class F64Raster:
    """float64 view of float32 GPU rasters, for feeding the oracle the GPU's own data."""

    def __init__(self, terrain, water, valid):
        self.terrain = np.ascontiguousarray(terrain, dtype=np.float64)
        self.water = np.ascontiguousarray(water, dtype=np.float64)
        self.valid = np.ascontiguousarray(valid, dtype=bool)

    def layer(self, name):
        return self.terrain if name == "terrain" else self.water

"""The benchmark configurations C1-C5 of BASELINE.json / SURVEY.md §8(d).

Each config is a synthetic grid (built by `generate_synthetic`, identical to the
reference generator), a cascade setup and one or more cameras.  Cameras use
up=(0,0,1), fov_y=55, near=1, far=6000 and overlap="auto" throughout.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

from .cascade import CameraView
from .render import CascadeSettings, FrameConfig


@dataclass(frozen=True)
class BenchConfig:
    name: str
    description: str
    kind: str
    seed: int
    cells: int
    max_depth: int | None
    sigma: float
    cascades: int
    resolution: int
    width: int
    height: int
    eye: tuple
    look_at: tuple
    views: int = 1                 # C4: orbit views
    orbit: dict = field(default_factory=dict)

    def settings(self) -> CascadeSettings:
        return CascadeSettings(resolution=self.resolution, overlap="auto", count=self.cascades)

    def camera(self, view: int = 0) -> CameraView:
        eye, la = self.eye, self.look_at
        if self.views > 1 or self.orbit:
            o = self.orbit
            ang = 2.0 * math.pi * view / max(self.views, 1)
            eye = (o["cx"] + o["radius"] * math.cos(ang), o["cy"] + o["radius"] * math.sin(ang), o["z"])
            la = (o["cx"], o["cy"], o["look_z"])
        look = tuple(b - a for a, b in zip(eye, la))
        return CameraView(eye=eye, look_dir=look, up=(0.0, 0.0, 1.0), fov_y=55.0,
                          aspect=self.width / self.height, near_clip=1.0, far_clip=6000.0)

    def frame_config(self, view: int = 0) -> FrameConfig:
        return FrameConfig(width=self.width, height=self.height, camera=self.camera(view))

    def grid(self):
        from .synth import generate_synthetic
        return generate_synthetic(self.kind, self.seed, self.cells, max_depth=self.max_depth)


CONFIGS = {
    "C1": BenchConfig("C1", "synthetic 256x256 uniform-grid heightfield, 1 cascade, 512x512 image",
                      "ramp", 0, 65536, None, 1.0, 1, 1024, 512, 512, (-100.0, -100.0, 250.0),
                      (600.0, 600.0, 20.0)),
    "C2": BenchConfig("C2", "synthetic 1024x1024 adaptive quadtree DEM, 4 cascades, 1920x1080",
                      "pond", 7, 100_000, 7, 1.0, 4, 1024, 1920, 1080, (200.0, 150.0, 300.0),
                      (1100.0, 1200.0, 40.0)),
    "C3": BenchConfig("C3", "synthetic 4096x4096 adaptive quadtree, 8 cascades, 3840x2160, wide support",
                      "pond", 11, 300_000, 9, 2.0, 8, 2048, 3840, 2160, (150.0, 100.0, 350.0),
                      (1150.0, 1250.0, 50.0)),
    "C4": BenchConfig("C4", "64 camera views over the 4096^2 heightfield, 1920x1080 each",
                      "pond", 11, 300_000, 9, 2.0, 8, 2048, 1920, 1080, (0, 0, 0), (0, 0, 0), views=64,
                      orbit={"cx": 1024.0, "cy": 1024.0, "radius": 1100.0, "z": 350.0, "look_z": 40.0}),
    "C5": BenchConfig("C5", "16384x16384 adaptive quadtree lattice, 8 cascades, 4K in screen strips",
                      "pond", 13, 2_000_000, 11, 1.0, 8, 2048, 3840, 2160, (150.0, 100.0, 350.0),
                      (1150.0, 1250.0, 50.0)),
}

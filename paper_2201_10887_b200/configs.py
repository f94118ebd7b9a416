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

    # ---- benchmark camera path (both bench.py arms render the same frames)

    def path_camera(self, i: int, rank: int = 0, world: int = 1) -> CameraView:
        """Camera of frame i of the benchmark's moving-camera path.

        The reference's benchmark moves the camera every frame by lerping eye and
        look_at between two poses (cli.py:127-131).  Here pose 1 is pose 0's eye
        turned PATH_TURN_DEG about the look-at point; the lerp parameter runs
        0 -> 1 -> 0 over 2 * PATH_FRAMES frames (a triangle wave, so any number of
        steps stays on the path).  C4 cycles through its orbit views instead.
        With world > 1 (view sharding) rank r's path is turned by 360 r / world
        degrees about the domain centre (1024, 1024)."""
        if self.views > 1:
            return self.camera((i * max(world, 1) + rank) % self.views)
        ph = i % (2 * PATH_FRAMES)
        a = (ph if ph <= PATH_FRAMES else 2 * PATH_FRAMES - ph) / PATH_FRAMES
        eye0, la = self.eye, self.look_at
        ang = math.radians(PATH_TURN_DEG)
        ca, sa = math.cos(ang), math.sin(ang)
        ex, ey = eye0[0] - la[0], eye0[1] - la[1]
        eye1 = (la[0] + ca * ex - sa * ey, la[1] + sa * ex + ca * ey, eye0[2])
        eye = tuple((1 - a) * p + a * q for p, q in zip(eye0, eye1))
        if world > 1:
            rot = 2.0 * math.pi * rank / world
            cr, sr = math.cos(rot), math.sin(rot)
            turn = lambda p: (1024.0 + cr * (p[0] - 1024.0) - sr * (p[1] - 1024.0),
                              1024.0 + sr * (p[0] - 1024.0) + cr * (p[1] - 1024.0), p[2])
            eye, la = turn(eye), turn(la)
        look = tuple(b - p for p, b in zip(eye, la))
        return CameraView(eye=eye, look_dir=look, up=(0.0, 0.0, 1.0), fov_y=55.0,
                          aspect=self.width / self.height, near_clip=1.0, far_clip=6000.0)

    def path_frame_config(self, i: int, rank: int = 0, world: int = 1) -> FrameConfig:
        return FrameConfig(width=self.width, height=self.height, camera=self.path_camera(i, rank, world))

    def workload(self, grid=None, table=None) -> dict:
        """The `config` dict of a bench.py line (identical in both arms)."""
        d = {"workload": f"{self.name}: {self.description}", "sigma": self.sigma, "cascades": self.cascades,
             "cascade_res": self.resolution, "image": [self.width, self.height],
             "camera_path": (f"{self.views} orbit views, cycled" if self.views > 1 else
                             f"eye lerped {PATH_TURN_DEG:g} deg about look_at and back over "
                             f"{2 * PATH_FRAMES} frames (cli.py:127-131 style), one pose per step")}
        if grid is not None:
            d["grid_cells"] = grid.n_cells
        if table is not None and grid is not None:
            d["mean_influence_list"] = round(len(table.indices) / max(grid.n_cells, 1), 2)
        return d

    def grid(self, native_paint: bool = True):
        from .synth import generate_synthetic
        return generate_synthetic(self.kind, self.seed, self.cells, max_depth=self.max_depth,
                                  native_paint=native_paint)


PATH_FRAMES = 60          # frames from pose 0 to pose 1 of the benchmark camera path
PATH_TURN_DEG = 45.0      # pose 1: pose 0's eye turned about the look-at point


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

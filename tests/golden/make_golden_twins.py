"""Golden outputs of the reference's scalar ray API (raycast.py:195-256):
`traverse_cascade` and `cast_through_cascades` on K=3 cascades planned by the
reference over the pond3000 grid, with deterministic float32-representable
rasters (tests/golden_inputs.py:twin_raster), for every pixel ray of a 48x32
image from three poses.  Writes tests/golden/scalar_twins.npz.

Run in the build container only (needs /root/reference):
    python tests/golden/make_golden_twins.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import golden_inputs as gi  # noqa: E402
import refload  # noqa: E402


def main():
    ref = refload.load()
    ref.synth._MAX_DEPTH = 6
    g = ref.generate_synthetic(gi.TWIN_GRID["kind"], gi.TWIN_GRID["seed"], gi.TWIN_GRID["cells"])
    out = {}
    for p, pose in enumerate(gi.TWIN_POSES):
        cam = ref.CameraView(**gi.twin_camera_args(pose))
        _, _, lays = ref.plan_cascades(cam, g, pose["res"], "auto")
        rasters, mips = [], {"terrain": [], "water": []}
        for L in lays:
            if L is None:
                rasters.append(None)
                for layer in mips:
                    mips[layer].append(None)
                continue
            ter, wat, val = gi.twin_raster(L.world_origin, L.texel_size, L.resolution, L.mask)
            r = ref.raycast.CascadeRaster(L, ter, wat, val, float(ter.min()) - 1.0)
            rasters.append(r)
            for layer in mips:
                mips[layer].append(ref.build_max_mipmap(r, layer))
        origin = np.asarray(cam.eye, dtype=np.float64)
        dirs = ref.render.camera_ray_dirs(cam, gi.TWIN_W, gi.TWIN_H).reshape(-1, 3)
        n = len(dirs)
        out[f"p{p}_dirs"] = dirs
        out[f"p{p}_n_cascades"] = np.array(len(lays))
        for layer in ("terrain", "water"):
            # cast_through_cascades: (hit, t, x, y, z, cascade, u, v, ix, iy, blend_k, blend_w)
            cast = np.full((n, 12), np.nan)
            for i in range(n):
                h = ref.cast_through_cascades(origin, dirs[i], rasters, mips[layer], lays)
                if h is None:
                    cast[i, 0] = 0
                    continue
                b = h.blend if h.blend is not None else (-1, np.nan)
                cast[i] = (1, h.t, *h.world_pos, h.cascade, *h.uv, *h.patch, b[0], b[1])
            out[f"p{p}_{layer}_cast"] = cast
            # traverse_cascade on every cascade: (hit, t, u, v, ix, iy)
            for k, (r, m) in enumerate(zip(rasters, mips[layer])):
                if r is None:
                    continue
                tr = np.full((n, 6), np.nan)
                for i in range(n):
                    h = ref.traverse_cascade(origin, dirs[i], r, m)
                    tr[i] = (0, np.nan, np.nan, np.nan, -1, -1) if h is None else (1, h.t, *h.uv, *h.patch)
                out[f"p{p}_{layer}_trav{k}"] = tr
        hits = int(np.nansum(out[f"p{p}_terrain_cast"][:, 0]))
        blends = int(np.sum(out[f"p{p}_terrain_cast"][:, 10] >= 0))
        print(f"pose {p}: {len(lays)} cascades, {n} rays, {hits} terrain hits, {blends} blended")
    np.savez_compressed(os.path.join(HERE, "scalar_twins.npz"), **out)


if __name__ == "__main__":
    main()

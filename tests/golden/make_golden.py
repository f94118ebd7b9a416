"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Every value stored here was produced by the reference package
(pkg/src/heightcast, imported as `heightcast_ref`); inputs are regenerated in
the tests from the seeds recorded here (numpy's PCG64 streams are stable), so
only outputs are stored.  Bit-exact quantities are stored as sha256 digests or
float.hex strings; tolerance quantities as float64 arrays.  Nothing on the GPU
box reads /root/reference: the tests only read these files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import refload  # noqa: E402

sys.path.insert(0, os.path.dirname(HERE))
import golden_inputs as gi  # noqa: E402  (tests/golden_inputs.py: shared input generators)


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(str(a.dtype).encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def hx(x) -> str:
    return float(x).hex()


def grid_digest(g) -> dict:
    return {"centers": sha(g.centers), "sizes": sha(g.sizes), "terrain": sha(g.terrain),
            "water_depth": sha(g.water_depth), "tile_index": sha(g._tile_index),
            "height_range": [hx(v) for v in g.height_range], "min_cell": hx(g.min_cell_size),
            "n_cells": int(g.n_cells)}


def main():
    ref = refload.load()
    out = {}

    # -- 1. synthetic grids + influence tables ---------------------------------
    grids = {}
    for spec in gi.GRID_SPECS:
        ref.synth._MAX_DEPTH = spec["max_depth"] if spec["max_depth"] is not None else 6
        g = ref.generate_synthetic(spec["kind"], spec["seed"], spec["cells"])
        d = grid_digest(g)
        for sigma in spec["sigmas"]:
            t = ref.build_influence_table(g, sigma)
            d[f"table_{sigma}"] = {"offsets": sha(t.offsets), "indices": sha(t.indices)}
        grids[spec["name"]] = d
    ref.synth._MAX_DEPTH = 6
    out["grids"] = grids

    # -- 2. SPEC known answers (SPEC.md examples), evaluated by the reference --
    P1 = ref.RbfParams(sigma=1.0)
    known = {
        "weight_0": hx(ref.weight((0.0, 0.0), 1.0, (0.0, 0.0), P1)),
        "weight_trunc": hx(ref.weight((0.0, 0.0), 2.0, (7.0, 0.0), P1)),
        "weight_far": hx(ref.weight((0.0, 0.0), 1.0, (10.0, 0.0), P1)),
        "split_1_8": [hx(v) for v in ref.split_depths(1.0, 8.0)],
        "split_10_1000": [hx(v) for v in ref.split_depths(10.0, 1000.0)],
        "patch_flat": None,
    }
    r = ref.intersect_bilinear_patch((0.5, 0.5, 10.0), (0.0, 0.0, -1.0), (7.0, 7.0, 7.0, 7.0), (0.0, 0.0), 1.0)
    known["patch_flat"] = [hx(r[0]), hx(r[1][0]), hx(r[1][1])]
    known["colormap"] = [list(ref.depth_colormap(v, (0.0, 4.0))) for v in (0.0, 2.0, 4.0, float("nan"))]
    poly = ref.CascadePolygon(np.array([[0.0, 0.0], [4.1, 0.0], [4.1, 3.0], [0.0, 3.0]]), 0.0, 1.0,
                              ref.ViewAxis((0.0, 0.0), (1.0, 0.0)))
    lay = ref.fit_layout(poly, 64, 2.0)
    lo, hi = lay.widened_box()
    known["fit_4.1x3"] = {"box": [hx(v) for v in (hi - lo)], "origin": [hx(v) for v in lay.world_origin],
                          "texel": hx(lay.texel_size), "mask": sha(lay.mask)}
    out["known"] = known

    # -- 3. cascade plans (K=3) over random poses ------------------------------
    plans = []
    for gname, grid_args in gi.PLAN_GRIDS.items():
        ref.synth._MAX_DEPTH = grid_args.get("max_depth") or 6
        g = ref.generate_synthetic(grid_args["kind"], grid_args["seed"], grid_args["cells"])
        for pose in gi.plan_poses(gname):
            cam = ref.CameraView(**pose["camera"])
            rec = {"grid": gname, "pose": pose["id"]}
            try:
                hull, polys, lays = ref.plan_cascades(cam, g, pose["res"], pose["overlap"])
            except ref.NothingVisibleError:
                rec["nothing_visible"] = True
                plans.append(rec)
                continue
            rec["hull"] = sha(hull)
            rec["cascades"] = []
            for L in lays:
                if L is None:
                    rec["cascades"].append(None)
                    continue
                rec["cascades"].append({
                    "origin": [hx(v) for v in L.world_origin], "texel": hx(L.texel_size),
                    "res": int(L.resolution), "verts": sha(L.polygon.vertices),
                    "near": hx(L.polygon.near_offset), "far": hx(L.polygon.far_offset),
                    "box_texel": list(L.box_texel), "box_steps": list(L.box_steps),
                    "mask": sha(L.mask), "mask_sum": int(L.mask.sum()), "index": L.index})
            plans.append(rec)
    ref.synth._MAX_DEPTH = 6
    out["plans"] = plans

    # -- 4. traversal on random rasters (SPEC acceptance: >=1e4 rays, >=20 rasters)
    trav = {}
    for case in gi.traversal_cases():
        h, valid = case["heights"], case["valid"]
        rr = ref.raycast.CascadeRaster(None, h, h, valid, float(h.min()) - 1.0)
        mip = ref.build_max_mipmap(rr, "terrain")
        rx, ry, rz, dx, dy, dz = case["rays"]
        n = len(dx)
        o = (np.zeros(n, np.uint8), np.zeros(n), np.full(n, -1, np.int32), np.full(n, -1, np.int32),
             np.zeros(n), np.zeros(n))
        vr = rr.valid_range("terrain")
        ref._kernels.traverse_batch(h, valid, mip._flat, mip._off, mip._w, mip._h, mip.n_levels,
                                    h.shape[0] - 1, rx, ry, rz, dx, dy, dz, vr[0], vr[1], *o)
        trav[case["name"]] = {"mip": sha(mip._flat), "hit": o[0], "t": o[1], "ix": o[2], "iy": o[3],
                              "u": o[4], "v": o[5], "vrange": np.array(vr)}
    np.savez_compressed(os.path.join(HERE, "traverse_rays.npz"),
                        **{f"{name}__{k}": v for name, d in trav.items() for k, v in d.items() if k != "mip"})
    out["traverse_mip_sha"] = {name: d["mip"] for name, d in trav.items()}

    # -- 5. Eq. 2 at random points on random small grids -----------------------
    rbf = {}
    for case in gi.rbf_cases():
        ref.synth._MAX_DEPTH = case["max_depth"]
        g = ref.generate_synthetic(case["kind"], case["seed"], case["cells"])
        t = ref.build_influence_table(g, case["sigma"])
        P = ref.RbfParams(sigma=case["sigma"])
        pts = gi.rbf_points(g.domain, case["seed"], case["n_points"])
        vals = np.array([[ref.approximate(p, "terrain", g, t, P).value,
                          ref.approximate(p, "water", g, t, P).value,
                          ref.approximate(p, "terrain", g, t, P).weight_sum,
                          ref.approximate(p, "terrain", g, t, P).influencer_count] for p in pts])
        rbf[case["name"]] = vals
    ref.synth._MAX_DEPTH = 6
    np.savez_compressed(os.path.join(HERE, "rbf_points.npz"), **rbf)

    # -- 6. demo scene frame: reference rasters, and the reference raycast on the
    #       float32-rounded rasters (what the GPU path stores in HBM)
    sc = ref.demo_scene()
    g = ref.scene.scene_grid(sc)
    t = ref.build_influence_table(g, sc.sigma)
    cfg = ref.scene.scene_frame_config(sc)
    st = ref.CascadeSettings(resolution=sc.cascade_res, overlap=sc.overlap)
    fr = ref.render_frame(cfg, g, t, ref.RbfParams(sigma=sc.sigma), st, debug=True)
    demo = {"pixels_sha": sha(fr.pixels), "visible_texels": fr.visible_texels, "rays_hit": fr.rays_hit}
    rng = np.random.default_rng(7)
    samples = {}
    r32 = []
    for k, R in enumerate(fr.debug["rasters"]):
        demo[f"valid_{k}"] = sha(R.valid)
        iy, ix = np.nonzero(R.valid)
        pick = rng.choice(len(ix), size=min(2000, len(ix)), replace=False)
        samples[f"idx_{k}"] = np.stack([iy[pick], ix[pick]], axis=1)
        samples[f"terrain_{k}"] = R.terrain[iy[pick], ix[pick]]
        samples[f"water_{k}"] = R.water[iy[pick], ix[pick]]
        q = ref.raycast.CascadeRaster(R.layout, R.terrain.astype(np.float32).astype(np.float64),
                                      R.water.astype(np.float32).astype(np.float64), R.valid, R.sentinel)
        demo[f"terrain32_{k}"] = sha(q.terrain)
        demo[f"water32_{k}"] = sha(q.water)
        r32.append(q)
    lays = fr.debug["layouts"]
    mips = {layer: [ref.build_max_mipmap(r, layer) for r in r32] for layer in ("terrain", "water")}
    origin = np.asarray(cfg.camera.eye, dtype=np.float64)
    dirs = ref.render.camera_ray_dirs(cfg.camera, cfg.width, cfg.height).reshape(-1, 3)
    demo["dirs_sha"] = sha(dirs)
    res = {}
    for layer in ("terrain", "water"):
        lr = ref.render._resolve_layer(origin, dirs, r32, mips[layer], lays)
        res[layer] = lr
        for name in ("hit", "t", "near", "far", "w"):
            demo[f"{layer}_{name}"] = sha(getattr(lr, name))
        for k, raw in lr.raw.items():
            for name, arr in zip(("hit", "t", "ix", "iy", "u", "v"), raw):
                demo[f"{layer}_raw{k}_{name}"] = sha(arr)
        for k, m in enumerate(mips[layer]):
            demo[f"{layer}_mip{k}"] = sha(m._flat)
    tsh = ref.render._shade_terrain(res["terrain"], r32, g, origin, dirs)
    wsh, wdep = ref.render._shade_water(res["water"], r32, cfg, origin, dirs)
    px = np.empty((cfg.height * cfg.width, 3), dtype=np.uint8)
    px[:] = np.array(cfg.background, dtype=np.uint8)
    use_w = res["water"].hit & (res["water"].t < res["terrain"].t)
    use_t = res["terrain"].hit & ~use_w
    px[use_t] = tsh[use_t]
    px[use_w] = wsh[use_w]
    demo["pixels32_sha"] = sha(px.reshape(cfg.height, cfg.width, 3))
    demo["water_depth32_sha"] = sha(wdep)
    out["demo"] = demo
    np.savez_compressed(os.path.join(HERE, "demo_frame.npz"), pixels32=px.reshape(cfg.height, cfg.width, 3),
                        pixels=fr.pixels, **samples)

    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()

"""Pin the CPU oracle and the host planner against fixtures produced by the reference.

tests/golden/make_golden.py ran the reference (pkg/src/heightcast) on the inputs
of tests/golden_inputs.py; these CPU tests check that
  * this package's synthetic grids / influence tables are the reference's arrays,
  * the host cascade planner reproduces the reference's layouts bit for bit,
  * the oracle (oracle/hc_oracle.c) reproduces the reference's masks, mip
    pyramids, traversal outputs, resolve, shading and pixels bit for bit, and its
    float64 Eq. 2 within 1e-12 relative (numpy's exp / reduceat order differ).
Only after these pass is the oracle trusted as the GPU checker.
"""

import math

import numpy as np
import pytest

import golden_inputs as gi
from helpers import F64Raster, demo_setup, golden, npz, sha, unhex

from paper_2201_10887_b200 import cascade, grid as G, synth
from paper_2201_10887_b200.raycast import intersect_bilinear_patch
from paper_2201_10887_b200.rbf import RbfParams, weight
from paper_2201_10887_b200.render import depth_colormap

GOLD = golden()


def oracle_table(g, sigma):
    import heightcast_oracle as O
    return O.build_influence_table(g, sigma)


@pytest.mark.parametrize("spec", gi.GRID_SPECS, ids=lambda s: s["name"])
def test_synthetic_grid_and_table_match_reference(spec):
    g = synth.generate_synthetic(spec["kind"], spec["seed"], spec["cells"], max_depth=spec["max_depth"])
    d = GOLD["grids"][spec["name"]]
    assert g.n_cells == d["n_cells"]
    assert sha(g.centers) == d["centers"] and sha(g.sizes) == d["sizes"]
    assert sha(g.terrain) == d["terrain"] and sha(g.water_depth) == d["water_depth"]
    assert sha(g.tile_index) == d["tile_index"]
    assert [unhex(v) for v in d["height_range"]] == list(g.height_range)
    for sigma in spec["sigmas"]:
        t = oracle_table(g, sigma)
        assert sha(t.offsets) == d[f"table_{sigma}"]["offsets"]
        assert sha(t.indices) == d[f"table_{sigma}"]["indices"]


def test_spec_known_answers(oracle):
    k = GOLD["known"]
    P = RbfParams(sigma=1.0)
    assert weight((0.0, 0.0), 1.0, (0.0, 0.0), P) == unhex(k["weight_0"])
    assert abs(weight((0, 0), 1.0, (0, 0), P) - 0.9978125088818172) < 1e-15
    assert weight((0.0, 0.0), 2.0, (7.0, 0.0), P) == unhex(k["weight_trunc"]) == 0.0
    assert weight((0.0, 0.0), 1.0, (10.0, 0.0), P) == unhex(k["weight_far"]) == 0.0
    assert weight((0.0, 0.0), 2.0, (0.999 * 7.0, 0.0), P) > 0.0
    assert cascade.split_depths(1.0, 8.0) == tuple(unhex(v) for v in k["split_1_8"]) == (2.0, 4.0)
    assert cascade.split_depths(10.0, 1000.0) == tuple(unhex(v) for v in k["split_10_1000"])
    t, uv = intersect_bilinear_patch((0.5, 0.5, 10.0), (0.0, 0.0, -1.0), (7.0,) * 4, (0.0, 0.0), 1.0)
    assert (t, uv[0], uv[1]) == tuple(unhex(v) for v in k["patch_flat"]) == (3.0, 0.5, 0.5)
    got = [list(depth_colormap(v, (0.0, 4.0))) for v in (0.0, 2.0, 4.0, float("nan"))]
    assert got == k["colormap"]
    assert got[:3] == [[0, 0, 128], [0, 180, 220], [240, 248, 255]]
    poly = cascade.CascadePolygon(np.array([[0.0, 0.0], [4.1, 0.0], [4.1, 3.0], [0.0, 3.0]]), 0.0, 1.0,
                                  cascade.ViewAxis((0.0, 0.0), (1.0, 0.0)))
    lay = cascade.fit_layout(poly, 64, 2.0)
    lo, hi = lay.widened_box()
    f = k["fit_4.1x3"]
    assert [unhex(v) for v in f["box"]] == list(hi - lo) == [8.0, 4.0]
    assert [unhex(v) for v in f["origin"]] == list(lay.world_origin)
    assert unhex(f["texel"]) == lay.texel_size


def test_k_split_generalisation():
    for n, f in ((1.0, 8.0), (10.0, 1000.0), (0.37, 5123.0)):
        assert cascade.split_depths_k(n, f, 3) == list(cascade.split_depths(n, f))
        for K in (1, 2, 4, 8):
            d = cascade.split_depths_k(n, f, K)
            chain = [n] + d + [f]
            assert len(d) == K - 1 and all(a < b for a, b in zip(chain, chain[1:]))


def _plan_grid(name):
    a = gi.PLAN_GRIDS[name]
    return synth.generate_synthetic(a["kind"], a["seed"], a["cells"], max_depth=a.get("max_depth"))


@pytest.mark.parametrize("gname", list(gi.PLAN_GRIDS))
def test_planner_matches_reference(gname, oracle):
    g = _plan_grid(gname)
    poses = {p["id"]: p for p in gi.plan_poses(gname)}
    recs = [r for r in GOLD["plans"] if r["grid"] == gname]
    assert len(recs) == len(poses)
    n_vis = 0
    for rec in recs:
        pose = poses[rec["pose"]]
        cam = cascade.CameraView(**pose["camera"])
        if rec.get("nothing_visible"):
            with pytest.raises(cascade.NothingVisibleError):
                cascade.plan_cascades(cam, g, pose["res"], pose["overlap"])
            continue
        n_vis += 1
        hull, polys, lays = cascade.plan_cascades(cam, g, pose["res"], pose["overlap"])
        assert sha(hull) == rec["hull"]
        assert len(lays) == len(rec["cascades"])
        for L, want in zip(lays, rec["cascades"]):
            assert (L is None) == (want is None)
            if L is None:
                continue
            assert [unhex(v) for v in want["origin"]] == list(L.world_origin)
            assert unhex(want["texel"]) == L.texel_size and want["res"] == L.resolution
            assert sha(L.polygon.vertices) == want["verts"]
            assert unhex(want["near"]) == L.polygon.near_offset
            assert unhex(want["far"]) == L.polygon.far_offset
            assert list(L.box_texel) == want["box_texel"] and list(L.box_steps) == want["box_steps"]
            assert L.index == want["index"]
            mask, _ = oracle.visibility_cells(L, g)
            assert int(mask.sum()) == want["mask_sum"]
            assert sha(mask) == want["mask"]
    assert n_vis >= 20


def test_oracle_traversal_matches_reference_kernel(oracle):
    """SPEC acceptance: >= 1e4 rays over >= 20 rasters, identical to the reference kernel."""
    data = npz("traverse_rays.npz")
    n_rays = 0
    for case in gi.traversal_cases():
        name = case["name"]
        h, valid = case["heights"], case["valid"]
        mip = oracle.maxmip(h)
        assert sha(mip.flat) == GOLD["traverse_mip_sha"][name]
        vr = data[f"{name}__vrange"]
        out = oracle.traverse_batch(h, valid, mip, *case["rays"], vr[0], vr[1])
        for key, got in zip(("hit", "t", "ix", "iy", "u", "v"), out):
            want = data[f"{name}__{key}"]
            assert np.array_equal(got, want), (name, key, int((got != want).sum()))
        n_rays += len(out[0])
    assert n_rays >= 10_000


def _dda_agreement(got, want, case):
    """same hit/miss verdict, t within 1e-9, hit residual < 1e-6 m (and the
    same patch) between a traversal result and the brute-force DDA walk."""
    hit_g, t_g, ix_g, iy_g, u_g, v_g = (np.asarray(a) for a in got[:6])
    hit_w, t_w, ix_w, iy_w = want[:4]
    assert np.array_equal(hit_g.astype(bool), hit_w.astype(bool)), case["name"]
    m = hit_w.astype(bool)
    assert np.array_equal(ix_g[m], ix_w[m]) and np.array_equal(iy_g[m], iy_w[m]), case["name"]
    assert np.all(np.abs(t_g[m] - t_w[m]) <= 1e-9 * np.maximum(1.0, np.abs(t_w[m]))), case["name"]
    rx, ry, rz, dx, dy, dz = (np.broadcast_to(np.asarray(a, dtype=np.float64), hit_w.shape) for a in case["rays"])
    h = np.asarray(case["heights"], dtype=np.float64)
    ix, iy, u, v = ix_g[m], iy_g[m], u_g[m], v_g[m]
    surf = ((h[iy, ix] * (1 - u) + h[iy, ix + 1] * u) * (1 - v) + (h[iy + 1, ix] * (1 - u) + h[iy + 1, ix + 1] * u) * v)
    resid = np.abs(rz[m] + t_g[m] * dz[m] - surf)
    assert np.all(resid < 1e-6), (case["name"], float(resid.max()) if resid.size else 0.0)
    return int(m.sum())


def test_oracle_traversal_equals_dda_walk(oracle):
    """SPEC.md:473 [PRIMARY]: the max-mip traversal equals brute-force sequential patch
    testing along the ray's DDA cell walk on >= 1e4 random rays over >= 20 rasters."""
    n_rays = n_hits = 0
    for case in gi.traversal_cases():
        h, valid = case["heights"], case["valid"]
        vals = h[valid.astype(bool)]
        lo, hi = float(vals.min()), float(vals.max())
        mip = oracle.maxmip(h)
        got = oracle.traverse_batch(h, valid, mip, *case["rays"], lo, hi)
        want = oracle.dda_batch(h, valid, *case["rays"], lo, hi)
        n_hits += _dda_agreement(got, want, case)
        n_rays += len(got[0])
    assert n_rays >= 10_000 and n_hits >= 1000


def test_oracle_eq2_matches_reference(oracle):
    data = npz("rbf_points.npz")
    worst = 0.0
    for case in gi.rbf_cases():
        g = synth.generate_synthetic(case["kind"], case["seed"], case["cells"], max_depth=case["max_depth"])
        t = oracle_table(g, case["sigma"])
        pts = gi.rbf_points(g.domain, case["seed"], case["n_points"])
        ter, wat, ws, cnt = oracle.eval_points(pts, g.cells_at(pts), g, t, case["sigma"])
        want = data[case["name"]]
        rel = np.abs(np.stack([ter, wat, ws]) - want[:, :3].T) / np.abs(want[:, :3].T)
        worst = max(worst, float(rel.max()))
        assert np.array_equal(cnt, want[:, 3].astype(np.int64))
    assert worst <= 1e-12, worst


def test_oracle_demo_frame_matches_reference(oracle):
    """Demo scene: rasters to 1e-12; mips, rays, resolve, shading and pixels bit-exact
    on the float32-rounded rasters the GPU path stores."""
    sc, g, t, cfg, st = demo_setup()
    D = GOLD["demo"]
    samples = npz("demo_frame.npz")
    _, _, lays = cascade.plan_cascades(cfg.camera, g, st.resolution, st.overlap, st.count)
    lays = [L for L in lays if L is not None]
    r32 = []
    for k, L in enumerate(lays):
        r = oracle.discretize(L, g, t, sc.sigma)
        assert sha(r.valid) == D[f"valid_{k}"]
        iy, ix = samples[f"idx_{k}"].T
        for layer in ("terrain", "water"):
            got = r.layer(layer)[iy, ix]
            want = samples[f"{layer}_{k}"]
            assert np.max(np.abs(got - want) / np.abs(want)) <= 1e-12
        q = F64Raster(r.terrain.astype(np.float32), r.water.astype(np.float32), r.valid)
        assert sha(q.terrain) == D[f"terrain32_{k}"] and sha(q.water) == D[f"water32_{k}"]
        r32.append(q)
    px, dbg = oracle.raycast(cfg.camera, cfg.width, cfg.height, lays, r32, g.height_range,
                             cfg.colormap_range, cfg.background)
    assert sha(dbg["dirs"]) == D["dirs_sha"]
    for layer in ("terrain", "water"):
        lr = dbg[layer]
        assert sha(lr.hit.astype(bool)) == D[f"{layer}_hit"]
        assert sha(lr.t) == D[f"{layer}_t"]
        assert sha(lr.near) == D[f"{layer}_near"] and sha(lr.far) == D[f"{layer}_far"]
        assert sha(lr.w) == D[f"{layer}_w"]
        for k, raw in lr.raw.items():
            for name, arr in zip(("hit", "t", "ix", "iy", "u", "v"), raw):
                assert sha(arr) == D[f"{layer}_raw{k}_{name}"], (layer, k, name)
        for k, r in enumerate(r32):
            assert sha(oracle.maxmip(r.layer(layer)).flat) == D[f"{layer}_mip{k}"]
    assert sha(dbg["water_depth"]) == D["water_depth32_sha"]
    assert sha(px) == D["pixels32_sha"]
    assert np.array_equal(px, samples["pixels32"])
    # and the oracle's own float64 frame equals the reference's frame
    px64, st64 = oracle.render_frame(cfg, g, t, RbfParams(sigma=sc.sigma), st)
    assert sha(px64) == D["pixels_sha"]
    assert st64["visible_texels"] == D["visible_texels"] and st64["rays_hit"] == D["rays_hit"]

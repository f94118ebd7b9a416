"""GPU parity: the sm_100a path (through the C ABI) against the pinned oracle.

Bit-exact: visibility masks, valid bits, max pyramids, valid ranges, ray
directions, traversal (hit, t, patch, uv), layer resolve (hit, t, near, far,
blend w), shading and pixels -- on identical (float32) rasters.
Tolerance: discretized heights vs the float64 oracle,
  |h_gpu - h_ref| <= HEIGHT_ABS + HEIGHT_REL * |h_ref|   (float32 Eq. 1/2).
"""

import numpy as np
import pytest

import golden_inputs as gi
from helpers import F64Raster, demo_setup, golden, npz, sha

pytestmark = pytest.mark.gpu

HEIGHT_ABS = 2e-4   # metres
HEIGHT_REL = 2e-6

GOLD = golden()


def _np(t):
    return t.detach().cpu().numpy()


def test_traverse_batch_matches_reference_kernel(cuda):
    """hc_traverse_batch (drop-in for _kernels.traverse_batch) on the golden rays."""
    import torch
    from paper_2201_10887_b200 import raycast
    from paper_2201_10887_b200.discretize import CascadeRaster
    data = npz("traverse_rays.npz")
    total = 0
    for case in gi.traversal_cases():
        name = case["name"]
        h = torch.from_numpy(case["heights"].astype(np.float32)).to(cuda)
        v = torch.from_numpy(case["valid"]).to(cuda)
        ras = CascadeRaster(None, h, h, v, float(case["heights"].min()) - 1.0)
        mip = raycast.build_max_mipmap(ras, "terrain")
        assert sha(_np(mip._flat).astype(np.float64)) == GOLD["traverse_mip_sha"][name]
        vr = data[f"{name}__vrange"]
        assert mip.valid_range() == (vr[0], vr[1])
        out = raycast.traverse_batch(h, v, mip, *case["rays"], vr[0], vr[1])
        for key, got in zip(("hit", "t", "ix", "iy", "u", "v"), out):
            want = data[f"{name}__{key}"]
            g = _np(got)
            assert np.array_equal(g, want), (name, key, int((g != want).sum()))
        total += len(case["rays"][3])
    assert total >= 10_000


def test_traverse_batch_equals_dda_walk(cuda, oracle):
    """SPEC.md:473 [PRIMARY] on the GPU: hc_traverse_batch (max-mip walk) against the
    brute-force DDA patch walk on >= 1e4 random rays over >= 20 rasters: same verdict
    and patch, t within 1e-9, hit residual < 1e-6 m."""
    import torch
    from test_oracle_golden import _dda_agreement
    from paper_2201_10887_b200 import raycast
    from paper_2201_10887_b200.discretize import CascadeRaster
    n_rays = n_hits = 0
    for case in gi.traversal_cases():
        hf = case["heights"].astype(np.float32)
        case = dict(case, heights=hf.astype(np.float64))         # the GPU walks float32 heights
        h = torch.from_numpy(hf).to(cuda)
        v = torch.from_numpy(case["valid"]).to(cuda)
        ras = CascadeRaster(None, h, h, v, float(hf.min()) - 1.0)
        mip = raycast.build_max_mipmap(ras, "terrain")
        lo, hi = mip.valid_range()
        got = [_np(o) for o in raycast.traverse_batch(h, v, mip, *case["rays"], lo, hi)]
        want = oracle.dda_batch(case["heights"], case["valid"], *case["rays"], lo, hi)
        n_hits += _dda_agreement(got, want, case)
        n_rays += len(got[0])
    assert n_rays >= 10_000 and n_hits >= 1000


def test_visibility_masks_match_reference(cuda, oracle):
    from paper_2201_10887_b200 import cascade, synth
    from paper_2201_10887_b200.discretize import compute_visibility_mask
    for gname, a in gi.PLAN_GRIDS.items():
        g = synth.generate_synthetic(a["kind"], a["seed"], a["cells"])
        recs = {r["pose"]: r for r in GOLD["plans"] if r["grid"] == gname}
        for pose in gi.plan_poses(gname):
            rec = recs[pose["id"]]
            if rec.get("nothing_visible"):
                continue
            _, _, lays = cascade.plan_cascades(cascade.CameraView(**pose["camera"]), g, pose["res"],
                                               pose["overlap"])
            for L, want in zip(lays, rec["cascades"]):
                if L is None:
                    continue
                m = _np(compute_visibility_mask(L))
                assert sha(m) == want["mask"], (gname, pose["id"])


def _check_heights(gpu, ref, valid, what):
    d = np.abs(gpu.astype(np.float64) - ref)[valid]
    bound = (HEIGHT_ABS + HEIGHT_REL * np.abs(ref))[valid]
    assert np.all(d <= bound), (what, float(d.max()), int((d > bound).sum()))
    return float(d.max()) if d.size else 0.0


def test_discretize_demo_matches_oracle(cuda, oracle):
    from paper_2201_10887_b200 import cascade, discretize_cascade
    from paper_2201_10887_b200.rbf import RbfParams
    sc, g, t, cfg, st = demo_setup()
    _, _, lays = cascade.plan_cascades(cfg.camera, g, st.resolution, st.overlap, st.count)
    for k, L in enumerate(l for l in lays if l is not None):
        r = discretize_cascade(L, g, t, RbfParams(sigma=sc.sigma))
        o = oracle.discretize(L, g, t, sc.sigma)
        valid = _np(r.valid)
        assert sha(valid) == GOLD["demo"][f"valid_{k}"]
        assert np.array_equal(_np(L.mask), o.mask)
        _check_heights(_np(r.terrain), o.terrain, valid, "terrain")
        _check_heights(_np(r.water), o.water, valid, "water")
        assert np.all(_np(r.terrain)[~valid] == np.float32(g.height_range[0] - 1.0))
        assert np.all(_np(r.water) >= _np(r.terrain))


def test_discretize_non_power_of_two_min_cell(cuda, oracle):
    """min_cell = 3 x the demo's: the cell lookup takes the IEEE-division path."""
    import dataclasses
    from paper_2201_10887_b200 import AdaptiveGrid, cascade, discretize_cascade
    from paper_2201_10887_b200.cascade import CameraView
    from paper_2201_10887_b200.grid import Rect
    from paper_2201_10887_b200.rbf import RbfParams
    import heightcast_oracle as O
    sc, g0, _, cfg, st = demo_setup()
    d = g0.domain
    g = AdaptiveGrid(Rect(3 * d.xmin, 3 * d.ymin, 3 * d.xmax, 3 * d.ymax), 3 * g0.min_cell_size,
                     3 * g0.centers, 3 * g0.sizes, g0.terrain, g0.water_depth)
    t = O.build_influence_table(g, sc.sigma)
    c = cfg.camera
    cam = dataclasses.replace(c, eye=(3 * c.eye[0], 3 * c.eye[1], c.eye[2]),
                              look_dir=(3 * c.look_dir[0], 3 * c.look_dir[1], c.look_dir[2]))
    assert isinstance(cam, CameraView)
    _, _, lays = cascade.plan_cascades(cam, g, st.resolution, st.overlap, st.count)
    n = 0
    for L in (l for l in lays if l is not None):
        r = discretize_cascade(L, g, t, RbfParams(sigma=sc.sigma))
        o = oracle.discretize(L, g, t, sc.sigma)
        valid = _np(r.valid)
        assert np.array_equal(valid, o.valid)
        _check_heights(_np(r.terrain), o.terrain, valid, "terrain")
        _check_heights(_np(r.water), o.water, valid, "water")
        n += int(valid.sum())
    assert n > 0


def _frame_vs_oracle(frame, oracle, cfg, g):
    """Feed the oracle the GPU's own rasters; every raycast output must match bitwise."""
    dbg = frame.debug
    lays = [L for L in dbg["layouts"] if L is not None]
    r64 = [F64Raster(_np(r.terrain), _np(r.water), _np(r.valid)) for r in dbg["rasters"] if r is not None]
    px, od = oracle.raycast(cfg.camera, cfg.width, cfg.height, lays, r64, g.height_range,
                            cfg.colormap_range, cfg.background)
    assert np.array_equal(_np(dbg["dirs"]), od["dirs"])
    for layer in ("terrain", "water"):
        G, O = dbg[layer], od[layer]
        hit = _np(G.hit)
        assert np.array_equal(hit, O.hit.astype(bool)), layer
        assert np.array_equal(_np(G.near), O.near) and np.array_equal(_np(G.far), O.far), layer
        assert np.array_equal(_np(G.t), O.t), layer
        assert np.array_equal(_np(G.w), O.w), layer
        for s, kk in ((0, O.near), (1, O.far)):
            sel = kk >= 0
            for j, name in ((1, "t"), (2, "ix"), (3, "iy"), (4, "u"), (5, "v")):
                want = np.zeros_like(_np(G.raw_slots[name][s]))
                for k in range(len(lays)):
                    m = sel & (kk == k)
                    want[m] = O.raw[k][j][m]
                got = _np(G.raw_slots[name][s])
                assert np.array_equal(got[sel], want[sel]), (layer, s, name)
    wd = _np(dbg["water_depth"])
    assert np.array_equal(np.isnan(wd), np.isnan(od["water_depth"]))
    assert np.array_equal(wd[~np.isnan(wd)], od["water_depth"][~np.isnan(wd)])
    assert np.array_equal(frame.pixels, px)
    # the frame's max mips (built per cascade as (terrain, water) pairs) and valid ranges
    from paper_2201_10887_b200._engine import key_to_float
    keys = _np(dbg["vrange_keys"])
    for k, r in enumerate(r64):
        for li, (layer, h) in enumerate((("terrain", r.terrain), ("water", r.water))):
            m = oracle.maxmip(h)
            assert np.array_equal(_np(dbg["mips"][layer][k]).astype(np.float64)[:m.flat.size], m.flat), (k, layer)
            vals = h[r.valid]
            if vals.size:
                lo, hi = key_to_float(keys[k, li, 0]), key_to_float(keys[k, li, 1])
                assert (lo, hi) == (float(vals.min()), float(vals.max())), (k, layer)
    return px


def test_render_frame_demo_bit_exact_on_gpu_rasters(cuda, oracle):
    from paper_2201_10887_b200 import render_frame
    from paper_2201_10887_b200.rbf import RbfParams
    sc, g, t, cfg, st = demo_setup()
    fr = render_frame(cfg, g, t, RbfParams(sigma=sc.sigma), st, debug=True)
    _frame_vs_oracle(fr, oracle, cfg, g)
    assert fr.visible_texels == GOLD["demo"]["visible_texels"]
    # end to end against the reference's own frame: only float32-height effects allowed
    want = npz("demo_frame.npz")["pixels"]
    diff = np.any(fr.pixels != want, axis=2)
    assert diff.mean() < 0.002, int(diff.sum())


def test_render_frame_is_deterministic(cuda):
    from paper_2201_10887_b200 import render_frame
    from paper_2201_10887_b200.rbf import RbfParams
    sc, g, t, cfg, st = demo_setup()
    a = render_frame(cfg, g, t, RbfParams(sigma=sc.sigma), st)
    b = render_frame(cfg, g, t, RbfParams(sigma=sc.sigma), st)
    assert np.array_equal(a.pixels, b.pixels) and a.rays_hit == b.rays_hit


def test_approximate_fp64_matches_reference(cuda):
    from paper_2201_10887_b200 import approximate, build_influence_table, synth
    from paper_2201_10887_b200.rbf import RbfParams
    data = npz("rbf_points.npz")
    for case in gi.rbf_cases()[:6]:
        g = synth.generate_synthetic(case["kind"], case["seed"], case["cells"], max_depth=case["max_depth"])
        t = build_influence_table(g, case["sigma"])
        P = RbfParams(sigma=case["sigma"])
        want = data[case["name"]]
        for p, w in zip(gi.rbf_points(g.domain, case["seed"], case["n_points"])[:25], want[:25]):
            s = approximate(p, "terrain", g, t, P)
            assert abs(s.value - w[0]) <= 1e-12 * abs(w[0])
            assert abs(approximate(p, "water", g, t, P).value - w[1]) <= 1e-12 * abs(w[1])
            assert s.influencer_count == int(w[3])


_GRIDS: dict = {}


def _config_inputs(name, width=None, height=None, view=0):
    from paper_2201_10887_b200 import build_influence_table
    from paper_2201_10887_b200.configs import CONFIGS
    from paper_2201_10887_b200.render import FrameConfig
    cfg = CONFIGS[name]
    key = (cfg.kind, cfg.seed, cfg.cells, cfg.max_depth, cfg.sigma)
    if key not in _GRIDS:                  # C3 and C4 share their grid
        g = cfg.grid()
        _GRIDS.clear()
        _GRIDS[key] = (g, build_influence_table(g, cfg.sigma))
    g, t = _GRIDS[key]
    fc = cfg.frame_config(view)
    if width:
        fc = FrameConfig(width=width, height=height, camera=fc.camera)
    return cfg, g, t, fc


# End-to-end against the float64 pipeline (SURVEY.md §8 c): the GPU frame (float32
# Eq. 1/2 rasters) against the oracle frame cast through the oracle's own float64
# rasters.  Only float32 height rounding separates the two, so hits can flip only
# where a ray grazes the surface within ~1e-5 m.  Bounds (per layer, all configs):
E2E_HIT_FLIP = 1e-4        # fraction of rays whose hit/miss differs (measured: 0 on every config)
E2E_PATCH_MISMATCH = 5e-5  # fraction of common hits on a different cascade or patch (measured <= 6.8e-6)
E2E_DT_P99 = 1e-6          # p99 of |dt| / t over common hits on the same patch (measured <= 3.1e-8)
E2E_PIXEL_MISMATCH = 5e-4  # fraction of pixels whose RGB differs at all (measured <= 1.0e-4)
E2E_PIXEL_LSB = 1          # max RGB difference on pixels whose hits, patches and shown layer agree


def _e2e_vs_float64(frame, oracle, fc, g, lays, rasters64):
    """Statistics of the GPU frame against the oracle's float64 frame (same plan)."""
    px, od = oracle.raycast(fc.camera, fc.width, fc.height, lays, rasters64, g.height_range,
                            fc.colormap_range, fc.background)
    dbg = frame.debug
    n = fc.width * fc.height
    stats = {"rays": n}
    agree_all = np.ones(n, dtype=bool)
    for layer in ("terrain", "water"):
        G, O = dbg[layer], od[layer]
        gh, oh = _np(G.hit).astype(bool), O.hit.astype(bool)
        gnear = _np(G.near)
        gix, giy = _np(G.raw_slots["ix"][0]), _np(G.raw_slots["iy"][0])
        oix = np.full(n, -1, np.int64)
        oiy = np.full(n, -1, np.int64)
        for k in range(len(lays)):
            m = oh & (O.near == k)
            oix[m] = O.raw[k][2][m]
            oiy[m] = O.raw[k][3][m]
        both = gh & oh
        same = both & (gnear == O.near) & (gix == oix) & (giy == oiy) & (_np(G.far) == O.far)
        gt, ot = _np(G.t), O.t
        rel = np.abs(gt[same] - ot[same]) / np.maximum(np.abs(ot[same]), 1e-300)
        stats[layer] = {
            "hits": int(oh.sum()), "hit_flips": int((gh != oh).sum()),
            "hit_flip_rate": float((gh != oh).mean()),
            "patch_mismatch": int(both.sum() - same.sum()),
            "patch_mismatch_rate": float((both.sum() - same.sum()) / max(both.sum(), 1)),
            "dt_rel_p99": float(np.quantile(rel, 0.99)) if rel.size else 0.0,
            "dt_rel_max": float(rel.max()) if rel.size else 0.0,
        }
        agree_all &= (gh == oh) & (~both | same)
    # which layer colours the pixel (render.py:253-256): water iff it hits nearer than the
    # terrain.  Where float64 water lies a hair above the terrain but float32 rounds the
    # depth away (or the reverse), the two frames pick different layers.
    def water_shown(G_or_O_w, G_or_O_t, gpu):
        wh = (_np(G_or_O_w.hit) if gpu else G_or_O_w.hit).astype(bool)
        wt = _np(G_or_O_w.t) if gpu else G_or_O_w.t
        tt = _np(G_or_O_t.t) if gpu else G_or_O_t.t
        th = (_np(G_or_O_t.hit) if gpu else G_or_O_t.hit).astype(bool)
        return wh & (~th | (wt < tt))
    sel_g = water_shown(dbg["water"], dbg["terrain"], True)
    sel_o = water_shown(od["water"], od["terrain"], False)
    stats["layer_select_flips"] = int((sel_g != sel_o).sum())
    agree_all &= sel_g == sel_o
    diff = np.abs(frame.pixels.astype(np.int16) - px.astype(np.int16)).max(axis=2).reshape(-1)
    stats["pixel_mismatch"] = int((diff > 0).sum())
    stats["pixel_mismatch_rate"] = float((diff > 0).mean())
    stats["pixel_lsb_max_where_agree"] = int(diff[agree_all].max()) if agree_all.any() else 0
    for layer in ("terrain", "water"):
        s = stats[layer]
        assert s["hit_flip_rate"] <= E2E_HIT_FLIP, (layer, s)
        assert s["patch_mismatch_rate"] <= E2E_PATCH_MISMATCH, (layer, s)
        assert s["dt_rel_p99"] <= E2E_DT_P99, (layer, s)
    assert stats["pixel_mismatch_rate"] <= E2E_PIXEL_MISMATCH, stats
    assert stats["pixel_lsb_max_where_agree"] <= E2E_PIXEL_LSB, stats
    return stats


def _record_stats(key, stats):
    import json
    import os
    print(key, json.dumps(stats))
    d = os.environ.get("HC_STATS_DIR")
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, "e2e_float64_stats.jsonl"), "a") as fh:
            fh.write(json.dumps({"case": key, **stats}) + "\n")


@pytest.mark.parametrize("name,view", [
    ("C1", 0), ("C2", 0), ("C2", 30), ("C3", 0), ("C4", 0), ("C4", 16), ("C4", 32), ("C4", 48), ("C5", 0),
])
def test_benchmark_config_frame_parity(cuda, oracle, name, view):
    """The five BASELINE configs at full size (C2: two poses of the bench camera path;
    C4: four orbit views of 64): rays/traversal/resolve/shading bit-exact on the GPU's
    rasters, masks and valid bits exact, heights within the float32 tolerance of the
    float64 oracle, and the end-to-end frame against the oracle's float64 frame within
    the E2E_* bounds (rates recorded under $HC_STATS_DIR)."""
    from paper_2201_10887_b200 import render_frame
    from paper_2201_10887_b200.rbf import RbfParams
    cfg, g, t, fc = _config_inputs(name, view=view)
    if name == "C2" and view:
        fc = cfg.path_frame_config(view)
    fr = render_frame(fc, g, t, RbfParams(sigma=cfg.sigma), cfg.settings(), debug=True)
    assert fr.visible
    _frame_vs_oracle(fr, oracle, fc, g)
    # the production launch (launch list: only blocks that may see the mask polygon get
    # a discretize CTA) renders the same frame as the debug launch (every block)
    prod = render_frame(fc, g, t, RbfParams(sigma=cfg.sigma), cfg.settings())
    assert np.array_equal(prod.pixels, fr.pixels)
    assert (prod.visible_texels, prod.valid_texels, prod.rays_hit, prod.work) == \
        (fr.visible_texels, fr.valid_texels, fr.rays_hit, fr.work)
    lays = [L for L in fr.debug["layouts"] if L is not None]
    assert len(lays) == cfg.cascades
    worst = 0.0
    r64 = []
    for L, r in zip(lays, fr.debug["rasters"]):
        o = oracle.discretize(L, g, t, cfg.sigma)
        r64.append(o)
        valid = _np(r.valid)
        assert np.array_equal(valid, o.valid) and np.array_equal(_np(L.mask), o.mask)
        for layer in ("terrain", "water"):
            worst = max(worst, _check_heights(_np(r.layer(layer)), o.layer(layer), valid, f"{name} {layer}"))
    stats = _e2e_vs_float64(fr, oracle, fc, g, lays, r64)
    stats["max_abs_dh"] = worst
    _record_stats(f"{name} view {view}", stats)
    if name == "C5":
        # sharded screen strips (2 and 8 ranks emulated on this GPU: footprint
        # discretization, MAX-reduced mip exchange) reproduce the full frame bit for bit
        from paper_2201_10887_b200 import _cuda, multi
        total_pairs = fr.work["pairs"]
        for world in (2, 8):
            img, cnt = multi.render_strips_one_gpu(fc, g, t, RbfParams(sigma=cfg.sigma), cfg.settings(), world)
            assert np.array_equal(img, fr.pixels), world
            pairs = [int(c[_cuda.CNT_PAIRS]) for c in cnt]
            print(f"C5 x{world}: per-rank pairs / full = {[round(p / total_pairs, 3) for p in pairs]}")
            assert max(pairs) < total_pairs and sum(pairs) >= total_pairs


def test_patch_early_rejection_selftest(cuda):
    """The ray/patch test with its exact early rejections equals the reference's
    sequence bit for bit on 2^26 generated cases (roots at the segment ends,
    near-tangent rays, rays starting under the patch)."""
    import torch
    from paper_2201_10887_b200 import _cuda
    cnt = torch.zeros(3, dtype=torch.int64, device=cuda)
    _cuda.check(_cuda.lib().hc_selftest_patch(1 << 26, 77, cnt.data_ptr(), _cuda.stream_ptr()), "selftest")
    bad, hits, below = (int(x) for x in cnt.tolist())
    print(f"patch selftest: {bad} mismatches, {hits} hits, {below} misses from below")
    assert hits > 1000 and below > 1000
    assert bad == 0


def test_slab_pretest_selftest(cuda):
    """The render's certified slab pre-test never calls a slab empty that the exact
    setup (traverse_raster's divisions) does not miss, on 2^26 generated cases --
    half of them aimed within ulps of a slab corner or edge, with zero and tiny
    direction components -- and it catches most exact misses."""
    import torch
    from paper_2201_10887_b200 import _cuda
    cnt = torch.zeros(3, dtype=torch.int64, device=cuda)
    _cuda.check(_cuda.lib().hc_selftest_slab(1 << 26, 91, cnt.data_ptr(), _cuda.stream_ptr()), "selftest")
    bad, pre, exact = (int(x) for x in cnt.tolist())
    print(f"slab selftest: {bad} false empties, {pre} pre-test empties of {exact} exact misses")
    assert bad == 0
    assert exact > 1000 and pre > 0.5 * exact


def _random_poses():
    """Camera poses over the C2 grid (domain [0, 2048]^2, heights ~12-100 m) that
    stress the traversal's exact shortcuts: axis-aligned and integer-coordinate
    eyes (rays through node corners, dx = 0 / dy = 0 columns), a horizontal view
    axis (dz = 0 rows), grazing eyes just above the terrain, an eye below the
    terrain, eyes outside the domain, plus seeded random poses."""
    rng = np.random.default_rng(2201)
    poses = [
        ((1024.0, 1024.0, 400.0), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), 50.0),     # straight down
        ((512.0, 512.0, 60.0), (1.0, 0.0, 0.0), (0.0, 0.0, 1.0), 60.0),         # horizontal, +x
        ((1500.0, 300.0, 45.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0), 70.0),        # horizontal, +y
        ((256.0, 256.0, 150.0), (1.0, 1.0, -0.25), (0.0, 0.0, 1.0), 55.0),      # diagonal through corners
        ((-200.0, 1024.0, 90.0), (1.0, 0.0, -0.05), (0.0, 0.0, 1.0), 40.0),     # outside, grazing in
        ((1024.0, 1024.0, 20.0), (0.3, -1.0, 0.0), (0.0, 0.0, 1.0), 80.0),      # low, near the terrain
        ((900.0, 1100.0, 5.0), (1.0, 0.2, 0.1), (0.0, 0.0, 1.0), 60.0),         # below most of the terrain
        ((2300.0, 2300.0, 800.0), (-1.0, -1.0, -0.8), (0.0, 0.0, 1.0), 35.0),   # far outside, high
    ]
    for _ in range(8):
        eye = (float(rng.uniform(-300, 2350)), float(rng.uniform(-300, 2350)), float(rng.uniform(15, 600)))
        tgt = (float(rng.uniform(200, 1850)), float(rng.uniform(200, 1850)), float(rng.uniform(0, 80)))
        look = tuple(b - a for a, b in zip(eye, tgt))
        poses.append((eye, look, (0.0, 0.0, 1.0), float(rng.uniform(30, 90))))
    return poses


@pytest.mark.parametrize("i", range(16))
def test_random_pose_frame_parity(cuda, oracle, i):
    """Bit-exact ray casting on the GPU's rasters for 16 poses (see _random_poses),
    with 1..6 cascades of 256^2 or 512^2 at 320x200."""
    from paper_2201_10887_b200 import render_frame
    from paper_2201_10887_b200.cascade import CameraView
    from paper_2201_10887_b200.rbf import RbfParams
    from paper_2201_10887_b200.render import CascadeSettings, FrameConfig
    cfg, g, t, _ = _config_inputs("C2")
    eye, look, up, fov = _random_poses()[i]
    W, H = 320, 200
    cam = CameraView(eye=eye, look_dir=look, up=up, fov_y=fov, aspect=W / H, near_clip=1.0, far_clip=6000.0)
    st = CascadeSettings(resolution=(256, 512)[i % 2], count=1 + i % 6)
    fc = FrameConfig(width=W, height=H, camera=cam)
    fr = render_frame(fc, g, t, RbfParams(sigma=cfg.sigma), st, debug=True)
    if not fr.visible:
        pytest.skip("nothing visible from this pose")
    _frame_vs_oracle(fr, oracle, fc, g)
    prod = render_frame(fc, g, t, RbfParams(sigma=cfg.sigma), st)     # launch-list path
    assert np.array_equal(prod.pixels, fr.pixels) and prod.work == fr.work
    print(f"pose {i}: K={st.count} R={st.resolution} rays_hit={fr.rays_hit}")


@pytest.mark.parametrize("R,K,overlap", [(300, 2, 5.0), (1000, 3, "auto"), (129, 5, 0.0), (777, 8, 12.5),
                                         (4, 1, 0.0), (5, 2, "auto"), (33, 3, 1.0), (65, 2, "auto"),
                                         (4096, 2, "auto")])
def test_odd_resolution_frame_parity(cuda, oracle, R, K, overlap):
    """Non-power-of-two cascade resolutions (odd pyramid widths, -inf padding, partial
    CTA tiles in every kernel), explicit overlaps and up to 8 cascades, down to the
    reference's minimum R = 4 (cascade.py:454) and up to 4096^2 cascades: bit-exact ray
    casting on the GPU's rasters, exact masks/valid bits, heights within tolerance."""
    from paper_2201_10887_b200 import render_frame
    from paper_2201_10887_b200.rbf import RbfParams
    from paper_2201_10887_b200.render import CascadeSettings, FrameConfig
    cfg, g, t, fc = _config_inputs("C2", 480, 300)
    st = CascadeSettings(resolution=R, count=K, overlap=overlap)
    fr = render_frame(fc, g, t, RbfParams(sigma=cfg.sigma), st, debug=True)
    assert fr.visible
    _frame_vs_oracle(fr, oracle, fc, g)
    for L, r in zip([L for L in fr.debug["layouts"] if L is not None], fr.debug["rasters"]):
        o = oracle.discretize(L, g, t, cfg.sigma)
        valid = _np(r.valid)
        assert np.array_equal(valid, o.valid) and np.array_equal(_np(L.mask), o.mask)
        for layer in ("terrain", "water"):
            _check_heights(_np(r.layer(layer)), o.layer(layer), valid, f"R={R} {layer}")


def test_sharded_strips_need_six_mip_levels(cuda):
    """Screen-strip sharding exchanges level-5 mip nodes, so it needs 7 mip levels,
    R >= 34 (hc_frame_xchg_floats == 0 below); a smaller raster is refused, not
    mis-rendered, and the smallest allowed one renders bit-identical strips."""
    from paper_2201_10887_b200 import multi
    from paper_2201_10887_b200.render import CascadeSettings
    cfg, g, t, fc = _config_inputs("C2", 480, 300)
    with pytest.raises(ValueError, match="at least 34"):
        multi.StripFrame(fc, g, t, CascadeSettings(resolution=33, count=2), multi.screen_strips(480, 2), 0)
    img, _ = multi.render_strips_one_gpu(fc, g, t, None, CascadeSettings(resolution=34, count=2), 2)
    from paper_2201_10887_b200 import render_frame
    from paper_2201_10887_b200.rbf import RbfParams
    full = render_frame(fc, g, t, RbfParams(sigma=cfg.sigma), CascadeSettings(resolution=34, count=2)).pixels
    assert np.array_equal(img, full)


@pytest.mark.parametrize("i", range(8))
def test_sharded_strips_random_poses(cuda, i):
    """Sharded screen strips at the stress poses (grazing, below-terrain, outside the
    domain, straight down -- where a strip may reach the whole plane), random strip
    counts and uneven cuts, 1-6 cascades: the emulated ranks' image equals the
    single-GPU frame bit for bit."""
    from paper_2201_10887_b200 import multi, render_frame
    from paper_2201_10887_b200.cascade import CameraView
    from paper_2201_10887_b200.rbf import RbfParams
    from paper_2201_10887_b200.render import CascadeSettings, FrameConfig
    cfg, g, t, _ = _config_inputs("C2")
    rng = np.random.default_rng(77 + i)
    eye, look, up, fov = _random_poses()[2 * i]
    W, H = 480, 270
    cam = CameraView(eye=eye, look_dir=look, up=up, fov_y=fov, aspect=W / H, near_clip=1.0, far_clip=6000.0)
    st = CascadeSettings(resolution=(256, 512, 300)[i % 3], count=1 + (i * 5) % 6)
    fc = FrameConfig(width=W, height=H, camera=cam)
    full = render_frame(fc, g, t, RbfParams(sigma=cfg.sigma), st)
    if not full.visible:
        pytest.skip("nothing visible from this pose")
    world = int(rng.integers(2, 7))
    cuts = sorted(set(int(c) for c in rng.integers(1, W // 8, world - 1) * 8))
    rects = [(a, b) for a, b in zip([0] + cuts, cuts + [W])]
    img, _ = multi.render_strips_one_gpu(fc, g, t, None, st, len(rects), rects)
    assert np.array_equal(img, full.pixels), (i, rects)


def test_division_selftest(cuda):
    """The traversal's hoisted float64 division equals IEEE a / b on 2^28 operand pairs."""
    import torch
    from paper_2201_10887_b200 import _cuda
    mm = torch.zeros(1, dtype=torch.int64, device=cuda)
    _cuda.check(_cuda.lib().hc_selftest_division(1 << 28, 2024, mm.data_ptr(), _cuda.stream_ptr()), "selftest")
    assert int(mm.item()) == 0


def test_edge_cases_k_counts_and_nothing_visible(cuda, oracle):
    """K = 1 / 2 / 8 cascades, tiny rasters, a camera looking away (background frame)."""
    from paper_2201_10887_b200 import render_frame, CascadeSettings
    from paper_2201_10887_b200.cascade import CameraView
    from paper_2201_10887_b200.render import FrameConfig
    from paper_2201_10887_b200.rbf import RbfParams
    sc, g, t, cfg, st = demo_setup()
    for K, R in ((1, 64), (2, 128), (8, 256), (5, 32)):
        fr = render_frame(cfg, g, t, RbfParams(sigma=sc.sigma), CascadeSettings(resolution=R, count=K), debug=True)
        _frame_vs_oracle(fr, oracle, cfg, g)
    away = FrameConfig(width=64, height=48, camera=CameraView(eye=(-500.0, -500.0, 100.0), look_dir=(-1.0, -1.0, 0.5),
                                                                up=(0, 0, 1), fov_y=30.0, aspect=64 / 48,
                                                                near_clip=1.0, far_clip=100.0))
    fr = render_frame(away, g, t, RbfParams(sigma=sc.sigma), st)
    assert not fr.visible and np.all(fr.pixels == np.array(away.background, dtype=np.uint8))


def test_screen_strips_equal_full_frame(cuda):
    """C5-style screen strips reproduce the single-GPU frame bit for bit: each rank with
    full cascades, and sharded (each rank discretizes its strip's footprint, level-5
    mips and valid partials MAX-reduced), ranks emulated one after another."""
    import torch
    from paper_2201_10887_b200 import multi, render_frame
    from paper_2201_10887_b200.rbf import RbfParams
    sc, g, t, cfg, st = demo_setup()
    full = render_frame(cfg, g, t, RbfParams(sigma=sc.sigma), st).pixels
    for world in (2, 3, 8):
        parts = [multi.render_strip(cfg, g, t, RbfParams(sigma=sc.sigma), st, r)
                 for r in multi.screen_strips(cfg.width, world)]
        img = torch.cat(parts, dim=1).cpu().numpy()
        assert np.array_equal(img, full), world
        # sharded: each rank discretizes its footprint only, mips exchanged by MAX
        img, _ = multi.render_strips_one_gpu(cfg, g, t, RbfParams(sigma=sc.sigma), st, world)
        assert np.array_equal(img, full), ("sharded", world)
    # C2 at 1080p, 2..8 strips, also with uneven (cost-balanced style) cuts
    cfg2, g2, t2, fc2 = _config_inputs("C2")
    P2 = RbfParams(sigma=cfg2.sigma)
    full2 = render_frame(fc2, g2, t2, P2, cfg2.settings()).pixels
    for world, rects in ((2, None), (4, None), (8, None), (3, [(0, 200), (200, 1304), (1304, 1920)])):
        img, _ = multi.render_strips_one_gpu(fc2, g2, t2, P2, cfg2.settings(), world, rects)
        assert np.array_equal(img, full2), ("C2 sharded", world)


@pytest.mark.parametrize("spec", gi.GRID_SPECS, ids=lambda s: s["name"])
def test_gpu_influence_table_matches_reference(cuda, spec):
    """hc_influence_build reproduces the reference's CSR arrays exactly."""
    from paper_2201_10887_b200 import build_influence_table, synth
    g = synth.generate_synthetic(spec["kind"], spec["seed"], spec["cells"], max_depth=spec["max_depth"])
    d = GOLD["grids"][spec["name"]]
    for sigma in spec["sigmas"]:
        t = build_influence_table(g, sigma)
        assert sha(t.offsets) == d[f"table_{sigma}"]["offsets"]
        assert sha(t.indices) == d[f"table_{sigma}"]["indices"]


def test_gpu_influence_table_large_configs(cuda, oracle):
    from paper_2201_10887_b200 import build_influence_table
    from paper_2201_10887_b200.configs import CONFIGS
    for name in ("C2", "C3"):
        cfg = CONFIGS[name]
        g = cfg.grid()
        a = build_influence_table(g, cfg.sigma)
        b = oracle.build_influence_table(g, cfg.sigma)
        assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.indices, b.indices), name


def test_render_frames_pipeline_equals_render_frame(cuda):
    """render_frames (two buffer sets, read-back on a copy stream overlapping the next
    frame) yields exactly render_frame's pixels and counters for every pose."""
    import dataclasses
    from paper_2201_10887_b200 import render_frame, render_frames
    from paper_2201_10887_b200.rbf import RbfParams
    sc, g, t, cfg, st = demo_setup()
    cam = cfg.camera
    poses = []
    for k in range(5):
        eye = (cam.eye[0] + 7.0 * k, cam.eye[1] - 5.0 * k, cam.eye[2] + 3.0 * k)
        poses.append(dataclasses.replace(cfg, camera=dataclasses.replace(cam, eye=eye)))
    P = RbfParams(sigma=sc.sigma)
    seq = list(render_frames(poses, g, t, P, st))
    assert len(seq) == len(poses)
    for f, c in zip(seq, poses):
        ref = render_frame(c, g, t, P, st)
        assert np.array_equal(f.pixels, ref.pixels)
        assert (f.visible_texels, f.rays_hit, f.work) == (ref.visible_texels, ref.rays_hit, ref.work)


def test_scalar_twins_match_reference(cuda):
    """traverse_cascade and cast_through_cascades (raycast.py:195-256, the scalar
    API) against the reference's own outputs (tests/golden/make_golden_twins.py):
    3 poses x 1536 pixel rays x 2 layers over K=3 cascades planned by both sides,
    every field bit-exact (hit, t, world position, cascade, uv, patch, blend)."""
    import torch
    from paper_2201_10887_b200 import build_max_mipmap, cast_through_cascades, plan_cascades, synth, traverse_cascade
    from paper_2201_10887_b200.cascade import CameraView
    from paper_2201_10887_b200.discretize import CascadeRaster, compute_visibility_mask
    data = npz("scalar_twins.npz")
    g = synth.generate_synthetic(gi.TWIN_GRID["kind"], gi.TWIN_GRID["seed"], gi.TWIN_GRID["cells"])
    n_hits = n_blend = 0
    for p, pose in enumerate(gi.TWIN_POSES):
        cam = CameraView(**gi.twin_camera_args(pose))
        _, _, lays = plan_cascades(cam, g, pose["res"], "auto")
        assert len(lays) == int(data[f"p{p}_n_cascades"])
        rasters, mips = [], {"terrain": [], "water": []}
        for L in lays:
            if L is None:
                rasters.append(None)
                for layer in mips:
                    mips[layer].append(None)
                continue
            mask = _np(compute_visibility_mask(L)).astype(bool)
            ter, wat, val = gi.twin_raster(L.world_origin, L.texel_size, L.resolution, mask)
            dev = lambda a: torch.from_numpy(a.astype(np.float32)).to(cuda)
            r = CascadeRaster(L, dev(ter), dev(wat), torch.from_numpy(val).to(cuda), float(ter.min()) - 1.0)
            rasters.append(r)
            for layer in mips:
                mips[layer].append(build_max_mipmap(r, layer))
        origin = np.asarray(cam.eye, dtype=np.float64)
        dirs = data[f"p{p}_dirs"]
        for layer in ("terrain", "water"):
            want = data[f"p{p}_{layer}_cast"]
            for i, d in enumerate(dirs):
                h = cast_through_cascades(origin, d, rasters, mips[layer], lays)
                w = want[i]
                assert (h is not None) == bool(w[0]), (p, layer, i)
                if h is None:
                    continue
                b = h.blend if h.blend is not None else (-1, np.nan)
                got = np.array([1, h.t, *h.world_pos, h.cascade, *h.uv, *h.patch, b[0], b[1]])
                assert np.array_equal(got, w, equal_nan=True), (p, layer, i, got, w)
                n_hits += 1
                n_blend += b[0] >= 0
            for k, (r, m) in enumerate(zip(rasters, mips[layer])):
                if r is None:
                    continue
                want = data[f"p{p}_{layer}_trav{k}"]
                for i in range(0, len(dirs), 3):
                    h = traverse_cascade(origin, dirs[i], r, m)
                    got = (np.array([0, np.nan, np.nan, np.nan, -1, -1]) if h is None
                           else np.array([1, h.t, *h.uv, *h.patch]))
                    assert np.array_equal(got, want[i], equal_nan=True), (p, layer, k, i)
    assert n_hits > 3000 and n_blend > 100


def test_nccl_exchange_and_gather_single_rank(cuda):
    """The sharded frame's collectives on the NCCL backend (one rank on this GPU: the
    only multi-GPU evidence one GPU can give): a sharded C2 strip frame whose exchange
    buffer goes through dist.all_reduce(MAX) and whose image goes through
    dist.gather equals the plain frame."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_2201_10887_b200 import multi, render_frame
    from paper_2201_10887_b200.rbf import RbfParams
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    try:
        cfg, g, t, fc = _config_inputs("C2")
        P = RbfParams(sigma=cfg.sigma)
        rects = [(0, fc.width)]
        f = multi.StripFrame(fc, g, t, cfg.settings(), rects, 0, staged=True)
        f.stage1()
        before = f.xchg.clone()
        multi.all_reduce_max(f.xchg)
        assert torch.equal(before, f.xchg)           # one rank: MAX is the identity
        f.stage2()
        img = multi.gather_strips(f.strip().clone(), rects, 0, 1)
        full = render_frame(fc, g, t, P, cfg.settings()).pixels
        assert np.array_equal(img.cpu().numpy(), full)
    finally:
        dist.destroy_process_group()

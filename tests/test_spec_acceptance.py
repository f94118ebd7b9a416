"""The reference SPEC's acceptance properties (`SPEC.md:468-479`, `:131`, `:211-216`,
`:255`), checked on this package: host planning properties on the CPU, the
discretization and RBF properties through the GPU path (`-m gpu`).

(The ray-cast property -- max-mip traversal == brute-force DDA patch walk -- is in
test_oracle_golden.py / test_gpu_parity.py; determinism and benchmark structure
in test_gpu_parity.py / test_cli.py.)
"""

import math

import numpy as np
import pytest

import golden_inputs as gi
from paper_2201_10887_b200 import cascade, synth
from paper_2201_10887_b200.cascade import CameraView


def _random_pose(rng, grid):
    d = grid.domain
    w, h = d.xmax - d.xmin, d.ymax - d.ymin
    lo, hi = grid.height_range
    eye = (float(rng.uniform(d.xmin - 0.2 * w, d.xmax + 0.2 * w)),
           float(rng.uniform(d.ymin - 0.2 * h, d.ymax + 0.2 * h)), float(hi + rng.uniform(5.0, 0.5 * w)))
    tgt = (float(rng.uniform(d.xmin, d.xmax)), float(rng.uniform(d.ymin, d.ymax)), float(rng.uniform(lo, hi)))
    look = tuple(b - a for a, b in zip(eye, tgt))
    return CameraView(eye=eye, look_dir=look, up=(0.0, 0.0, 1.0), fov_y=float(rng.uniform(30.0, 80.0)),
                      aspect=float(rng.uniform(1.0, 2.0)), near_clip=1.0, far_clip=float(rng.uniform(2.0, 4.0) * w))


_GRID = {}


def _pond():
    if "g" not in _GRID:
        s = next(s for s in gi.GRID_SPECS if s["name"] == "pond3000")
        _GRID["g"] = synth.generate_synthetic(s["kind"], s["seed"], s["cells"])
    return _GRID["g"]


def test_split_depths_monotone():
    """split_depths(1, 8) = (2, 4) exactly; n < d1 < d2 < f on 10^3 random (n, f)."""
    assert cascade.split_depths(1.0, 8.0) == (2.0, 4.0)
    rng = np.random.default_rng(474)
    for _ in range(1000):
        n = float(10 ** rng.uniform(-3, 2))
        f = n * float(10 ** rng.uniform(0.05, 5))
        d1, d2 = cascade.split_depths(n, f)
        assert n < d1 < d2 < f, (n, f, d1, d2)


def test_lattice_stability_and_monotone_texels():
    """moving the camera by one min_cell along an axis moves every
    cascade's origin by a whole number of texels (the texel-centre lattice is unchanged
    modulo min_cell), and texel sizes grow from near to far cascades."""
    g = _pond()
    mc = g.min_cell_size
    rng = np.random.default_rng(475)
    checked = 0
    for _ in range(1000):
        cam = _random_pose(rng, g)
        try:
            _, _, lays = cascade.plan_cascades(cam, g, 256, "auto", 3)
        except cascade.NothingVisibleError:
            continue
        present = [L for L in lays if L is not None]
        for a, b in zip(present, present[1:]):
            assert a.texel_size <= b.texel_size
        axis = int(rng.integers(0, 2))
        eye = list(cam.eye)
        eye[axis] += mc * float(rng.choice([-1.0, 1.0]))
        moved = CameraView(eye=tuple(eye), look_dir=cam.look_dir, up=cam.up, fov_y=cam.fov_y, aspect=cam.aspect,
                           near_clip=cam.near_clip, far_clip=cam.far_clip)
        try:
            _, _, lays2 = cascade.plan_cascades(moved, g, 256, "auto", 3)
        except cascade.NothingVisibleError:
            continue
        for L1, L2 in zip(lays, lays2):
            if L1 is None or L2 is None or L1.texel_size != L2.texel_size:
                continue
            for k in range(2):
                shift = (L2.world_origin[k] - L1.world_origin[k]) / L1.texel_size
                assert abs(shift - round(shift)) < 1e-6, (k, shift)
            checked += 1
    assert checked >= 500


def test_hull_coverage(oracle):
    """random points inside the visible hull fall in at least one cascade
    polygon and in a masked-visible texel of that cascade's layout (100 poses x 1000 points)."""
    g = _pond()
    rng = np.random.default_rng(476)
    poses = 0
    while poses < 100:
        cam = _random_pose(rng, g)
        try:
            hull, polys, lays = cascade.plan_cascades(cam, g, 256, "auto", 3)
        except cascade.NothingVisibleError:
            continue
        hull = np.asarray(hull, dtype=np.float64)
        lo, hi = hull.min(axis=0), hull.max(axis=0)
        pts = rng.uniform(lo, hi, size=(4000, 2))
        pts = pts[_inside(hull, pts)][:1000]
        if len(pts) < 100:
            continue
        masks = [oracle.visibility_cells(L, g)[0] if L is not None else None for L in lays]
        covered = np.zeros(len(pts), dtype=bool)
        for poly, L, mask in zip(polys, lays, masks):
            if poly is None or L is None:
                continue
            inp = _inside(np.asarray(poly.vertices, dtype=np.float64), pts)
            ij = np.rint((pts - np.asarray(L.world_origin)) / L.texel_size).astype(np.int64)
            ok = (ij >= 0).all(axis=1) & (ij < L.resolution).all(axis=1)
            vis = np.zeros(len(pts), dtype=bool)
            vis[ok] = mask[ij[ok, 1], ij[ok, 0]].astype(bool)
            assert np.all(vis[inp]), "a point inside a cascade polygon has an unmasked texel"
            covered |= inp
        assert covered.all(), f"{int((~covered).sum())} hull points outside every cascade polygon"
        poses += 1


def _inside(poly, pts, eps=1e-9):
    """Points inside (or on) a counter-clockwise convex polygon."""
    ok = np.ones(len(pts), dtype=bool)
    n = len(poly)
    for i in range(n):
        a, b = poly[i], poly[(i + 1) % n]
        cross = (b[0] - a[0]) * (pts[:, 1] - a[1]) - (b[1] - a[1]) * (pts[:, 0] - a[0])
        ok &= cross >= -eps * max(1.0, float(np.hypot(*(b - a))))
    return ok


@pytest.mark.gpu
def test_constant_reproduction(cuda):
    """a constant grid discretizes to the constant exactly in every valid
    texel (terrain 100, water 100; and with depth 2, water 102)."""
    from paper_2201_10887_b200 import AdaptiveGrid, build_influence_table, discretize_cascade
    from paper_2201_10887_b200.rbf import RbfParams
    g0 = _pond()
    for depth in (0.0, 2.0):
        g = AdaptiveGrid(g0.domain, g0.min_cell_size, g0.centers, g0.sizes, np.full(g0.n_cells, 100.0),
                         np.full(g0.n_cells, depth))
        t = build_influence_table(g, 1.0)
        rng = np.random.default_rng(471)
        n = 0
        while n < 3:
            try:
                _, _, lays = cascade.plan_cascades(_random_pose(rng, g), g, 256, "auto", 3)
            except cascade.NothingVisibleError:
                continue
            for L in (L for L in lays if L is not None):
                r = discretize_cascade(L, g, t, RbfParams(1.0))
                v = r.valid.cpu().numpy()
                assert v.any()
                assert np.all(r.terrain.cpu().numpy()[v] == np.float32(100.0))
                assert np.all(r.water.cpu().numpy()[v] == np.float32(100.0 + depth))
            n += 1


@pytest.mark.gpu
def test_approximate_equals_exhaustive_sum(cuda):
    """approximate() equals the exhaustive Eq. 2 sum over ALL cells
    (no influence table) within 1e-12 relative, on 20 random grids x 100 interior points."""
    from paper_2201_10887_b200 import approximate, build_influence_table
    from paper_2201_10887_b200.rbf import RbfParams
    rem = math.exp(-0.5 * 3.5 ** 2)
    n_pts = 0
    for case in gi.rbf_cases():
        g = synth.generate_synthetic(case["kind"], case["seed"], case["cells"], max_depth=case["max_depth"])
        P = RbfParams(sigma=case["sigma"])
        t = build_influence_table(g, case["sigma"])
        c = np.asarray(g.centers, dtype=np.float64)
        cs = np.asarray(g.sizes, dtype=np.float64) * case["sigma"]
        for p in gi.rbf_points(g.domain, case["seed"], case["n_points"]):
            r2 = ((c[:, 0] - p[0]) ** 2 + (c[:, 1] - p[1]) ** 2) / cs ** 2
            w = np.maximum(np.exp(-0.5 * r2) - rem, 0.0)
            w[r2 >= 12.25 * (1.0 - 1e-12)] = 0.0
            for layer, vals in (("terrain", g.terrain), ("water", g.terrain + g.water_depth)):
                want = float(np.sum(w * vals) / np.sum(w)) if layer == "terrain" else None
                got = approximate(tuple(p), layer, g, t, P).value
                if layer == "terrain":
                    assert abs(got - want) <= 1e-12 * abs(want), (case["name"], p, got, want)
                else:
                    ter = float(np.sum(w * g.terrain) / np.sum(w))
                    dep = max(float(np.sum(w * g.water_depth) / np.sum(w)), 0.0)
                    assert abs(got - (ter + dep)) <= 1e-12 * abs(ter + dep), (case["name"], p, got, ter + dep)
            n_pts += 1
    assert n_pts >= 2000


@pytest.mark.gpu
def test_blend_endpoints_and_convexity(cuda):
    """blended depths are convex combinations of the two cascades'
    hits and the blend endpoints reproduce single-cascade hits exactly (w = 0: the
    near cascade's t; w = 1: the far one's), on the C2 frame and one orbit pose."""
    from paper_2201_10887_b200 import build_influence_table, render_frame
    from paper_2201_10887_b200.configs import CONFIGS
    from paper_2201_10887_b200.rbf import RbfParams
    cfg = CONFIGS["C2"]
    g = cfg.grid()
    t = build_influence_table(g, cfg.sigma)
    n_blend = 0
    for view in (0, 1):
        fc = cfg.frame_config(view)
        fr = render_frame(fc, g, t, RbfParams(cfg.sigma), cfg.settings(), debug=True)
        for layer in ("terrain", "water"):
            L = fr.debug[layer]
            hit = L.hit.cpu().numpy()
            far = L.far.cpu().numpy()
            w = L.w.cpu().numpy()
            tt = L.t.cpu().numpy()
            t0 = L.raw_slots["t"][0].cpu().numpy()
            t1 = L.raw_slots["t"][1].cpu().numpy()
            b = hit & (far >= 0)
            assert np.all((w[b] >= 0.0) & (w[b] <= 1.0))
            lo, hi = np.minimum(t0[b], t1[b]), np.maximum(t0[b], t1[b])
            assert np.all((tt[b] >= lo * (1 - 1e-15)) & (tt[b] <= hi * (1 + 1e-15)))
            e0, e1 = b & (w == 0.0), b & (w == 1.0)
            assert np.array_equal(tt[e0], t0[e0]) and np.array_equal(tt[e1], t1[e1])
            single = hit & (far < 0)
            assert np.array_equal(tt[single], t0[single])
            n_blend += int(b.sum())
    assert n_blend > 1000

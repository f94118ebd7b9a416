"""Native (C++) cascade planner vs the numpy restatement of the reference planner.

K=3 is pinned against the reference itself in test_oracle_golden.py; here the
native planner is compared bit for bit with oracle/plan_numpy.py (same numpy
calls as cascade.py) on many random poses and for K = 1..8.
"""

import numpy as np
import pytest

import plan_numpy as PN
from helpers import sha

from paper_2201_10887_b200 import cascade, synth


def _poses(n, seed, ext):
    rng = np.random.default_rng(seed)
    for i in range(n):
        eye = (float(rng.uniform(-0.3, 1.3) * ext), float(rng.uniform(-0.3, 1.3) * ext),
               float(rng.uniform(5.0, 0.5 * ext)))
        la = (float(rng.uniform(0, ext)), float(rng.uniform(0, ext)), float(rng.uniform(0, 80)))
        if i % 17 == 3:
            la = (eye[0] - 400.0, eye[1] + 10.0, eye[2] + 50.0)   # looking up and away
        look = tuple(b - a for a, b in zip(eye, la))
        yield dict(eye=eye, look_dir=look, up=(0.0, 0.0, 1.0), fov_y=float(rng.uniform(20, 100)),
                   aspect=float(rng.uniform(0.5, 2.5)), near_clip=float(rng.choice([0.5, 1.0, 5.0])),
                   far_clip=float(rng.choice([0.5 * ext, 2.0 * ext, 6000.0]))), int(rng.choice([16, 64, 256, 1024, 2048])), \
            ("auto" if rng.random() < 0.6 else float(rng.uniform(0, 0.03 * ext)))


@pytest.mark.parametrize("K", [1, 2, 3, 4, 5, 8])
def test_native_planner_matches_numpy_restatement(K):
    g = synth.generate_synthetic("pond", 42, 3000)
    n_vis = 0
    for kw, R, ov in _poses(60, 100 + K, 2048.0):
        try:
            want = PN.plan_cascades(PN.CameraView(**kw), g, R, ov, K)
        except PN.NothingVisibleError:
            with pytest.raises(cascade.NothingVisibleError):
                cascade.plan_cascades(cascade.CameraView(**kw), g, R, ov, K)
            continue
        n_vis += 1
        got = cascade.plan_cascades(cascade.CameraView(**kw), g, R, ov, K)
        assert sha(got[0]) == sha(want[0])
        for a, b in zip(got[2], want[2]):
            assert (a is None) == (b is None)
            if a is None:
                continue
            assert a.world_origin.tolist() == b.world_origin.tolist() and a.texel_size == b.texel_size
            assert sha(a.polygon.vertices) == sha(b.polygon.vertices)
            assert a.polygon.near_offset == b.polygon.near_offset and a.polygon.far_offset == b.polygon.far_offset
            assert tuple(a.polygon.axis.anchor) == tuple(b.polygon.axis.anchor)
            assert tuple(a.polygon.axis.direction) == tuple(b.polygon.axis.direction)
            assert a.box_texel == b.box_texel and a.box_steps == b.box_steps and a.index == b.index
            assert sha(a.edge_table()) == sha(b.edge_table())
    assert n_vis >= 30


def test_individual_planner_functions_match():
    g = synth.generate_synthetic("hill", 9, 2000)
    for kw, R, ov in _poses(25, 7, 2048.0):
        try:
            hull = PN.visible_hull(PN.CameraView(**kw), g)
        except PN.NothingVisibleError:
            continue
        assert sha(cascade.visible_hull(cascade.CameraView(**kw), g)) == sha(hull)
        ax = PN.view_axis_2d(PN.CameraView(**kw))
        ov = 3.0 if ov == "auto" else ov
        for K in (1, 3, 6):
            P = PN.clip_cascade_polygons(hull, ax, ov, kw["eye"][:2], K)
            Q = cascade.clip_cascade_polygons(hull, ax, ov, kw["eye"][:2], K)
            for p, q in zip(P, Q):
                assert (p is None) == (q is None)
                if p is not None:
                    assert sha(p.vertices) == sha(q.vertices) and p.near_offset == q.near_offset
                    a = PN.fit_layout(p, R, g.min_cell_size, 0.5)
                    b = cascade.fit_layout(q, R, g.min_cell_size, 0.5)
                    assert a.world_origin.tolist() == b.world_origin.tolist() and a.texel_size == b.texel_size


def test_python_hypot_replica():
    import math
    from paper_2201_10887_b200 import _cuda
    rng = np.random.default_rng(1)
    hyp = _cuda.lib().hc_py_hypot
    for x, y in rng.normal(0, 500, (20000, 2)).tolist():
        assert hyp(x, y) == math.hypot(x, y)

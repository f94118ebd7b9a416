"""Dev analysis (CPU): how much of the heaviest rays' max-mip walks a min pyramid
would skip.  For the given pixels of a config, every cascade traversal of the
terrain layer is replayed in Python (the reference walk, _kernels.py:75-215) with
visit counts, and again with an additional skip of nodes the ray segment passes
entirely below (max(za, zb) < node min - margin, min over the node's valid
patches' corners).

    python tools/underground_probe.py --config C2 --pixels 836,487 562,514 1047,491
"""

import argparse
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

FAR = 1e300


def pyramids(h, valid):
    n0 = h.shape[0] - 1
    pv = valid[:-1, :-1] & valid[1:, :-1] & valid[:-1, 1:] & valid[1:, 1:]
    c = np.stack([h[:-1, :-1], h[:-1, 1:], h[1:, :-1], h[1:, 1:]])
    mx = [c.max(axis=0)]
    mn = [np.where(pv, c.min(axis=0), np.inf)]
    while mx[-1].shape[0] > 1:
        a, b = mx[-1], mn[-1]
        w = (a.shape[0] + 1) // 2
        pa = np.full((2 * w, 2 * w), -np.inf)
        pb = np.full((2 * w, 2 * w), np.inf)
        pa[:a.shape[0], :a.shape[1]] = a
        pb[:b.shape[0], :b.shape[1]] = b
        mx.append(pa.reshape(w, 2, w, 2).max(axis=(1, 3)))
        mn.append(pb.reshape(w, 2, w, 2).min(axis=(1, 3)))
    return mx, mn, pv, n0


def patch_roots(h00, h10, h01, h11, u0, v0, du, dv, z0, dz, seg):
    """_kernels.py:26-72 (first root in [0, seg])."""
    e10, e01 = h10 - h00, h01 - h00
    kk = ((h11 - h10) - h01) + h00
    a = (du * dv) * kk
    b = (((du * e10) + (dv * e01)) + (kk * ((u0 * dv) + (v0 * du)))) - dz
    c = (((h00 + (u0 * e10)) + (v0 * e01)) + ((kk * u0) * v0)) - z0
    r1 = r2 = FAR
    if abs(a) < 1e-12 * abs(b):
        if b != 0.0:
            r1 = -c / b
    else:
        disc = (b * b) - ((4.0 * a) * c)
        if disc >= 0.0:
            sq = math.sqrt(disc)
            q = (-0.5 * (b + sq)) if b >= 0.0 else (-0.5 * (b - sq))
            if q != 0.0:
                r1, r2 = q / a, c / q
            else:
                r1, r2 = 0.0, -b / a
            if r2 < r1:
                r1, r2 = r2, r1
    for r in (r1, r2):
        if 0.0 <= r <= seg:
            return r
    return None


def walk(P, h, rx, ry, rz, dx, dy, dz, hmin, hmax, use_min, margin=1e-6):
    mx, mn, pv, n0 = P
    t0, t1 = 0.0, FAR
    for o, d, lo, hi in ((rx, dx, 0.0, float(n0)), (ry, dy, 0.0, float(n0)), (rz, dz, hmin, hmax)):
        if d != 0.0:
            ta, tb = (lo - o) / d, (hi - o) / d
            if ta > tb:
                ta, tb = tb, ta
            t0, t1 = max(t0, ta), min(t1, tb)
        elif o < lo or o > hi:
            return 0, None
    if t0 > t1:
        return 0, None
    cx = min(max(int(math.floor(rx + t0 * dx)), 0), n0 - 1)
    cy = min(max(int(math.floor(ry + t0 * dy)), 0), n0 - 1)
    t = t0
    level = len(mx) - 1
    visits = 0
    while True:
        visits += 1
        nx, ny = cx >> level, cy >> level
        x0, y0 = float(nx << level), float(ny << level)
        x1, y1 = x0 + (1 << level), y0 + (1 << level)
        tx = (x1 - rx) / dx if dx > 0 else ((x0 - rx) / dx if dx < 0 else FAR)
        ty = (y1 - ry) / dy if dy > 0 else ((y0 - ry) / dy if dy < 0 else FAR)
        t_wall = min(tx, ty)
        seg_end = min(t_wall, t1)
        za, zb = rz + t * dz, rz + seg_end * dz
        nmax = mx[level][ny, nx]
        below = use_min and max(za, zb) < mn[level][ny, nx] - margin
        if min(za, zb) > nmax or below:
            pass
        elif level > 0:
            level -= 1
            continue
        else:
            if pv[cy, cx]:
                u0, v0 = (rx + t * dx) - cx, (ry + t * dy) - cy
                tau = patch_roots(h[cy, cx], h[cy, cx + 1], h[cy + 1, cx], h[cy + 1, cx + 1], u0, v0, dx, dy,
                                  za, dz, seg_end - t)
                if tau is not None:
                    return visits, (cx, cy, t + tau)
        if t_wall > t1:
            return visits, None
        if tx <= ty:
            t = tx
            cx = (nx + 1) << level if dx > 0 else (nx << level) - 1
            cy = min(max(int(math.floor(ry + t * dy)), ny << level), ((ny + 1) << level) - 1)
        else:
            t = ty
            cy = (ny + 1) << level if dy > 0 else (ny << level) - 1
            cx = min(max(int(math.floor(rx + t * dx)), nx << level), ((nx + 1) << level) - 1)
        if cx < 0 or cx > n0 - 1 or cy < 0 or cy > n0 - 1 or t > t1:
            return visits, None
        if level < len(mx) - 1:
            level += 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--pixels", nargs="+", default=["836,487", "562,514", "1047,491", "658,492", "1048,491"])
    a = ap.parse_args()
    import heightcast_oracle as O
    import plan_numpy as PN
    from paper_2201_10887_b200.configs import CONFIGS
    cfg = CONFIGS[a.config]
    g = cfg.grid()
    table = O.build_influence_table(g, cfg.sigma)
    fc, st = cfg.frame_config(), cfg.settings()
    c = fc.camera
    cam = PN.CameraView(eye=c.eye, look_dir=c.look_dir, up=c.up, fov_y=c.fov_y, aspect=c.aspect,
                        near_clip=c.near_clip, far_clip=c.far_clip)
    plan = PN.plan_cascades(cam, g, st.resolution, st.overlap, st.count)
    lays = [L for L in plan[2] if L is not None]
    rasters, pyr = [], []
    for L in lays:
        r = O.discretize(L, g, table, cfg.sigma)
        h = r.terrain.astype(np.float32).astype(np.float64)
        v = r.valid.astype(bool)
        vals = h[v]
        rasters.append((h, v, float(vals.min()), float(vals.max())))
        pyr.append(pyramids(h, v))
    dirs = O.ray_dirs(fc.camera, fc.width, fc.height)
    for px in a.pixels:
        i, j = (int(x) for x in px.split(","))
        d = dirs[j, i]
        print(f"pixel ({i},{j}):")
        for k, (L, (h, v, lo, hi), P) in enumerate(zip(lays, rasters, pyr)):
            s = L.texel_size
            rx, ry = (c.eye[0] - L.world_origin[0]) / s, (c.eye[1] - L.world_origin[1]) / s
            n_max, r_max = walk(P, h, rx, ry, c.eye[2], d[0] / s, d[1] / s, d[2], lo, hi, False)
            n_min, r_min = walk(P, h, rx, ry, c.eye[2], d[0] / s, d[1] / s, d[2], lo, hi, True)
            print(f"  cascade {k}: visits max-mip {n_max:5d} -> with min skip {n_min:5d}   "
                  f"first candidate {r_max} / {r_min}")


if __name__ == "__main__":
    main()

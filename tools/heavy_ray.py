"""Isolated latency of the heaviest render tile (dev tool, GPU box).

    python tools/heavy_ray.py --config C2

Renders the full frame, finds the tile with the largest per-lane node-visit
count, then renders only that tile (hc_render's pixel rectangle) and reports
the render-kernel time: the latency floor of the frame's longest ray chain
when it runs alone, vs. the full launch."""

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--frames", type=int, default=5)
    a = ap.parse_args()
    from paper_2201_10887_b200 import build_influence_table
    from paper_2201_10887_b200.configs import CONFIGS
    from paper_2201_10887_b200.multi import TILE_H, TILE_W
    from paper_2201_10887_b200.render import enqueue_frame
    cfg = CONFIGS[a.config]
    g = cfg.grid()
    t = build_influence_table(g, cfg.sigma)
    fc, st = cfg.frame_config(), cfg.settings()

    def run(rect=None):
        r = []
        for _ in range(a.frames):
            buf, _p, _ms = enqueue_frame(fc, g, t, st, rect=rect)
            buf.ev[2].synchronize()
            r.append(buf.ev[4].elapsed_time(buf.ev[2]))
        return buf, float(np.median(r))

    buf, full = run()
    cost = buf.tile_cost.cpu().numpy().copy()
    tx = (fc.width + TILE_W - 1) // TILE_W
    order = np.argsort(cost)[::-1]
    print(f"{a.config}: full render {full:.3f} ms; heaviest tiles {cost[order[:4]].tolist()}")
    for k in order[:3]:
        x0, y0 = int(k % tx) * TILE_W, int(k // tx) * TILE_H
        rect = (x0, y0, min(x0 + TILE_W, fc.width), min(y0 + TILE_H, fc.height))
        _b, ms = run(rect)
        print(f"  tile {int(k)} rect {rect} visits {int(cost[k])}: alone {ms:.3f} ms "
              f"({ms * 1e3 / max(int(cost[k]), 1):.3f} us/visit)")
    # per-lane visits of the heaviest tile, and its heaviest pixel alone
    from paper_2201_10887_b200.rbf import RbfParams
    from paper_2201_10887_b200.render import render_frame
    f = render_frame(fc, g, t, RbfParams(sigma=cfg.sigma), st, debug=True)
    v = f.debug["visits"].cpu().numpy().astype(np.int64).sum(axis=0).reshape(fc.height, fc.width)
    k = order[0]
    x0, y0 = int(k % tx) * TILE_W, int(k // tx) * TILE_H
    blk = v[y0:y0 + TILE_H, x0:x0 + TILE_W]
    print("  heaviest tile per-lane visits:\n" + "\n".join("    " + " ".join(f"{x:4d}" for x in row) for row in blk))
    yy, xx = np.unravel_index(np.argmax(blk), blk.shape)
    px = (x0 + int(xx), y0 + int(yy))
    _b, ms = run((px[0], px[1], px[0] + 1, px[1] + 1))
    print(f"  pixel {px} alone ({int(blk.max())} visits): {ms:.3f} ms ({ms * 1e3 / max(int(blk.max()), 1):.3f} us/visit)")
    from paper_2201_10887_b200 import _cuda
    L = _cuda.lib()
    if hasattr(L, "hc_debug_visit_trace"):     # HC_VISIT_TRACE dev build: per-visit clock stamps
        import ctypes as C
        rect1 = (px[0], px[1], px[0] + 1, px[1] + 1)
        run(rect1)
        L.hc_debug_visit_trace(1, None, None, None, 0)
        b1 = enqueue_frame(fc, g, t, st, rect=rect1)[0]
        b1.ev[2].synchronize()
        L.hc_debug_visit_trace(0, None, None, None, 0)
        nv = int(b1.counters.cpu()[5])
        nt = int(b1.counters.cpu()[6])
        vclk = (C.c_longlong * 4096)()
        vlev = (C.c_int * 4096)()
        tclk = (C.c_longlong * 4096)()
        L.hc_debug_visit_trace(-1, vclk, vlev, tclk, 4096)
        vc = np.frombuffer(vclk, dtype=np.int64)[:min(nv, 4096)]
        lv = np.frombuffer(vlev, dtype=np.int32)[:min(nv, 4096)]
        tc = np.frombuffer(tclk, dtype=np.int64)[:min(nt, 4096)]
        dt = np.diff(vc)
        print(f"  trace: {nv} visits, {nt} tests, {int(vc[-1] - vc[0])} cycles first->last visit")
        for c in np.unique(lv[:-1]):
            sel = dt[lv[:-1] == c]
            print(f"    visit at level {int(c):2d}: n={len(sel):4d} median {int(np.median(sel))} "
                  f"mean {sel.mean():.0f} cycles to the next visit")
        # test stamp -> next visit stamp
        nxt = np.searchsorted(vc, tc)
        ok = nxt < len(vc)
        if ok.any():
            print(f"    patch test -> next visit: median {int(np.median(vc[nxt[ok]] - tc[ok]))} cycles")
        print("    first 30 (level, cycles):", list(zip(lv[:30].tolist(), dt[:30].tolist())))
    # full frame again (the rect runs overwrote the shared tile-cost buffer)
    run()
    _b, full2 = run()
    print(f"  full render again {full2:.3f} ms")


if __name__ == "__main__":
    main()

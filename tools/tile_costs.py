"""Per-tile cost distribution of the render kernel (dev tool, GPU box).

    python tools/tile_costs.py --config C2

Prints the heaviest tiles' max-lane node visits, a log2 histogram and the render
time, to tell a tail-bound launch (one long ray chain) from a throughput-bound one."""

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
    ap.add_argument("--path", type=int, default=0,
                    help="instead: N poses of the bench camera path, render ms vs max tile cost per pose")
    a = ap.parse_args()
    import torch
    from paper_2201_10887_b200 import build_influence_table
    from paper_2201_10887_b200.configs import CONFIGS
    from paper_2201_10887_b200.render import enqueue_frame
    cfg = CONFIGS[a.config]
    g = cfg.grid()
    t = build_influence_table(g, cfg.sigma)
    fc, st = cfg.frame_config(), cfg.settings()
    if a.path:
        for i in range(0, 2 * 60, max(1, 120 // a.path)):
            pc = cfg.path_frame_config(i)
            rr = []
            for _ in range(3):        # the third launch orders its queue from the same pose
                buf, _p, _ms = enqueue_frame(pc, g, t, st)
                buf.ev[2].synchronize()
                rr.append(buf.ev[4].elapsed_time(buf.ev[2]))
            cost = buf.tile_cost.cpu().numpy()
            cnt = buf.counters.cpu().numpy()
            print(f"pose {i}: render {rr[-1]:.3f} ms, max tile {int(cost.max())}, top8 {np.sort(cost)[-8:][::-1].tolist()}, "
                  f"visits {cnt[5]}, sum tile max {int(cost.sum())}", flush=True)
        return
    r = []
    for _ in range(a.frames):
        buf, _p, _ms = enqueue_frame(fc, g, t, st)
        buf.ev[2].synchronize()
        r.append(buf.ev[4].elapsed_time(buf.ev[2]))
    cost = buf.tile_cost.cpu().numpy()
    cnt = buf.counters.cpu().numpy()
    print(f"{a.config}: render {np.median(r):.3f} ms, tiles {len(cost)}, visits {cnt[5]}, tests {cnt[6]}")
    srt = np.sort(cost)[::-1]
    print("top tile max-lane visits:", srt[:16].tolist())
    print("percentiles 50/90/99/99.9:", [int(np.percentile(cost, q)) for q in (50, 90, 99, 99.9)])
    h = np.bincount(np.where(cost > 0, np.log2(np.maximum(cost, 1)).astype(int), 0))
    print("log2 histogram:", {1 << i: int(c) for i, c in enumerate(h) if c})
    W = fc.width if hasattr(fc, "width") else None
    print("sum of tile max-lane visits:", int(cost.sum()), "width", W)
    # per-pixel, per-layer visits of the heaviest pixels (debug launch)
    from paper_2201_10887_b200.render import render_frame
    from paper_2201_10887_b200.rbf import RbfParams
    f = render_frame(fc, g, t, RbfParams(sigma=cfg.sigma), st, debug=True)
    v = f.debug["visits"].cpu().numpy().astype(np.int64)
    tot = v.sum(axis=0)
    top = np.argsort(tot)[::-1][:12]
    Wd = fc.width
    for p in top:
        print(f"  pixel ({p % Wd},{p // Wd}): terrain {v[0, p]} water {v[1, p]}")
    print("pixels with a water trace:", int((v[1] > 0).sum()), "of", v.shape[1],
          "; water visits", int(v[1].sum()), "terrain visits", int(v[0].sum()))


if __name__ == "__main__":
    main()

"""Render one pixel (or a small rectangle) of a config repeatedly -- a target for
ncu source-level stall sampling of a single long ray chain (dev tool, GPU box).

    python tools/heavy_pixel.py --config C2 --rect 836 487 837 488 --frames 6
"""

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--rect", type=int, nargs=4, default=(836, 487, 837, 488))
    ap.add_argument("--frames", type=int, default=6)
    a = ap.parse_args()
    from paper_2201_10887_b200 import build_influence_table
    from paper_2201_10887_b200.configs import CONFIGS
    from paper_2201_10887_b200.render import enqueue_frame
    cfg = CONFIGS[a.config]
    g = cfg.grid()
    t = build_influence_table(g, cfg.sigma)
    fc, st = cfg.frame_config(), cfg.settings()
    r = []
    for _ in range(a.frames):
        buf, _p, _ms = enqueue_frame(fc, g, t, st, rect=tuple(a.rect))
        buf.ev[2].synchronize()
        r.append(buf.ev[4].elapsed_time(buf.ev[2]))
    print(f"{a.config} rect {tuple(a.rect)}: render median {np.median(r):.3f} ms, "
          f"visits {int(buf.counters.cpu()[5])}")


if __name__ == "__main__":
    main()

"""End-to-end frames/s of `render_frames` along a config's camera path for several
pipeline depths (frames in flight), as bench.py's e2e leg measures it (an L2
flush enqueued before every frame, pixels read back into pinned memory).

    python tools/e2e_depth.py --config C2 --frames 200 --depths 2 4 6 8
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--frames", type=int, default=200)
    ap.add_argument("--depths", type=int, nargs="+", default=[2, 4, 6, 8])
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    import torch
    from paper_2201_10887_b200 import RbfParams, build_influence_table, render_frames
    from paper_2201_10887_b200.configs import CONFIGS
    cfg = CONFIGS[a.config]
    g = cfg.grid()
    table = build_influence_table(g, cfg.sigma)
    P, st = RbfParams(sigma=cfg.sigma), cfg.settings()
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    seq = [cfg.path_frame_config(i) for i in range(a.frames)]
    out = {"config": a.config, "frames": a.frames}
    for rep in range(a.reps):
        for d in a.depths:
            for _ in render_frames(seq[:16], g, table, P, st, depth=d):
                pass
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in render_frames(seq, g, table, P, st, before_frame=lambda i: flush.zero_(), depth=d):
                pass
            out.setdefault(f"depth{d}", []).append(round(a.frames / (time.perf_counter() - t0), 1))
    print(json.dumps(out))


if __name__ == "__main__":
    main()

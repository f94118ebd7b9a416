"""Render frames of a benchmark config along its camera path (dev tool, GPU box).

    python tools/frames.py --config C2 --frames 8 [--start 0]

Enqueues `frames` frames (no L2 flush, no read-back), prints the mean per-kernel
event times and the frame work counters.  Small and quick, so it is the command
to wrap in ncu:  ncu -k regex:k_discretize -s 3 -c 1 python tools/frames.py ...
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--frames", type=int, default=8)
    ap.add_argument("--start", type=int, default=0)
    ap.add_argument("--balance", action="store_true", help="with --strips: rebalance cuts from per-rank times")
    ap.add_argument("--strips", default="",
                    help="emulate N sharded screen-strip ranks on this GPU: per-rank stage-1 "
                         "(footprint discretization) and stage-2 (mips + strip render) event times")
    a = ap.parse_args()
    import torch
    from paper_2201_10887_b200 import _cuda, _engine, build_influence_table
    from paper_2201_10887_b200.configs import CONFIGS
    from paper_2201_10887_b200.render import enqueue_frame
    cfg = CONFIGS[a.config]
    g = cfg.grid()
    t = build_influence_table(g, cfg.sigma)
    st = cfg.settings()
    mk = lambda: torch.cuda.Event(enable_timing=True)
    for n_strips in [int(x) for x in a.strips.split(",") if x]:
        from paper_2201_10887_b200 import multi
        bal = multi.StripBalancer(cfg.width, n_strips)
        rects = bal.rects
        rows = []
        for i in range(a.frames):
            if a.balance and rows:
                # every rank's time of the previous frame (in a real run: exchanged in the
                # frame's all-reduce, used LAG frames later)
                rects = bal.update([d + r for d, r, _ in rows[-1]])
            fc = cfg.path_frame_config(a.start + i)
            evs = [[mk() for _ in range(4)] for _ in rects]
            for e4 in evs:
                for e in e4:
                    e.record()
            fr = [multi.StripFrame(fc, g, t, st, rects, r, slot=r, events=_engine.event_handles(evs[r]))
                  for r in range(n_strips)]
            for f in fr:
                f.stage1()
            torch.cuda.synchronize()
            red = fr[0].xchg.clone()
            for f in fr[1:]:
                torch.maximum(red, f.xchg, out=red)
            for f in fr:
                f.xchg.copy_(red)
            for f in fr:
                f.stage2()
            torch.cuda.synchronize()
            rows.append([(e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3]),
                          int(f.buf.counters[_cuda.CNT_PAIRS])) for e, f in zip(evs, fr)])
        mean = lambda xs: sum(xs) / len(xs)
        per = [max(d + r for d, r, _ in row) for row in rows]
        out = {"strips": n_strips, "balanced": bool(a.balance), "rects": rects,
               "max_rank_ms_per_frame": [round(x, 4) for x in per],
               "discretize_ms": [round(mean([r[k][0] for r in rows]), 4) for k in range(n_strips)],
               "render_ms": [round(mean([r[k][1] for r in rows]), 4) for k in range(n_strips)],
               "pairs": [mean([r[k][2] for r in rows]) for k in range(n_strips)]}
        print(json.dumps(out), flush=True)
    if a.strips:
        return
    ev = [[mk() for _ in range(4)] for _ in range(a.frames)]
    for e4 in ev:
        for e in e4:
            e.record()
    torch.cuda.synchronize()
    cnt = []
    for i in range(a.frames):
        buf, plan, _ = enqueue_frame(cfg.path_frame_config(a.start + i), g, t, st, events=_engine.event_handles(ev[i]))
        cnt.append(buf.counters.clone())
    torch.cuda.synchronize()
    mean = lambda xs: sum(xs) / len(xs)
    names = ("discretize", "mip_top", "render")
    out = {n: round(mean([e[j].elapsed_time(e[j + 1]) for e in ev]), 4) for j, n in enumerate(names)}
    c = torch.stack(cnt).double().mean(0).tolist()
    out["pairs"] = c[_cuda.CNT_PAIRS]
    out["valid_texels"] = c[_cuda.CNT_VALID]
    out["node_visits"] = c[_cuda.CNT_NODE_VISITS]
    print(json.dumps(out))


if __name__ == "__main__":
    main()

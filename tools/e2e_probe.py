"""Dev probe: where does an end-to-end frame of `render_frames` go?

Prints wall ms/frame for several pipeline depths, with and without the bench's
L2 flush, the host time spent inside the API per frame (enqueue vs finish), and
the device time of a lone frame.  python tools/e2e_probe.py [--config C2]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2201_10887_b200 import configs, render as R  # noqa: E402
from paper_2201_10887_b200.rbf import RbfParams  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--frames", type=int, default=200)
    a = ap.parse_args()
    cfg = configs.CONFIGS[a.config]
    g, table, _ = bench.build_inputs(cfg)
    st, P = cfg.settings(), RbfParams(cfg.sigma)
    dev = torch.device("cuda", 0)
    g.device_view(dev).influence(table)
    fc = cfg.frame_config(0)
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
    seq = [fc] * a.frames
    for _ in R.render_frames(seq[:8], g, table, P, st):
        pass
    torch.cuda.synchronize()

    # host cost of the API calls, split
    enq, fin = [], []
    orig_enq, orig_fin = R.enqueue_frame, R._finish_pending

    def t_enq(*x, **k):
        t = time.perf_counter()
        r = orig_enq(*x, **k)
        enq.append(time.perf_counter() - t)
        return r

    def t_fin(*x, **k):
        t = time.perf_counter()
        r = orig_fin(*x, **k)
        fin.append(time.perf_counter() - t)
        return r

    import gc
    for depth, fl in [(d, f) for d in (1, 2, 3, 4, 5, 6, 8) for f in (False, True)] * 3:
        if True:
            bf = (lambda i: flush.zero_()) if fl else None
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in R.render_frames(seq, g, table, P, st, before_frame=bf, depth=depth):
                pass
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) * 1e3 / len(seq)
            print(f"depth {depth} flush {int(fl)}: {ms:.4f} ms/frame  {1e3 / ms:.1f} frames/s  "
                  f"gc {gc.get_count()}", flush=True)

    R.enqueue_frame, R._finish_pending = t_enq, t_fin
    for _ in R.render_frames(seq, g, table, P, st, depth=3):
        pass
    R.enqueue_frame, R._finish_pending = orig_enq, orig_fin
    torch.cuda.synchronize()
    enq.sort()
    fin.sort()
    print(f"host enqueue_frame median {enq[len(enq) // 2] * 1e3:.4f} ms, finish median "
          f"{fin[len(fin) // 2] * 1e3:.4f} ms")

    # host busy time: the loop minus the time blocked in the read-back waits
    waits = []
    orig_sync = torch.cuda.Event.synchronize

    def t_sync(self):
        t = time.perf_counter()
        orig_sync(self)
        waits.append(time.perf_counter() - t)

    torch.cuda.Event.synchronize = t_sync
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in R.render_frames(seq, g, table, P, st, depth=3):
        pass
    wall = time.perf_counter() - t0
    torch.cuda.Event.synchronize = orig_sync
    print(f"depth 3: wall {wall * 1e3 / len(seq):.4f} ms/frame, blocked {sum(waits) * 1e3 / len(seq):.4f}, "
          f"host busy {(wall - sum(waits)) * 1e3 / len(seq):.4f} ms/frame")
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in R.render_frames(seq, g, table, P, st, depth=3):
        pass
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)

    # device time of lone frames
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(20):
        flush.zero_()
        e0.record()
        R.enqueue_frame(fc, g, table, st)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"lone frame device median {ts[len(ts) // 2]:.4f} ms")

    # back-to-back frames on one stream, no host waits, no flush
    torch.cuda.synchronize()
    e0.record()
    for i in range(a.frames):
        R.enqueue_frame(fc, g, table, st)
    e1.record()
    t0 = time.perf_counter()
    e1.synchronize()
    print(f"one stream back to back: {e0.elapsed_time(e1) / a.frames:.4f} ms/frame device")


if __name__ == "__main__":
    main()

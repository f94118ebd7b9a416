"""A/B timing of libheightcast_cuda variants on one config (dev tool, GPU box).

    python tools/ab_render.py --config C2 lib1.so lib2.so ...

For each library (loaded via HC_LIB_PATH in a subprocess) prints the mean
per-kernel event times over N frames and a hash of the frame's pixels, so
variants can be compared for speed and for identical output.
"""

import argparse
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(cfg_name, frames, selftest):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2201_10887_b200 import _cuda, build_influence_table
    from paper_2201_10887_b200.configs import CONFIGS
    from paper_2201_10887_b200.render import enqueue_frame
    cfg = CONFIGS[cfg_name]
    g = cfg.grid()
    t = build_influence_table(g, cfg.sigma)
    fc, st = cfg.frame_config(), cfg.settings()
    out = {"lib": _cuda.LIB_PATH}
    if selftest:
        mm = torch.zeros(1, dtype=torch.int64, device="cuda")
        _cuda.check(_cuda.lib().hc_selftest_division(selftest, 12345, mm.data_ptr(), _cuda.stream_ptr()), "selftest")
        torch.cuda.synchronize()
        out["division_mismatches"] = int(mm.item())
        out["division_pairs"] = selftest
    for _ in range(3):
        enqueue_frame(fc, g, t, st)
    torch.cuda.synchronize()
    d, m, r = [], [], []
    for _ in range(frames):
        buf, _plan, _ms = enqueue_frame(fc, g, t, st)
        buf.ev[2].synchronize()
        d.append(buf.ev[0].elapsed_time(buf.ev[1]))
        m.append(buf.ev[1].elapsed_time(buf.ev[4]))
        r.append(buf.ev[4].elapsed_time(buf.ev[2]))
    # pipelined sequence (the e2e path): 200 frames through render_frames, L2 flush per frame
    import time
    from paper_2201_10887_b200 import render_frames
    from paper_2201_10887_b200.rbf import RbfParams
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    for _ in render_frames([fc] * 16, g, t, RbfParams(cfg.sigma), st):
        pass
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in render_frames([fc] * 200, g, t, RbfParams(cfg.sigma), st, before_frame=lambda i: flush.zero_()):
        pass
    out["pipelined_ms"] = (time.perf_counter() - t0) * 1e3 / 200
    out.update({"discretize_ms": sum(d) / len(d), "maxmip_ms": sum(m) / len(m), "render_ms": sum(r) / len(r),
                "render_min_ms": min(r),
                "pixels_sha": hashlib.sha256(buf.rgb.cpu().numpy().tobytes()).hexdigest()[:16],
                "counters": buf.counters.cpu().tolist()})
    print("RESULT " + json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--frames", type=int, default=10)
    ap.add_argument("--selftest", type=int, default=0)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("libs", nargs="*")
    a = ap.parse_args()
    if a.child:
        child(a.config, a.frames, a.selftest)
        return
    for lib in a.libs or [""]:
        env = dict(os.environ)
        if lib:
            env["HC_LIB_PATH"] = os.path.abspath(lib)
        p = subprocess.run([sys.executable, __file__, "--child", "--config", a.config, "--frames", str(a.frames),
                            "--selftest", str(a.selftest)], env=env, capture_output=True, text=True)
        res = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
        print(res[0][7:] if res else f"FAILED {lib}: {p.stderr[-2000:]}", flush=True)


if __name__ == "__main__":
    main()

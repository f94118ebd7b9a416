"""Time the reference package itself (pkg/src/heightcast, numpy + Numba) on the
host cores, for a few frames of a benchmark config's camera path.

    python tools/ref_package_timing.py --config C2 --frames 3 > profiles/r2_reference_package_c2.json

Needs the unmodified reference installed under baseline/_ref (git-ignored, it
travels to the GPU box):
    python -m pip install --no-index --no-build-isolation --no-deps \
        --find-links /opt/wheelhouse --target baseline/_ref <copy of /root/reference/pkg>

The reference hard-codes K = 3 cascades (cascade.py:345-360), so the frames are
the config's camera path with 3 cascades of the config's resolution; its grid
comes from its own generator (same cells as ours, pinned in tests/golden), its
influence table from its own scipy build.  Output: one JSON line.
"""

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--frames", type=int, default=3)
    a = ap.parse_args()
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_hcref")
    import numba
    import heightcast as ref
    sys.path.insert(0, ROOT)
    from paper_2201_10887_b200.configs import CONFIGS
    cfg = CONFIGS[a.config]
    t0 = time.perf_counter()
    ref.synth._MAX_DEPTH = cfg.max_depth if cfg.max_depth is not None else 6
    g = ref.generate_synthetic(cfg.kind, cfg.seed, cfg.cells)
    t1 = time.perf_counter()
    table = ref.build_influence_table(g, cfg.sigma)
    t2 = time.perf_counter()
    params = ref.RbfParams(sigma=cfg.sigma)
    st = ref.CascadeSettings(resolution=cfg.resolution, overlap="auto")

    def frame(i):
        c = cfg.path_camera(i)
        cam = ref.CameraView(eye=c.eye, look_dir=c.look_dir, up=c.up, fov_y=c.fov_y, aspect=c.aspect,
                             near_clip=c.near_clip, far_clip=c.far_clip)
        fc = ref.FrameConfig(width=cfg.width, height=cfg.height, camera=cam)
        s = time.perf_counter()
        fr = ref.render_frame(fc, g, table, params, st)
        return time.perf_counter() - s, fr

    warm, _ = frame(0)                    # Numba JIT (cached afterwards) + page-in
    times, phases = [], []
    for i in range(a.frames):
        dt, fr = frame(i)
        times.append(dt)
        phases.append((fr.approximation_ms, fr.raycast_ms))
    per = statistics.median(times)
    print(json.dumps({
        "impl": "reference package (pkg/src/heightcast, unmodified, numpy + Numba)",
        "config": cfg.name, "cascades": 3, "cascade_res": cfg.resolution, "image": [cfg.width, cfg.height],
        "frames_timed": a.frames, "s_per_frame_median": per, "frames_per_s": 1.0 / per,
        "s_per_frame": times, "first_frame_s_incl_jit": warm,
        "phases_ms_median": {"approximation_ms": statistics.median(p[0] for p in phases),
                             "raycast_ms": statistics.median(p[1] for p in phases)},
        "numba_threads": numba.get_num_threads(), "host_cpus": os.cpu_count(),
        "startup_s": {"synth": round(t1 - t0, 2), "influence_table": round(t2 - t1, 2)},
    }))


if __name__ == "__main__":
    main()

"""Benchmark: frames/s of the B200 heightcast hot path (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step renders one full frame of the configuration (C2 by default: 100k-cell
adaptive quadtree, 4 cascades of 1024^2, 1920x1080) -- host cascade planning,
GPU mask + RBF discretization, max mipmaps, ray casting and shading.
`value`  : frames/s with the grid resident in HBM, each step timed with CUDA
           events on the launching stream (host planning included, since the GPU
           waits for it), L2 flushed (256 MiB write) between timed steps.
`e2e`    : frames/s through the public API `render_frames(...)` (every frame
           host-planned, kernel descriptors copied host->device as launch
           parameters, pixels read back into pinned host memory on a copy stream
           overlapping the next frame), host wall clock over the K frames.
`roofline`: the dominant kernel's algorithmic work per launch / its mean event
           duration vs MEASURED_PEAKS.json (see DESIGN.md for the unit models).
`cpu_baseline`: the float64 C oracle port of the reference pipeline
           (oracle/, OpenMP over all host cores) on rank 0, bounded sample.
N>1: one process per GPU (torchrun).  C1-C4: each rank renders its own camera
view of the same grid (view sharding, no data-path collective): weak scaling.
C5: screen strips of one frame (strong scaling): each rank discretizes its
strip's footprint, one NCCL MAX all-reduce exchanges the level-5 mips and valid
partials, each rank traces its strip; e2e gathers the image to rank 0.  The
reported value is total frames/s, timed as the max over ranks.
`--impl reference`: times the oracle port of the reference's CPU pipeline on
the host cores (rank 0 only) for the same config/metric.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2201_10887_b200.configs import PATH_FRAMES  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "ncu_r2.json")
B200_SMS = 148
MUFU_PER_SM_CLK = 16          # ex2 lanes per SM per clock (SURVEY.md §8 d)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="cpu_baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def load_peaks():
    try:
        with open(PEAKS_PATH) as fh:
            p = json.load(fh)
        return p, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def l2_bandwidth_gbs(dev):
    """L2 read bandwidth: one launch of hc_bench_l2_read streaming a 32 MiB buffer
    (L2-resident, 126 MB L2) 64 times, best of 5, CUDA events.  The secondary
    roofline of the max-mip builder, whose inputs the discretization has just
    written (SURVEY.md §8 d)."""
    import torch
    from paper_2201_10887_b200 import _cuda
    n = 32 << 20
    passes = 64
    buf = torch.ones(n // 4, dtype=torch.float32, device=dev)
    sink = torch.zeros(1, dtype=torch.float32, device=dev)
    lib = _cuda.lib()
    run = lambda: _cuda.check(lib.hc_bench_l2_read(buf.data_ptr(), n, passes, sink.data_ptr(),
                                                    _cuda.stream_ptr()), "hc_bench_l2_read")
    run()
    best = float("inf")
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return passes * n / (best * 1e-3) / 1e9


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed region.

    NVML polled from a background thread every ~1 ms (the timed region of a default
    run is only milliseconds long, too short for `nvidia-smi -lms`), plus one sample
    at entry and one at exit; falls back to a single nvidia-smi query."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index: int):
        self.index = index
        self.rows = []              # (sm_mhz, reasons bitmask)
        self.max_mhz = None
        self.nvml = None
        self.handle = None
        self.stop = threading.Event()
        self.thread = None

    def _open(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        self.nvml = pynvml
        try:
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            self.handle = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM))

    def _sample(self):
        n = self.nvml
        self.rows.append((float(n.nvmlDeviceGetClockInfo(self.handle, n.NVML_CLOCK_SM)),
                          int(n.nvmlDeviceGetCurrentClocksEventReasons(self.handle))))

    def _loop(self):
        while not self.stop.wait(0.001):
            try:
                self._sample()
            except Exception:
                return

    def __enter__(self):
        try:
            self._open()
            self._sample()
            self.thread = threading.Thread(target=self._loop, daemon=True)
            self.thread.start()
        except Exception:
            self.nvml = None
        return self

    def __exit__(self, *exc):
        if self.nvml is not None:
            self.stop.set()
            self.thread.join(timeout=5)
            try:
                self._sample()
            except Exception:
                pass
        return False

    def _smi_fallback(self):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20)
            sm, mx = [float(x) for x in out.stdout.strip().split(",")[:2]]
            return {"sm_mhz": sm, "sm_max_mhz": mx, "reasons": ["sampled after the timed region (nvidia-smi)"]}
        except Exception:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}

    def summary(self):
        if not self.rows:
            return self._smi_fallback()
        n = self.nvml
        mask = 0
        for _, r in self.rows:
            mask |= r
        reasons = sorted(name for name, attr in self.REASONS if mask & int(getattr(n, attr, 0)))
        return {"sm_mhz": statistics.median(sm for sm, _ in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml"}


def build_inputs(cfg):
    from paper_2201_10887_b200 import build_influence_table
    t0 = time.perf_counter()
    g = cfg.grid()
    t1 = time.perf_counter()
    table = build_influence_table(g, cfg.sigma)
    t2 = time.perf_counter()
    return g, table, {"synth_s": round(t1 - t0, 2), "influence_table_s": round(t2 - t1, 2)}


def cpu_frames(cfg, g, table, budget_s, max_frames=None):
    """Oracle (reference CPU port) frames along the benchmark camera path (frame i
    renders path pose i, as the GPU arm's step i does): returns (frames/s, last
    frame's stats, n, median s/frame).

    Every frame is planned by the numpy restatement of the reference planner
    (oracle/plan_numpy.py) inside the timed frame, then discretized, ray cast and
    shaded by the float64 C oracle -- no code of the B200 path runs."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import heightcast_oracle as O
    import plan_numpy as PN
    from paper_2201_10887_b200.rbf import RbfParams
    O.build()
    P = RbfParams(sigma=cfg.sigma)
    st = cfg.settings()

    def frame(i):
        fc = cfg.path_frame_config(i)
        c = fc.camera
        cam = PN.CameraView(eye=c.eye, look_dir=c.look_dir, up=c.up, fov_y=c.fov_y, aspect=c.aspect,
                            near_clip=c.near_clip, far_clip=c.far_clip)
        tp = time.perf_counter()
        plan = PN.plan_cascades(cam, g, st.resolution, st.overlap, st.count)
        plan_ms = (time.perf_counter() - tp) * 1e3
        _, stats = O.render_frame(fc, g, table, P, st, plan=plan)
        stats["plan_ms"] = plan_ms
        return stats

    frame(0)                                            # warm (page-in, thread pool)
    times, stats = [], None
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        stats = frame(len(times))
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start >= budget_s or (max_frames and len(times) >= max_frames):
            break
    per = statistics.median(times)
    return 1.0 / per, stats, len(times), per


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    # CPU only: the grid from the generator, the influence table from the oracle's
    # scipy builder (the reference's algorithm), nothing on the GPU
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import heightcast_oracle as O
    g = cfg.grid(native_paint=False)        # numpy tile painter: libheightcast_cuda stays unmapped
    table = O.build_influence_table(g, cfg.sigma)
    # K frames along the camera path, bounded to ~2 minutes of CPU time (C3/C4 frames
    # take seconds each)
    fps, stats, n, per = cpu_frames(cfg, g, table, budget_s=120.0, max_frames=args.steps)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    line = {
        "impl": "reference", "metric": "frames/sec", "value": fps, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "frames_timed": n, "warmup": args.warmup, "ms_per_step": per * 1e3,
        "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(cfg, g, table, args.gpus),
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": "port",
                         "sample": f"{n} full {cfg.name} frames along the camera path (float64 C oracle of the "
                                   f"reference pipeline, OpenMP {cores} threads), median"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "phases_ms": {k: round(stats[k], 3) for k in ("plan_ms", "approximation_ms", "raycast_ms")},
        "native_so_loaded": mapped_repo_libraries(),
    }
    print(json.dumps(line), flush=True)


def bench_config(cfg, g, table, n_gpus):
    """`config` of both arms' JSON lines: the same dict for the same workload."""
    d = cfg.workload(g, table)
    d["parallelism"] = f"{'screen strips' if cfg.name == 'C5' else 'view-sharded'} x{n_gpus}"
    d["l2"] = "GPU arm: 256 MiB L2 flush (int32 fill) between timed steps; CPU arm: none"
    return d


def mapped_repo_libraries():
    """Shared objects under this repository mapped into the process (/proc/self/maps):
    the reference arm must show only the oracle's library."""
    out = set()
    try:
        with open("/proc/self/maps") as fh:
            for line in fh:
                path = line.split()[-1] if len(line.split()) >= 6 else ""
                if path.endswith(".so") and path.startswith(ROOT + os.sep):
                    out.add(os.path.relpath(path, ROOT))
    except OSError:
        return None
    return sorted(out)


def main():
    args = parse()
    from paper_2201_10887_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun (rank 0 prints)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={29500 + os.getpid() % 1000}", os.path.abspath(__file__)]
        cmd += sys.argv[1:]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)

    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    if ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}")
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    from paper_2201_10887_b200 import _cuda, _engine
    from paper_2201_10887_b200.render import enqueue_frame
    from paper_2201_10887_b200.rbf import RbfParams

    from paper_2201_10887_b200 import multi

    g, table, prep = build_inputs(cfg)
    st = cfg.settings()
    P = RbfParams(sigma=cfg.sigma)
    strips = cfg.name == "C5"           # screen strips (strong scaling), else view sharding
    # step i renders frame i of the moving camera path (configs.path_camera): strips --
    # every rank the same frame; views -- rank r its own (C4: views r, r+N, ...)
    frame_of = (lambda i: cfg.path_frame_config(i)) if strips else \
        (lambda i: cfg.path_frame_config(i, rank, ws))
    rects = multi.screen_strips(cfg.width, ws) if strips else None
    rect = (rects[rank][0], 0, rects[rank][1], cfg.height) if strips else None
    t_up = time.perf_counter()
    gdev = g.device_view(dev)
    gdev.influence(table)
    torch.cuda.synchronize()
    prep["upload_s"] = round(time.perf_counter() - t_up, 3)

    # L2 flush: 256 MiB (> 126 MB L2) written with 4-byte elements (the fill kernel
    # runs at full HBM bandwidth; a byte-typed fill reaches about half of it)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # strips: cut from the ranks' measured frame times (multi.StripSequence)
    seq_strips = multi.StripSequence(cfg.width, ws, rank) if strips and ws > 1 else None

    def step(i, events=None):
        if seq_strips is not None:
            # sharded strip: footprint discretization, the one MAX all-reduce of the
            # mip exchange buffer and frame times (between events 1 and 2), upper mips +
            # the strip's rays
            f = seq_strips.frame(frame_of(i), g, table, st, events=events)
            return (f.buf, f.plan, f.plan_ms) if f.visible else None
        return enqueue_frame(frame_of(i), g, table, st, rect=rect, events=events)

    # ---- warm-up (device-resident path): the last warm-up poses of the path, so the
    # first timed frame's tile order comes from a different pose, as every later one does
    n_warm = max(args.warmup, 3)
    for i in range(-n_warm, 0):
        step(i % (2 * PATH_FRAMES))
    torch.cuda.synchronize()
    cnt_all = torch.zeros((args.steps, _cuda.N_COUNTERS), dtype=torch.int64, device=dev)

    # ---- timed: K steps, each bracketed by CUDA events (plus per-kernel events), L2
    # flushed between steps on the stream.  The host does not wait between steps, so
    # it plans and enqueues step i+1 while the GPU runs step i (stream order keeps
    # every frame's buffers consistent).
    mk = lambda: torch.cuda.Event(enable_timing=True)
    ev = [(mk(), mk()) for _ in range(args.steps)]
    kev = [[mk() for _ in range(4)] for _ in range(args.steps)]
    for k in kev:               # torch only reports elapsed times of events it has recorded once
        for e in k:
            e.record()
    kh = [_engine.event_handles(k) for k in kev]
    plan_ms_all = []
    barrier()
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record()
            buf, plan, plan_ms = step(i, kh[i])
            ev[i][1].record()
            cnt_all[i].copy_(buf.counters)       # outside the step's events (work totals)
            plan_ms_all.append(plan_ms)
        barrier()
    k_disc = [k[0].elapsed_time(k[1]) for k in kev]
    k_mip = [k[1].elapsed_time(k[2]) for k in kev]
    k_ren = [k[2].elapsed_time(k[3]) for k in kev]
    plan_ms = statistics.median(plan_ms_all)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    if ws > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    frames_per_step = 1 if strips else ws
    value = frames_per_step * args.steps / (total_ms / 1e3)

    # work per frame, averaged over the timed frames (the path changes it frame to frame)
    cnt = (cnt_all.double().mean(dim=0)).cpu().tolist()
    work = {"pairs": cnt[_cuda.CNT_PAIRS], "node_visits": cnt[_cuda.CNT_NODE_VISITS],
            "patch_tests": cnt[_cuda.CNT_PATCH_TESTS], "valid_texels": cnt[_cuda.CNT_VALID],
            "visible_texels": cnt[_cuda.CNT_VISIBLE], "rays_hit": cnt[_cuda.CNT_RAYS_HIT]}

    # ---- e2e through the public API, host wall clock: every frame planned on the host,
    # its descriptors passed to the GPU, its pixels read back into pinned host memory.
    # Views (and strips on one GPU, where the strip is the frame): render_frames
    # (frames overlap, read-back on a copy stream), an L2 flush enqueued before
    # every frame.  Strips on N > 1 GPUs: render_strip + image gather per step.
    if not strips or ws == 1:
        from paper_2201_10887_b200 import render_frames
        seq = [frame_of(i) for i in range(args.steps)]
        warm = [frame_of(i % (2 * PATH_FRAMES)) for i in range(-16, 0)]
        for _ in render_frames(warm, g, table, P, st):      # every buffer set, pinned blocks
            pass
        barrier()
        t0 = time.perf_counter()
        for _ in render_frames(seq, g, table, P, st, before_frame=lambda i: flush.zero_()):
            pass
        e2e_ms = [(time.perf_counter() - t0) * 1e3]
    else:
        def e2e_step(i):
            f = seq_strips.frame(frame_of(i), g, table, st)
            if not f.visible:
                return
            img = multi.gather_strips(f.strip().clone(), f.rects, rank, ws)
            if rank == 0:
                img.cpu()

        for i in range(-2, 0):
            e2e_step(i % (2 * PATH_FRAMES))
        barrier()
        e2e_ms = []
        for i in range(args.steps):
            flush.zero_()
            barrier()
            t0 = time.perf_counter()
            e2e_step(i)
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    barrier()
    e2e_total = sum(e2e_ms)
    if ws > 1:
        t = torch.tensor([e2e_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = frames_per_step * args.steps / (e2e_total / 1e3)

    # ---- rooflines (algorithmic work per launch / mean launch time)
    peaks, peak_kind = load_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    mufu_peak = B200_SMS * MUFU_PER_SM_CLK * sm_max * 1e6          # ex2/s = pairs/s bound
    hbm = float(peaks["hbm_gbs"])
    K = plan.n_active
    R = cfg.resolution
    off, wl, nodes = _engine.mip_shape(R)
    # k_mip_top reads level 5 and writes levels >= 6 of 2K pyramids (+ 2K x blocks partials)
    lv5 = wl[5] * wl[5] if len(wl) > 5 else 0
    above = nodes - off[6] if len(off) > 6 else 0
    top_bytes = 2 * K * (4 * (lv5 + above) + 8 * ((R + 31) // 32) ** 2)
    # HBM bytes the fused discretize writes: rasters (terrain, water f32; valid, mask u8),
    # mip levels 0..5 of both layers, patch bytes
    lv05 = off[6] if len(off) > 6 else nodes
    disc_bytes = K * R * R * 10 + 2 * K * 4 * lv05 + K * (R - 1) ** 2
    trav_bytes = 4 * work["node_visits"] + 20 * work["patch_tests"] + 3 * cfg.width * cfg.height
    mean = lambda xs: sum(xs) / len(xs)
    kernels = {
        "hc_discretize": {"ms": mean(k_disc), "bound": "sfu", "unit": "Gpairs/s",
                          "achieved": work["pairs"] / (mean(k_disc) * 1e-3) / 1e9,
                          "peak": mufu_peak / 1e9, "work_per_launch": work["pairs"],
                          "work_model": "(valid texel, influence-list entry) pairs; 1 ex2 each "
                                        "(the launch also writes rasters + mip levels 0..5)",
                          "hbm_bytes_written": disc_bytes,
                          "hbm_frac": disc_bytes / (mean(k_disc) * 1e-3) / 1e9 / hbm},
        "hc_mip_top": {"ms": mean(k_mip), "bound": "hbm", "unit": "GB/s",
                       "achieved": top_bytes / (mean(k_mip) * 1e-3) / 1e9, "peak": hbm,
                       "work_per_launch": top_bytes,
                       "work_model": "2K x 4 B x (level-5 nodes + nodes above) + 2K x 8 B x blocks "
                                     "(a ~10 us launch: latency, not bandwidth)"},
        "hc_render": {"ms": mean(k_ren), "bound": "hbm", "unit": "GB/s",
                      "achieved": trav_bytes / (mean(k_ren) * 1e-3) / 1e9, "peak": hbm,
                      "work_per_launch": trav_bytes,
                      "work_model": "4 B x node visits + 20 B x patch tests + 3 B x pixels"},
    }
    for k in kernels.values():
        k["frac"] = k["achieved"] / k["peak"]
    l2_gbs = l2_bandwidth_gbs(dev)
    kernels["hc_render"]["l2_peak_gbs"] = l2_gbs
    kernels["hc_render"]["frac_l2"] = kernels["hc_render"]["achieved"] / l2_gbs
    kernels["hc_render"]["rays_per_sec"] = 2 * cfg.width * cfg.height / (mean(k_ren) * 1e-3)
    work["pairs_per_valid_texel"] = work["pairs"] / max(work["valid_texels"], 1)
    dominant = max(kernels, key=lambda n: kernels[n]["ms"])
    # what ncu (profiles/ncu_r2.json, `ncu --set full` of this config's frame kernels)
    # says bounds each kernel: DRAM bytes per launch, issue-active, pipe utilisations
    prof = {}
    try:
        with open(PROFILE_SUMMARY) as fh:
            prof = json.load(fh).get(cfg.name, {})
    except (OSError, ValueError):
        pass
    clk_hz = None
    for name, k in kernels.items():
        if name in prof:
            k["ncu"] = prof[name]
    # issue roofline: warp instructions per unit of work from the ncu capture (per pair
    # for k_discretize, per node visit for k_render), times this run's work per launch,
    # over the live launch time, against 4 warp-instructions/clk/SM at the run's clock
    pw = prof.get("_work", {})
    unit_of = {"hc_discretize": "pairs", "hc_render": "node_visits"}
    for name, k in kernels.items():
        wi = (k.get("ncu") or {}).get("warp_instructions")
        u = unit_of.get(name)
        if wi and u and pw.get(u) and work.get(u):
            clk_hz = clk_hz or 1e6 * float(clocks.summary().get("sm_mhz") or sm_max)
            inst = wi / pw[u] * work[u]
            peak_i = B200_SMS * 4 * clk_hz
            k["issue_roofline"] = {"warp_instructions_per_launch": inst, "achieved_per_s": inst / (k["ms"] * 1e-3),
                                   "peak_per_s": peak_i, "frac": inst / (k["ms"] * 1e-3) / peak_i,
                                   "model": f"ncu warp instructions per {u} x this run's {u}"}
    d = kernels[dominant]
    nc = d.get("ncu") or {}
    roofline = {"kernel": dominant, "bound": "hbm" if d["bound"] == "hbm" else "sfu", "achieved": d["achieved"],
                "peak": d["peak"], "unit": d["unit"], "frac": d["frac"],
                "traffic": nc.get("dram_bytes"),
                "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs" if d["bound"] == "hbm"
                else f"148 SMs x 16 ex2/clk x {sm_max:.0f} MHz ({peak_kind} sm_max_mhz)"}
    if nc:
        # the ceiling the kernel actually hits, from the committed ncu capture
        pipes = {p: nc.get(p) for p in ("fp64_pipe", "xu_pipe", "fma_pipe", "lsu_pipe")}
        roofline["limiter"] = {"issue_active": nc.get("issue_active"), **pipes,
                               "occupancy": nc.get("occupancy"), "l1_hit": nc.get("l1_hit"),
                               "l2_hit": nc.get("l2_hit"), "source": f"profiles/{prof.get('_source')}"}
        if dominant == "hc_render":
            roofline["limiter"]["bound"] = "issue/latency (FP64 dependency chains)"
            roofline["limiter"]["frac_l2"] = d["frac_l2"]
        if d.get("issue_roofline"):
            roofline["limiter"]["issue_frac"] = d["issue_roofline"]["frac"]

    out = None
    if rank == 0:
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            fps, stats, n, per = cpu_frames(cfg, g, table, budget_s=args.cpu_seconds)
            cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
            cpu = {"value": fps, "unit": "frames/s", "cores": cores, "kind": "port",
                   "sample": f"{n} full {cfg.name} frames (float64 C oracle of the reference pipeline, "
                             f"OpenMP {cores} threads, ~{args.cpu_seconds:.0f} s budget), median",
                   "phases_ms": {k: round(stats[k], 3) for k in ("plan_ms", "approximation_ms", "raycast_ms")}}
        P_pix = cfg.width * cfg.height
        out = {
            "metric": "frames/sec", "value": value, "unit": "frames/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if strips else "weak",
            "vs_baseline": None, "dtype": "f64 traversal/shading, f32 RBF discretization", "data": "synthetic",
            "config": bench_config(cfg, g, table, ws),
            "rays_per_sec": value * P_pix, "layer_rays_per_sec": value * 2 * P_pix,
            "texels_per_sec": value * work["valid_texels"] / frames_per_step,
            "e2e": {"value": e2e_value, "unit": "frames/s",
                    "h2d_bytes_per_step": _frame_param_bytes(K),
                    "d2h_bytes_per_step": P_pix * 3 + 8 * _cuda.N_COUNTERS,
                    "ms_per_step": e2e_total / args.steps},
            "roofline": roofline, "kernels": kernels, "cpu_baseline": cpu,
            "clocks": clocks.summary(), "gpu_launches": _engine.LAUNCHES_PER_FRAME * args.steps,
            "work_per_frame": work,
            "phases_ms": {"plan_ms": round(plan_ms, 4), "approximation_ms": round(mean(k_disc), 4),
                          "raycast_ms": round(mean(k_mip) + mean(k_ren), 4)},
            "prep": prep,
        }
        print(json.dumps(out), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def _frame_param_bytes(K):
    import ctypes as C
    from paper_2201_10887_b200 import _cuda
    return (C.sizeof(_cuda.HcCascadeRaster) * K + C.sizeof(_cuda.HcMipJob) * 2 * K
            + C.sizeof(_cuda.HcRenderArgs))


if __name__ == "__main__":
    main()

"""Summarise ncu captures into profiles/ (run in the build container, no GPU needed).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep --tag r1_render --config C2
    python tools/ncu_summary.py --launches gpurun_out/launches.csv --tag r1_launches

Writes profiles/<tag>.md (key metrics per kernel) and merges per-launch DRAM
traffic (dram__bytes_read.sum + dram__bytes_write.sum) into
profiles/ncu_r2.json, which bench.py reports as roofline.traffic / limiter.
"""

import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__average_warp_latency_per_inst_issued.ratio", "cycles per issued inst"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp inst"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu (MUFU) pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu pipe %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__cycles_active.avg", "SM active cycles avg"),
    ("sm__cycles_active.max", "SM active cycles max"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_pipe_throttle"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard"),
]

KERNEL_KEY = {"k_render": "hc_render", "k_discretize": "hc_discretize", "k_mip_tiles": "hc_maxmip",
              "k_mip_top": "hc_mip_top"}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    return rows[0], rows[1], rows[2:]


def to_float(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def summarise(rep, tag, config, work=None):
    head, units, rows = raw_rows(rep)
    col = {c: i for i, c in enumerate(head)}
    lines = [f"# ncu --set full summary: {tag}", "", f"source: `{os.path.basename(rep)}` "
             f"(ncu --set full --clock-control none, one launch per kernel; cold-cache, serialised)", ""]
    kernels = []
    for r in rows:
        name = r[col["Kernel Name"]]
        short = name.split("(")[0].replace("hc::", "")
        kernels.append((short, r))
    lines.append("| metric | " + " | ".join(k for k, _ in kernels) + " |")
    lines.append("|---|" + "---|" * len(kernels))
    for m, label in METRICS:
        if m not in col:
            continue
        vals = []
        for _, r in kernels:
            v = r[col[m]]
            vals.append(f"{v} {units[col[m]]}".strip())
        lines.append(f"| {label} (`{m}`) | " + " | ".join(vals) + " |")
    with open(os.path.join(PROF, f"{tag}.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    # per-kernel metrics for bench.py (profiles/ncu_r2.json): DRAM traffic per launch and
    # the pipe / issue / occupancy figures that say what bounds each kernel
    path = os.path.join(PROF, "ncu_r2.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    pct = {"issue_active": "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "fp64_pipe": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "fma_pipe": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "xu_pipe": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "lsu_pipe": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
           "occupancy": "sm__warps_active.avg.pct_of_peak_sustained_active",
           "l1_hit": "l1tex__t_sector_hit_rate.pct", "l2_hit": "lts__t_sector_hit_rate.pct"}
    cfg = {"_source": f"{tag}.md (from {os.path.basename(rep)})"}
    seen = set()
    for short, r in kernels:
        key = KERNEL_KEY.get(short.replace("void ", "").split("<")[0].strip())
        if key is None or key in seen:          # first launch of each kernel
            continue
        seen.add(key)
        get = lambda m: to_float(r[col[m]]) if m in col else None
        rd = get("dram__bytes_read.sum") * scale[units[col["dram__bytes_read.sum"]]]
        wr = get("dram__bytes_write.sum") * scale[units[col["dram__bytes_write.sum"]]]
        dur = get("gpu__time_duration.sum")
        dur_us = dur * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(
            units[col["gpu__time_duration.sum"]], 1.0)
        k = {"dram_bytes": rd + wr, "duration_us": round(dur_us, 2),
             "registers": get("launch__registers_per_thread"),
             "warp_instructions": get("smsp__inst_executed.sum")}
        for name, m in pct.items():
            v = get(m)
            k[name] = None if v is None else round(v / 100.0, 4)
        k["stall_long_scoreboard"] = get("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio")
        cfg[key] = k
    if work:
        # the profiled frame's work counters (tools/frames.py output over the same
        # frames): bench.py scales instructions per unit of work to its own frames
        cfg["_work"] = {k: work[k] for k in ("pairs", "valid_texels", "node_visits") if k in work}
    data[config] = cfg
    with open(path, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)
    print("wrote", os.path.join(PROF, f"{tag}.md"), {k: v["dram_bytes"] for k, v in cfg.items() if k[0] != "_"})


def launches(csv_path, tag):
    rows = list(csv.reader(open(csv_path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    order = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        k = r[ki].split("(")[0]
        if k not in agg:
            order.append(k)
        agg[k].append(to_float(r[vi]) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3,
                                          "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0))
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# launch list: {tag}", "", f"source: `{os.path.basename(csv_path)}` "
             "(ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)", "",
             "| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
    for k in sorted(order, key=lambda k: -sum(agg[k])):
        v = agg[k]
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} | {sum(v) / tot:.1%} |")
    with open(os.path.join(PROF, f"{tag}.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("wrote", os.path.join(PROF, f"{tag}.md"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep", nargs="?")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--launches")
    ap.add_argument("--frames-log", help="tools/frames.py output of the profiled command (work counters)")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        launches(a.launches, a.tag)
    if a.rep:
        work = None
        if a.frames_log:
            lines = [l for l in open(a.frames_log) if l.startswith("{")]
            work = json.loads(lines[-1]) if lines else None
        summarise(a.rep, a.tag, a.config, work)


if __name__ == "__main__":
    main()

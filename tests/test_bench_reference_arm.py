"""bench.py's reference arm (`--impl reference`) runs on the CPU alone; its JSON line
keeps the driver's contract (metric/unit of the GPU arm, impl, cpu_baseline, e2e
with zero copy bytes)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_contract():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "0", "--config", "C1"], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "frames/sec" and d["unit"] == "frames/s"
    assert d["higher_is_better"] is True and d["value"] > 0 and d["steps"] == 2
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("C1")
    # the arm runs oracle code only: the product library is never mapped (/proc/self/maps)
    assert d["native_so_loaded"] == ["oracle/liboracle.so"], d["native_so_loaded"]


def test_both_arms_share_config_and_camera_path():
    """The GPU arm's and the reference arm's `config` dicts are built by the same
    function; the camera path moves every frame (cli.py:127-131)."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2201_10887_b200.configs import CONFIGS, PATH_FRAMES
    cfg = CONFIGS["C2"]
    a = bench.bench_config(cfg, None, None, 1)
    b = bench.bench_config(cfg, None, None, 1)
    assert a == b and a["camera_path"]
    eyes = [cfg.path_camera(i).eye for i in range(2 * PATH_FRAMES + 1)]
    assert eyes[0] == eyes[2 * PATH_FRAMES] == cfg.eye
    assert all(eyes[i] != eyes[i + 1] for i in range(2 * PATH_FRAMES))
    # view sharding: ranks see different poses of the same step
    assert cfg.path_camera(5, 0, 2).eye != cfg.path_camera(5, 1, 2).eye
    c4 = CONFIGS["C4"]
    assert {c4.path_camera(i, r, 4).eye for i in range(16) for r in range(4)} == \
        {c4.camera(v).eye for v in range(64)}

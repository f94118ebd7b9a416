"""CLI: formats and exit codes compatible with the reference's cli.py."""

import io
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_2201_10887_b200", *args], capture_output=True, text=True,
                          cwd=cwd or ROOT)


def test_synth_writes_reference_ahf(tmp_path):
    from paper_2201_10887_b200 import load_grid, synth
    out = tmp_path / "g.ahf"
    r = _run("synth", "hill", "--seed", "42", "--cells", "300", "-o", str(out))
    assert r.returncode == 0 and "wrote" in r.stderr
    g = synth.generate_synthetic("hill", 42, 300)
    buf = io.StringIO()
    g.save(buf)
    assert out.read_text() == buf.getvalue()
    h = load_grid(str(out))
    assert np.array_equal(h.centers, g.centers) and np.array_equal(h.terrain, g.terrain)


def test_bad_scene_exit_code(tmp_path):
    sc = tmp_path / "bad.txt"
    sc.write_text("synth = hill\nnear = 5\nfar = 1\n")
    r = _run("render", str(sc), "-o", str(tmp_path / "x.ppm"))
    assert r.returncode == 1 and "far" in r.stderr


@pytest.mark.gpu
def test_render_and_benchmark_commands(tmp_path, cuda):
    from paper_2201_10887_b200 import render_frame, scene
    from helpers import demo_setup
    from paper_2201_10887_b200.rbf import RbfParams
    sc = scene.demo_scene()
    path = tmp_path / "demo.txt"
    path.write_text(scene.serialize_scene(sc))
    out = tmp_path / "demo.ppm"
    r = _run("render", str(path), "-o", str(out), "--dump-cascades", str(tmp_path / "c.txt"),
             "--dump-raster", "2:water", str(tmp_path / "r.pgm"))
    assert r.returncode == 0, r.stderr
    assert r.stdout.startswith("approximation_ms=") and "raycast_ms=" in r.stdout
    data = out.read_bytes()
    header = f"P6\n{sc.width} {sc.height}\n255\n".encode()
    assert data.startswith(header)
    _, g, t, cfg, st = demo_setup()
    want = render_frame(cfg, g, t, RbfParams(sigma=sc.sigma), st).pixels
    assert data[len(header):] == want.tobytes()
    assert (tmp_path / "c.txt").read_text().startswith("# cascade polygons\n")
    assert (tmp_path / "r.pgm").read_bytes().startswith(f"P5\n{sc.cascade_res} {sc.cascade_res}\n65535\n".encode())
    r = _run("benchmark", str(path), "--frames", "3", "--pose2", "400", "280", "260", "1050", "1150", "40")
    lines = r.stdout.strip().splitlines()
    assert r.returncode == 0 and lines[0] == "frame,approximation_ms,raycast_ms,visible_texels,rays_hit"
    assert len(lines) == 5 and lines[-1].startswith("median,")

"""CPU checks of the native library boundary and host logic (no GPU needed)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol(native_lib_path):
    hdr = open(os.path.join(ROOT, "include", "heightcast.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(hc_\w+)\s*\(", hdr, flags=re.M))
    assert {"hc_render", "hc_discretize", "hc_maxmip", "hc_traverse_batch"} <= declared
    lib = C.CDLL(native_lib_path)
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    from paper_2201_10887_b200 import _cuda
    assert set(_cuda.EXPORTS) == declared
    lib.hc_abi_version.restype = C.c_int
    assert lib.hc_abi_version() == _cuda.HC_ABI_VERSION


def test_struct_layouts_match_header_sizes(native_lib_path):
    """ctypes mirrors of the ABI structs: field offsets follow C alignment rules."""
    from paper_2201_10887_b200 import _cuda
    assert C.sizeof(_cuda.HcCascadeRaster) == 8 * 3 + 4 * 2 + 8 * 160 + 8 * 4
    assert C.sizeof(_cuda.HcMipJob) == 8 * 6 + 4 * 2 + 8 * 20 + 4 * 20
    assert _cuda.HcRenderArgs.c.offset % 8 == 0 and _cuda.HcRenderArgs.dbg.offset % 8 == 0


def test_argument_validation_without_gpu(native_lib_path):
    """Invalid descriptors are rejected before any CUDA call (works with no device)."""
    from paper_2201_10887_b200 import _cuda
    L = _cuda.lib()
    d = (_cuda.HcCascadeRaster * 1)()
    d[0].resolution = 2          # < 4
    g = _cuda.HcGrid()
    assert L.hc_discretize(d, 1, C.byref(g), C.c_float(0.0), None, None) == _cuda.HC_EINVAL
    assert b"resolution" in L.hc_last_error()
    assert L.hc_discretize(d, 99, C.byref(g), C.c_float(0.0), None, None) == _cuda.HC_EINVAL
    a = _cuda.HcRenderArgs()
    assert L.hc_render(C.byref(a), None) == _cuda.HC_EINVAL
    assert L.hc_render_tiles(0, 0, 1920, 1080) == 240 * 270
    assert L.hc_render_order_words(0, 0, 1920, 1080) == 240 * 270 + 32 * 16
    assert L.hc_maxmip_workspace_bytes(8, 1024) == 8 * 32 * 32 * 2 * 4


def test_product_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import heightcast_oracle as O
    from paper_2201_10887_b200 import render_frame, scene
    from paper_2201_10887_b200._cuda import HeightcastCudaError
    from paper_2201_10887_b200.rbf import RbfParams
    sc = scene.demo_scene()
    g = scene.scene_grid(sc)
    t = O.build_influence_table(g, 1.0)
    with pytest.raises(HeightcastCudaError):
        render_frame(scene.scene_frame_config(sc), g, t, RbfParams(), scene.scene_settings(sc))


def test_scene_roundtrip_and_errors():
    from paper_2201_10887_b200 import scene
    sc = scene.demo_scene()
    txt = scene.serialize_scene(sc)
    assert scene.parse_scene(txt) == sc
    with pytest.raises(scene.SceneError, match="far"):
        scene.parse_scene("synth = hill\nnear = 5\nfar = 1\n")
    with pytest.raises(scene.SceneError, match="duplicate"):
        scene.parse_scene("synth = hill\nseed = 1\nseed = 2\n")


def test_grid_load_save_roundtrip_and_errors(tmp_path):
    from paper_2201_10887_b200 import grid as G, synth
    g = synth.generate_synthetic("hill", 3, 300)
    p = tmp_path / "g.ahf"
    g.save(str(p))
    h = G.load_grid(str(p))
    assert np.array_equal(g.centers, h.centers) and np.array_equal(g.tile_index, h.tile_index)
    with pytest.raises(G.GridFormatError, match="non-power-of-two"):
        G.load_grid("AHF 1\ndomain 0 0 8 8\nmin_cell 2\ncells 1\n1.5 1.5 3 0 0\n")
    with pytest.raises(G.GridFormatError, match="line 6"):
        G.load_grid("AHF 1\ndomain 0 0 8 8\nmin_cell 8\ncells 1\n4 4 8 100 0\ngarbage\n")
    one = G.load_grid("AHF 1\ndomain 0 0 8 8\nmin_cell 8\ncells 1\n4 4 8 100 0\n")
    assert one.height_range == (100.0, 100.0)
    with pytest.raises(G.GridFormatError, match="overlap"):
        G.load_grid("AHF 1\ndomain 0 0 8 8\nmin_cell 2\ncells 2\n2 2 4 1 0\n3 3 2 1 0\n")


def test_influence_table_two_cells_boundary():
    """SPEC: two size-1 cells 4 apart, sigma=1 -> mutual inclusion (boundary inclusive)."""
    from paper_2201_10887_b200 import grid as G
    g = G.AdaptiveGrid(G.Rect(0, 0, 8, 1), 1.0, [[0.5, 0.5], [4.5, 0.5]], [1.0, 1.0], [0.0, 10.0], [0.0, 0.0])
    import heightcast_oracle as O
    t = O.build_influence_table(g, 1.0)
    assert list(t.influencers(0)) == [0, 1] and list(t.influencers(1)) == [0, 1]


def test_struct_field_offsets_match_c_compiler(tmp_path):
    """Every ctypes field offset and struct size equals gcc's offsetof/sizeof on include/heightcast.h."""
    import shutil
    import subprocess
    from paper_2201_10887_b200 import _cuda
    cc = shutil.which("gcc") or "/usr/bin/gcc"
    structs = [getattr(_cuda, n) for n in dir(_cuda)
               if n.startswith("Hc") and isinstance(getattr(_cuda, n), type)
               and issubclass(getattr(_cuda, n), C.Structure)]
    assert len(structs) >= 10
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "heightcast.h"', "int main(void) {"]
    want = []
    for S in structs:
        lines.append(f'printf("%zu\\n", sizeof({S.__name__}));')
        want.append(C.sizeof(S))
        for name, *_ in S._fields_:
            lines.append(f'printf("%zu\\n", offsetof({S.__name__}, {name}));')
            want.append(getattr(S, name).offset)
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([cc, "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()]
    assert got == want

"""Native AHF parser (hc_ahf_parse) against the Python restatement of load_grid
(grid.py:236-331): same grids, same GridFormatError messages and line numbers."""

import numpy as np
import pytest

from paper_2201_10887_b200.grid import GridFormatError, _load_grid_text, load_grid
from paper_2201_10887_b200.synth import generate_synthetic

GOOD = "AHF 1\ndomain 0 0 8 8\nmin_cell 4\ncells 4\n2 2 4 10 0\n6 2 4 11 0.5\n2 6 4 12 0\n6 6 4 13 1.25\n"


def _same(a, b):
    assert (a.domain.xmin, a.domain.ymin, a.domain.xmax, a.domain.ymax) == \
        (b.domain.xmin, b.domain.ymin, b.domain.xmax, b.domain.ymax)
    assert a.min_cell_size == b.min_cell_size
    for x, y in ((a.centers, b.centers), (a.sizes, b.sizes), (a.terrain, b.terrain),
                 (a.water_depth, b.water_depth)):
        assert np.array_equal(np.asarray(x).view(np.uint64), np.asarray(y).view(np.uint64))


def _outcome(fn, text):
    try:
        # bytes for load_grid: a str without a newline would be read as a path
        return ("ok", fn(text.encode("ascii") if fn is load_grid else text))
    except GridFormatError as e:
        return ("err", str(e), e.line)


@pytest.mark.parametrize("text", [
    GOOD,
    GOOD.replace("\n", "\r\n"),
    GOOD.replace("\n", "\r"),
    "# comment\n\n  " + GOOD.replace("cells 4", "  cells  +0_4 ") + "\n# trailing\n\n",
    GOOD.replace("2 2 4 10 0", "2.0 2e0 4_0e-1_0 1.0e1 -0.0").replace("min_cell 4", "min_cell 0.4e1"),
    GOOD.replace("6 6 4 13 1.25", "6 6 4 inf NaN").replace("domain 0 0 8 8", "domain -0 .0 8. +8"),
    GOOD.replace("\n", "\x0b", 2),
    GOOD.replace("\n", "\x1c\n", 1),
])
def test_native_parser_matches_python_on_valid_text(text):
    a, b = _outcome(load_grid, text), _outcome(_load_grid_text, text)
    assert a[0] == b[0], (a, b)
    if a[0] == "ok":
        _same(a[1], b[1])
    else:
        assert a[1:] == b[1:]


@pytest.mark.parametrize("text", [
    "",
    "\n\n",
    "AHF 2\n",
    "AHF 1\ndomain 0 0 8\n",
    "AHF 1\ndomain 0 0 8 x\n",
    "AHF 1\ndomain 0 0 0 8\n",
    "AHF 1\ndomain 0 0 8 8\nmin_cell\n",
    "AHF 1\ndomain 0 0 8 8\nmin_cell 1__0\n",
    "AHF 1\ndomain 0 0 8 8\nmin_cell -1\n",
    "AHF 1\ndomain 0 0 8 8\nmin_cell 4\ncells 1.5\n",
    "AHF 1\ndomain 0 0 8 8\nmin_cell 4\ncells -3\n",
    "AHF 1\ndomain 0 0 8 8\nmin_cell 4\ncells 0007\n1 1 1 1 1\n",
    "AHF 1\ndomain 0 0 8 8\nmin_cell 4\ncells 99999999999999999999999\n",
    GOOD + "2 2 4 10 0\n",
    GOOD.replace("6 2 4 11 0.5", "6 2 4 11"),
    GOOD.replace("6 2 4 11 0.5", "6 2 4 11 0x1p3"),
    GOOD.replace("6 2 4 11 0.5", "6 2 4 11 1e"),
    GOOD.replace("6 2 4 11 0.5", "6 2 4 11 _1"),
    GOOD.replace("6 2 4 11 0.5", "6 2 4 11 1_"),
    GOOD.replace("6 2 4 11 0.5", "6 2 4 11 infinit"),
])
def test_native_parser_matches_python_on_malformed_text(text):
    a, b = _outcome(load_grid, text), _outcome(_load_grid_text, text)
    assert a[0] == b[0] == "err", (a, b)
    assert a[1:] == b[1:]


def test_native_parser_round_trips_a_synthetic_grid(tmp_path):
    g = generate_synthetic("pond", 3, 2000)
    path = tmp_path / "g.ahf"
    g.save(str(path))
    text = path.read_text()
    _same(load_grid(str(path)), _load_grid_text(text))
    _same(load_grid(str(path)), g)


@pytest.mark.parametrize("kind,seed,cells", [("pond", 7, 3000), ("hill", 1, 800), ("ramp", 0, 1024)])
def test_native_tile_painter_matches_numpy(kind, seed, cells):
    g = generate_synthetic(kind, seed, cells)
    for stop in (True, False):
        a, ca = g._paint(stop)
        b, cb = g._paint_numpy(stop)
        assert np.array_equal(a, b) and ca == cb


def test_native_tile_painter_reports_overlaps_like_numpy():
    from paper_2201_10887_b200.grid import AdaptiveGrid, Rect
    centers = np.array([[2.0, 2.0], [4.0, 4.0], [6.0, 6.0], [2.0, 6.0]])
    sizes = np.array([4.0, 4.0, 4.0, 4.0])
    z = np.zeros(4)
    g = AdaptiveGrid(Rect(0, 0, 8, 8), 2.0, centers, sizes, z + 10, z, check_overlap=False)
    for stop in (True, False):
        a, ca = g._paint(stop)
        b, cb = g._paint_numpy(stop)
        assert ca == cb == (0, 1)
        assert np.array_equal(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,seed,cells,max_depth", [("pond", 7, 100_000, 7), ("pond", 11, 300_000, 9),
                                                       ("hill", 3, 5000, None), ("ramp", 0, 4096, None)])
def test_gpu_tile_painter_matches_host(cuda, kind, seed, cells, max_depth):
    """hc_paint_tiles_device (the index painted in HBM) equals the host
    painter's index (itself pinned to the reference's tile_index digests) tile for tile;
    the frame kernels read the painted tensor without an upload."""
    import torch
    from paper_2201_10887_b200 import synth
    g = synth.generate_synthetic(kind, seed, cells, max_depth=max_depth)
    dev_index = g.device_tile_index(cuda)
    assert dev_index is not None, "grid was not painted on the GPU"
    host = synth.generate_synthetic(kind, seed, cells, max_depth=max_depth, native_paint=False).tile_index
    assert torch.equal(dev_index, torch.from_numpy(np.array(host, copy=True)).to(cuda))
    assert np.array_equal(g.tile_index, host)                   # the lazy host download
    assert g.device_view(cuda).tile_index.data_ptr() == dev_index.data_ptr()


@pytest.mark.gpu
def test_gpu_tile_painter_detects_overlaps(cuda):
    """Overlapping squares: the painted-tile count falls short of the summed areas and
    the reference's sequential paint names the first clash (same message as the host)."""
    from paper_2201_10887_b200 import AdaptiveGrid, GridFormatError, Rect
    centers = np.array([[1.0, 1.0], [3.0, 3.0], [2.0, 2.0], [7.0, 7.0]])
    sizes = np.array([2.0, 2.0, 4.0, 2.0])
    z = np.zeros(4)
    h = AdaptiveGrid(Rect(0, 0, 8, 8), 2.0, centers, sizes, z + 10, z, check_overlap=False, native_paint=False)
    first = h._paint_numpy(True)[1]
    assert first == (0, 2)
    with pytest.raises(GridFormatError, match="cells 0 and 2 overlap"):
        AdaptiveGrid(Rect(0, 0, 8, 8), 2.0, centers, sizes, z + 10, z)
    g = AdaptiveGrid(Rect(0, 0, 8, 8), 2.0, centers, sizes, z + 10, z, check_overlap=False)
    assert g.device_tile_index(cuda) is None                    # overlap: the host index is kept
    assert np.array_equal(g.tile_index, h.tile_index) and g.find_overlap() == first

"""ctypes binding of libheightcast_cuda.so (the C ABI in include/heightcast.h).

This is the only module that touches the native library.  Structures mirror the
header field for field; every pointer passed is a CUDA device pointer taken
from a torch tensor, and every call is enqueued on torch's current stream.
There is no CPU fallback: if the library or a GPU is missing, `lib()` raises.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(PKG_DIR, "_lib")
LIB_PATH = os.environ.get("HC_LIB_PATH") or os.path.join(LIB_DIR, "libheightcast_cuda.so")
CSRC = os.path.join(PKG_DIR, "csrc")

HC_ABI_VERSION = 7
HC_MAX_EDGES = 32
HC_MAX_CASCADES = 8
HC_MAX_LEVELS = 20
HC_MAX_STRIPS = 16
HC_OK, HC_EINVAL, HC_ECUDA, HC_ECAPACITY = 0, -1, -2, -3
(CNT_VISIBLE, CNT_VALID, CNT_ZERO_WEIGHT, CNT_RAYS_HIT, CNT_PAIRS, CNT_NODE_VISITS,
 CNT_PATCH_TESTS) = range(7)
N_COUNTERS = 8

# exported symbols, in header order (tests check the .so exports all of them)
EXPORTS = ("hc_py_hypot", "hc_visible_hull", "hc_clip_cascades", "hc_fit_layout", "hc_plan_cascades",
           "hc_abi_version", "hc_last_error", "hc_build_records", "hc_visibility_mask",
           "hc_discretize", "hc_maxmip_workspace_bytes", "hc_maxmip", "hc_render", "hc_render_tiles",
           "hc_render_order_words", "hc_traverse_batch", "hc_eval_points", "hc_influence_workspace_bytes",
           "hc_influence_build", "hc_frame_launch", "hc_frame_xchg_floats", "hc_frame_stage",
           "hc_selftest_division", "hc_selftest_patch", "hc_selftest_slab", "hc_bench_l2_read", "hc_ahf_parse",
           "hc_paint_tiles", "hc_paint_tiles_device")
HC_MAX_HULL = 64

_vp = C.c_void_p
_d = C.c_double
_i32 = C.c_int32
_i64 = C.c_int64


class HcCamera(C.Structure):
    _fields_ = [("eye", _d * 3), ("look", _d * 3), ("up", _d * 3), ("fov_y", _d), ("aspect", _d),
                ("near_clip", _d), ("far_clip", _d)]


class HcDomain(C.Structure):
    _fields_ = [("xmin", _d), ("ymin", _d), ("xmax", _d), ("ymax", _d), ("h_lo", _d), ("h_hi", _d),
                ("min_cell", _d)]


class HcCascadePlan(C.Structure):
    _fields_ = [("present", _i32), ("n_verts", _i32), ("verts", (_d * 2) * HC_MAX_EDGES),
                ("near_offset", _d), ("far_offset", _d), ("origin", _d * 2), ("texel", _d),
                ("resolution", _i32), ("box_texel", _i32 * 2), ("box_steps", _i32 * 2),
                ("edges", (_d * 5) * HC_MAX_EDGES)]


class HcPlan(C.Structure):
    _fields_ = [("status", _i32), ("n_hull", _i32), ("hull", (_d * 2) * HC_MAX_HULL), ("overlap", _d),
                ("axis_anchor", _d * 2), ("axis_dir", _d * 2), ("count", _i32), ("n_active", _i32),
                ("c", HcCascadePlan * HC_MAX_CASCADES)]


class HcGrid(C.Structure):
    _fields_ = [("cx", _vp), ("cy", _vp), ("size", _vp), ("terrain", _vp), ("depth", _vp),
                ("tile_index", _vp), ("ntx", _i64), ("nty", _i64),
                ("xmin", _d), ("ymin", _d), ("min_cell", _d), ("n_cells", _i32),
                ("offsets", _vp), ("indices", _vp), ("pair_offsets", _vp), ("rec", _vp),
                ("anchor_t", _vp), ("anchor_d", _vp), ("sigma", _d)]


class HcCascadeRaster(C.Structure):
    _fields_ = [("origin_x", _d), ("origin_y", _d), ("texel", _d), ("resolution", _i32),
                ("n_edges", _i32), ("edges", _d * (HC_MAX_EDGES * 5)),
                ("terrain", _vp), ("water", _vp), ("valid", _vp), ("mask", _vp)]


class HcMipJob(C.Structure):
    _fields_ = [("heights", _vp), ("valid", _vp), ("mip", _vp), ("patch_ok", _vp),
                ("heights_other", _vp), ("vrange_key", _vp), ("resolution", _i32), ("n_levels", _i32),
                ("level_off", _i64 * HC_MAX_LEVELS), ("level_w", _i32 * HC_MAX_LEVELS)]


class HcRenderCascade(C.Structure):
    _fields_ = [("origin_x", _d), ("origin_y", _d), ("texel", _d), ("rx", _d), ("ry", _d),
                ("near_offset", _d), ("far_offset", _d), ("resolution", _i32), ("n_levels", _i32),
                ("patch_diff", _i32), ("reserved", _i32), ("heights", _vp * 2), ("valid", _vp), ("patch_ok", _vp), ("mip", _vp * 2),
                ("vrange_key", _vp), ("level_off", _i64 * HC_MAX_LEVELS),
                ("level_w", _i32 * HC_MAX_LEVELS)]


class HcRenderDebug(C.Structure):
    _fields_ = [(n, _vp) for n in ("hit", "t", "near_k", "far_k", "w", "raw_t", "raw_ix", "raw_iy",
                                   "raw_u", "raw_v", "water_depth", "dirs", "visits")]


class HcRenderArgs(C.Structure):
    _fields_ = [("width", _i32), ("height", _i32), ("n_cascades", _i32), ("x0", _i32), ("y0", _i32),
                ("x1", _i32), ("y1", _i32), ("eye", _d * 3), ("look", _d * 3), ("right", _d * 3),
                ("up", _d * 3), ("tan_half", _d), ("aspect", _d), ("axis_anchor", _d * 2),
                ("axis_dir", _d * 2), ("h_lo", _d), ("h_hi", _d), ("light", _d * 3),
                ("cm_lo", _d), ("cm_hi", _d), ("stops", _d * 9), ("background", C.c_uint8 * 4),
                ("c", HcRenderCascade * HC_MAX_CASCADES), ("rgb", _vp), ("counters", _vp),
                ("tile_counter", _vp), ("tile_cost", _vp), ("tile_order", _vp), ("dbg", HcRenderDebug)]


HC_MAX_SIZE_CLASSES = 32


class HcInfluenceBins(C.Structure):
    _fields_ = [("n_classes", _i32), ("xmin", _d), ("ymin", _d), ("class_size", _d * HC_MAX_SIZE_CLASSES),
                ("bin_size", _d * HC_MAX_SIZE_CLASSES), ("nbx", _i32 * HC_MAX_SIZE_CLASSES),
                ("nby", _i32 * HC_MAX_SIZE_CLASSES), ("class_bin_base", _i64 * HC_MAX_SIZE_CLASSES),
                ("bin_start", _vp), ("cells", _vp)]


class HcFrameBuffers(C.Structure):
    _fields_ = [("terrain", _vp), ("water", _vp), ("valid", _vp), ("mask", _vp), ("patch_ok", _vp),
                ("mip", _vp), ("vrange", _vp), ("mip_ws", _vp), ("mip_ws_bytes", C.c_size_t), ("rgb", _vp),
                ("counters", _vp), ("tile_counter", _vp), ("tile_cost", _vp), ("tile_order", _vp),
                ("capacity", _i32), ("resolution", _i32), ("width", _i32), ("height", _i32),
                ("throughput", _i32), ("reserved", _i32)]


class HcFootprint(C.Structure):
    _fields_ = [("n_strips", _i32), ("rank", _i32), ("apex", _d * 2), ("dir", ((_d * 2) * 2) * HC_MAX_STRIPS),
                ("all", _i32 * HC_MAX_STRIPS), ("margin", _d)]


class HcAhfInfo(C.Structure):
    _fields_ = [("xmin", _d), ("ymin", _d), ("xmax", _d), ("ymax", _d), ("min_cell", _d),
                ("count", _i64), ("error_line", _i64), ("non_ascii", _i32), ("reserved", _i32)]


class HcShading(C.Structure):
    _fields_ = [("cm_lo", _d), ("cm_hi", _d), ("light", _d * 3), ("stops", _d * 9),
                ("background", C.c_uint8 * 4)]


ROOT_FN = C.CFUNCTYPE(C.c_double, C.c_double, C.c_int)


def _numpy_root(q, count):
    """The split ratio exactly as the reference evaluates it (cascade.py:306: np.cbrt)."""
    import numpy as np
    if count == 3:
        return float(np.cbrt(q))
    if count == 2:
        return float(np.sqrt(q))
    return float(np.power(q, 1.0 / count))


NUMPY_ROOT = ROOT_FN(_numpy_root)


class HeightcastCudaError(RuntimeError):
    """A libheightcast_cuda call failed (message from hc_last_error)."""


_lib = None


def build(force: bool = False) -> str:
    """Compile the sm_100a library in-tree (nvcc cross-compiles without a GPU)."""
    args = ["make", "-s", "-C", CSRC] + (["-B"] if force else [])
    subprocess.run(args, check=True)
    return LIB_PATH


def lib():
    """Load the native library; fails loudly (no fallback) when absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise HeightcastCudaError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            f"or `make -C {CSRC}`; this package has no CPU fallback")
    L = C.CDLL(LIB_PATH)
    L.hc_last_error.restype = C.c_char_p
    L.hc_abi_version.restype = C.c_int
    L.hc_py_hypot.restype = C.c_double
    L.hc_py_hypot.argtypes = [C.c_double, C.c_double]
    L.hc_visible_hull.argtypes = [C.POINTER(HcCamera), C.POINTER(HcDomain), _vp, C.c_int, C.POINTER(C.c_int)]
    L.hc_clip_cascades.argtypes = [_vp, C.c_int, _vp, C.c_double, _vp, C.c_int, ROOT_FN, C.POINTER(HcPlan)]
    L.hc_fit_layout.argtypes = [_vp, C.c_int, C.c_int, C.c_double, C.c_double, C.POINTER(HcCascadePlan)]
    L.hc_plan_cascades.argtypes = [C.POINTER(HcCamera), C.POINTER(HcDomain), C.c_int, C.c_double, C.c_int,
                                   ROOT_FN, C.POINTER(HcPlan)]
    L.hc_maxmip_workspace_bytes.restype = C.c_size_t
    L.hc_maxmip_workspace_bytes.argtypes = [C.c_int, C.c_int]
    L.hc_build_records.argtypes = [C.POINTER(HcGrid), _vp, _vp, _vp, _vp]
    L.hc_visibility_mask.argtypes = [C.POINTER(HcCascadeRaster), _vp]
    L.hc_discretize.argtypes = [C.POINTER(HcCascadeRaster), C.c_int, C.POINTER(HcGrid), C.c_float,
                                _vp, _vp]
    L.hc_maxmip.argtypes = [C.POINTER(HcMipJob), C.c_int, _vp, C.c_size_t, _vp]
    L.hc_render.argtypes = [C.POINTER(HcRenderArgs), _vp]
    L.hc_traverse_batch.argtypes = [_vp, _vp, _vp, _vp, _vp, C.c_int, C.c_int] + [_vp] * 6 + \
        [_i64, _d, _d] + [_vp] * 6 + [_vp]
    L.hc_frame_launch.argtypes = [C.POINTER(HcPlan), C.POINTER(HcCamera), C.POINTER(HcDomain), C.POINTER(HcGrid),
                                  C.POINTER(HcFrameBuffers), C.POINTER(HcShading), C.POINTER(HcRenderDebug),
                                  _vp, _vp, _vp]
    L.hc_frame_xchg_floats.restype = C.c_size_t
    L.hc_frame_xchg_floats.argtypes = [C.c_int, C.c_int]
    L.hc_frame_stage.argtypes = [C.c_int, C.POINTER(HcPlan), C.POINTER(HcCamera), C.POINTER(HcDomain),
                                 C.POINTER(HcGrid), C.POINTER(HcFrameBuffers), C.POINTER(HcShading),
                                 C.POINTER(HcRenderDebug), _vp, _vp, C.POINTER(HcFootprint), _vp, _vp]
    L.hc_influence_workspace_bytes.restype = C.c_size_t
    L.hc_influence_workspace_bytes.argtypes = [C.c_int]
    L.hc_influence_build.argtypes = [C.POINTER(HcGrid), C.POINTER(HcInfluenceBins), C.c_double, _vp, _vp,
                                     C.c_int64, _vp, C.c_size_t, _vp, _vp]
    L.hc_render_tiles.restype = C.c_size_t
    L.hc_render_tiles.argtypes = [C.c_int] * 4
    L.hc_render_order_words.restype = C.c_size_t
    L.hc_render_order_words.argtypes = [C.c_int] * 4
    L.hc_selftest_division.argtypes = [C.c_uint64, C.c_uint64, _vp, _vp]
    L.hc_selftest_patch.argtypes = [C.c_uint64, C.c_uint64, _vp, _vp]
    L.hc_selftest_slab.argtypes = [C.c_uint64, C.c_uint64, _vp, _vp]
    L.hc_bench_l2_read.argtypes = [_vp, C.c_size_t, C.c_int, _vp, _vp]
    L.hc_eval_points.argtypes = [C.POINTER(HcGrid), _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]
    L.hc_ahf_parse.argtypes = [C.c_char_p, _i64, C.POINTER(HcAhfInfo), _vp, _i64]
    L.hc_paint_tiles.argtypes = [_vp, _vp, _vp, _i64, _i64, _i64, C.c_int, _vp, _vp]
    L.hc_paint_tiles_device.argtypes = [_vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp]
    ver = L.hc_abi_version()
    if ver != HC_ABI_VERSION:
        raise HeightcastCudaError(f"libheightcast_cuda ABI {ver}, expected {HC_ABI_VERSION}")
    _lib = L
    return L


def check(code: int, what: str) -> None:
    if code != HC_OK:
        msg = lib().hc_last_error().decode(errors="replace")
        raise HeightcastCudaError(f"{what} failed ({code}): {msg}")


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise HeightcastCudaError("no CUDA device: the heightcast hot path runs on B200 GPUs only")
    lib()

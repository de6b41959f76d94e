"""ctypes binding of the C ABI (include/vidfeat_b200.h).

The library is the product's only compute path: there is no CPU fallback.  If
the shared object is missing or cannot be loaded this module raises, and so
does every call that needs it.
"""

from __future__ import annotations

import ctypes
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_uint8, c_uint64, c_void_p

import numpy as np

from . import build as _build

VF_OK = 0
ERRORS = {
    -1: ValueError, -2: ValueError, -3: ValueError, -4: ValueError, -5: ValueError, -6: ValueError,
    -7: ValueError, -8: ValueError, -9: RuntimeError, -10: RuntimeError, -11: ValueError,
    -12: IndexError, -13: KeyError, -14: RuntimeError, -15: RuntimeError, -16: ValueError, -17: ValueError,
    -18: ValueError, -19: ValueError,
}
MODES = {"none": 0, "intensity": 1, "binning": 2, "temporal": 3}


class VfConfig(ctypes.Structure):
    _fields_ = [
        ("width", c_int32), ("height", c_int32), ("n_octaves", c_int32), ("threshold", c_int32),
        ("mask_mode", c_int32), ("t_i", c_double), ("t_h", c_int32), ("grid_rows", c_int32),
        ("grid_cols", c_int32), ("octave_for_mask", c_int32), ("per_layer", c_int32),
        ("max_streams", c_int32), ("kp_capacity", c_int32),
        ("gop_delta", c_int32), ("gop_patch", c_int32), ("gop_t_bm", c_double), ("gop_t_et", c_double),
        ("gop_coarse_window", c_double), ("gop_coarse_step", c_double), ("gop_fine_window", c_double),
        ("gop_fine_step", c_double),
    ]


class VfReport(ctypes.Structure):
    _fields_ = [
        ("frame", c_int64), ("n_detected", c_int32), ("n_propagated", c_int32), ("n_total", c_int32),
        ("n_dropped", c_int32), ("coverage", c_double), ("n_survivors", c_int32), ("n_candidates", c_int32),
    ]


class VfFeatures(ctypes.Structure):
    _fields_ = [
        ("n", c_int32), ("x", c_void_p), ("y", c_void_p), ("sigma", c_void_p), ("theta", c_void_p),
        ("score", c_void_p), ("origin", c_void_p), ("age", c_void_p), ("desc", c_void_p),
    ]


_lib = None
_pattern_done = False

_P = c_void_p  # device / host pointers are passed as integers


def lib():
    """Load (building in-tree if needed) the sm_100a library.  Raises if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    import os

    path = _build.LIB
    if os.environ.get("VF_LIB"):          # experiment builds
        path = os.environ["VF_LIB"]
    elif _build.needs_build():
        path = _build.build()
    L = ctypes.CDLL(str(path))
    L.vf_version.restype = ctypes.c_char_p
    L.vf_strerror.restype = ctypes.c_char_p
    L.vf_strerror.argtypes = [c_int]
    L.vf_set_pattern.argtypes = [_P, _P, c_int, _P, c_int, _P, c_int]
    L.vf_create.argtypes = [POINTER(VfConfig), POINTER(c_void_p)]
    L.vf_destroy.argtypes = [c_void_p]
    L.vf_layer_geometry.argtypes = [c_void_p, _P, _P, _P]
    L.vf_reset.argtypes = [c_void_p, c_void_p]
    L.vf_process.argtypes = [c_void_p, _P, c_int64, c_int64, c_int, c_void_p]
    L.vf_process_host.argtypes = [c_void_p, _P, c_int64, c_int64, c_int, c_void_p]
    L.vf_get_report.argtypes = [c_void_p, c_int, POINTER(VfReport), c_void_p]
    L.vf_get_features.argtypes = [c_void_p, c_int, POINTER(VfFeatures), c_void_p]
    L.vf_copy_features.argtypes = [c_void_p, c_int, c_int32, _P, _P, _P, _P, _P, _P, _P, _P, POINTER(c_int32), c_void_p]
    L.vf_get_layer.argtypes = [c_void_p, c_int, c_int, POINTER(c_void_p), POINTER(c_int32)]
    L.vf_get_totals.argtypes = [c_void_p, c_int, _P, c_void_p]
    L.vf_set_timing.argtypes = [c_void_p, c_int]
    L.vf_get_diag.argtypes = [c_void_p, _P, c_void_p]
    L.vf_fetch_features.argtypes = [c_void_p, c_int, c_int64, _P, _P, _P, _P, _P, _P, _P, _P, _P, c_void_p]
    L.vf_pipeline_submit.argtypes = [c_void_p, _P, c_int64, c_int64, c_int]
    L.vf_pipeline_collect.argtypes = [c_void_p, c_int64, _P, _P, _P, _P, _P, _P, _P, _P, _P]
    L.vf_get_stage_ms.argtypes = [c_void_p, _P, POINTER(c_int32), c_void_p]
    L.vf_build_pyramid.argtypes = [_P, c_int, c_int, c_int64, c_int, _P, _P, c_void_p]
    L.vf_score_map.argtypes = [_P, c_int, c_int, c_int64, c_int, _P, c_int, c_int, _P, c_int64, c_void_p]
    L.vf_nms_refine.argtypes = [_P, _P, c_int, c_int, c_int, c_int32, _P, _P, _P, _P, POINTER(c_int32), c_void_p]
    L.vf_describe.argtypes = [_P, c_int, c_int, c_int64, c_int, _P, _P, _P, _P, _P, _P, c_void_p]
    L.vf_intensity_mask.argtypes = [_P, _P, c_int64, c_double, _P, c_void_p]
    L.vf_binning_histogram.argtypes = [c_int, _P, _P, c_int, c_int, c_int, c_int, _P, c_void_p]
    L.vf_upsample_mask.argtypes = [_P, c_int, c_int, c_int, c_int, c_int, c_int, _P, c_void_p]
    L.vf_mask_values.argtypes = [_P, c_int, c_int, c_int, _P, _P, _P, c_void_p]
    L.vf_hamming_matrix.argtypes = [_P, c_int64, _P, c_int64, c_int, _P, c_int64, c_void_p]
    L.vf_format_features.argtypes = [c_int64, _P, _P, _P, _P, _P, _P, _P, c_int64, POINTER(c_int64)]
    L.vf_block_match.argtypes = [_P, _P, c_int, c_int, c_int64, c_int, _P, _P, POINTER(VfConfig), _P, _P, _P, _P,
                                 c_void_p]
    L.vf_radius_match.argtypes = [_P, c_int64, _P, c_int64, c_int, c_int, _P, _P, _P, c_int64,
                                  POINTER(c_int64), c_void_p]
    L.vf_match_timing.argtypes = [c_int, POINTER(c_double)]
    L.vf_set_history.argtypes = [c_void_p, _P, c_int32]
    L.vf_set_graphs.argtypes = [c_void_p, c_int]
    L.vf_process_checked.argtypes = [c_void_p, _P, c_int64, c_int64, c_int, c_void_p]
    L.vf_get_capacity.argtypes = [c_void_p, POINTER(c_int32)]
    L.vf_ast_corner_score.argtypes = [_P, c_int, c_int, c_int64, c_int, _P, _P, c_int, _P, c_void_p]
    L.vf_sad_block.argtypes = [_P, _P, c_int64, c_int, _P, c_void_p]
    L.vf_process_host_checked.argtypes = [c_void_p, _P, c_int64, c_int64, c_int, c_void_p]
    L.vf_pipeline_set_delta.argtypes = [c_void_p, c_int]
    L.vf_pipeline_collect_delta.argtypes = [c_void_p, c_int64] + [_P] * 7 + [c_int64, _P, _P, _P]
    L.vf_delta_apply.argtypes = [c_int32] + [_P] * 8 + [c_int32] + [_P] * 6 + [c_int32, _P, c_int32] + [_P] * 9
    L.vf_ransac_homography.argtypes = [c_int, _P, _P, _P, c_int, c_double, c_uint64, _P, _P, _P, c_void_p]
    L.vf_ransac_samples.argtypes = [c_uint64, c_int64, c_int, _P, c_void_p]
    L.vf_ransac_samples_host.argtypes = [c_uint64, c_int64, c_int, _P]
    for name in ("vf_set_pattern", "vf_create", "vf_destroy", "vf_layer_geometry", "vf_reset", "vf_process",
                 "vf_process_host", "vf_get_report", "vf_get_features", "vf_copy_features", "vf_get_layer",
                 "vf_get_totals", "vf_set_timing", "vf_get_stage_ms", "vf_get_diag", "vf_fetch_features", "vf_pipeline_submit",
    "vf_pipeline_collect", "vf_build_pyramid", "vf_score_map", "vf_nms_refine", "vf_describe",
                 "vf_intensity_mask", "vf_binning_histogram", "vf_upsample_mask", "vf_mask_values",
                 "vf_set_timing", "vf_get_stage_ms", "vf_get_diag", "vf_fetch_features", "vf_pipeline_submit",
                 "vf_pipeline_collect", "vf_hamming_matrix", "vf_radius_match", "vf_block_match",
                 "vf_format_features", "vf_ransac_homography", "vf_ransac_samples", "vf_ransac_samples_host",
                 "vf_match_timing", "vf_set_history", "vf_set_graphs", "vf_process_checked", "vf_get_capacity",
                 "vf_ast_corner_score", "vf_sad_block", "vf_process_host_checked", "vf_pipeline_set_delta",
                 "vf_pipeline_collect_delta", "vf_delta_apply"):
        getattr(L, name).restype = c_int
    _lib = L
    return L


# every symbol include/vidfeat_b200.h declares
EXPORTS = (
    "vf_version", "vf_strerror", "vf_set_pattern", "vf_create", "vf_destroy", "vf_layer_geometry", "vf_reset",
    "vf_process", "vf_process_host", "vf_get_report", "vf_get_features", "vf_copy_features", "vf_get_layer",
    "vf_get_totals", "vf_set_timing", "vf_get_stage_ms", "vf_get_diag", "vf_fetch_features", "vf_pipeline_submit",
    "vf_pipeline_collect", "vf_build_pyramid", "vf_score_map", "vf_nms_refine", "vf_describe", "vf_intensity_mask",
    "vf_binning_histogram", "vf_upsample_mask", "vf_mask_values", "vf_hamming_matrix", "vf_radius_match",
    "vf_block_match", "vf_format_features", "vf_ransac_homography", "vf_ransac_samples", "vf_ransac_samples_host",
    "vf_match_timing", "vf_set_history", "vf_set_graphs", "vf_process_checked", "vf_get_capacity",
    "vf_ast_corner_score", "vf_sad_block", "vf_process_host_checked", "vf_pipeline_set_delta",
    "vf_pipeline_collect_delta", "vf_delta_apply",
)


def check(rc: int, what: str = "") -> None:
    if rc == VF_OK:
        return
    msg = lib().vf_strerror(rc).decode()
    exc = ERRORS.get(rc, RuntimeError)
    raise exc(f"{msg}{' (' + what + ')' if what else ''}")


def ensure_pattern(pattern=None) -> None:
    """Upload the descriptor sampling pattern (once per process)."""
    global _pattern_done
    if _pattern_done and pattern is None:
        return
    from .pattern import default_pattern

    p = pattern or default_pattern()
    pts = np.ascontiguousarray(p.points, np.float64)
    rad = np.ascontiguousarray(p.radii, np.float64)
    sp = np.ascontiguousarray(p.short_pairs, np.int32)
    lp = np.ascontiguousarray(p.long_pairs, np.int32)
    check(lib().vf_set_pattern(pts.ctypes.data, rad.ctypes.data, pts.shape[0], sp.ctypes.data, sp.shape[0],
                               lp.ctypes.data, lp.shape[0]), "vf_set_pattern")
    _pattern_done = True


def stream_handle(stream=None) -> int:
    """cudaStream_t of a torch stream (default: torch's current stream)."""
    import torch

    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)

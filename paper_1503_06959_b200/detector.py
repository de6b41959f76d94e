"""Segment-test detection + scale-space NMS (drop-in for vidfeat.detector).

detect_candidates / ast_corner_score run k_fast (vf_score_map) and
nms_and_refine runs k_nms (vf_nms_refine), which shares the pipeline's
nms_test / nms_refine device code (the pipeline itself runs them thread per
candidate in k_nms_test).
Reference: detector.py:1-324.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _dev, _native
from .pyramid import layer_geometry
from .types import (DEFAULT_THRESHOLD, RETRIEVAL_THRESHOLD, Candidate, GrayFrame, Keypoint,
                    ScaleSpacePyramid)

# Radius-3 Bresenham circle, clockwise from (0, -3) (detector.py:20-28)
CIRCLE = np.array(
    [(0, -3), (1, -3), (2, -2), (3, -1), (3, 0), (3, 1), (2, 2), (1, 3),
     (0, 3), (-1, 3), (-2, 2), (-3, 1), (-3, 0), (-3, -1), (-2, -2), (-1, -3)],
    dtype=np.int64,
)

__all__ = ["CIRCLE", "Candidate", "Keypoint", "DEFAULT_THRESHOLD", "RETRIEVAL_THRESHOLD", "score_map",
           "detect_candidates", "ast_corner_score", "ast_corner_scores", "nms_and_refine", "nms_from_maps"]


def score_map(data: np.ndarray, t: int, mask_bits: np.ndarray | None = None) -> np.ndarray:
    """_score_map (detector.py:166-172) with the gate given as a FULL-RES mask
    (projected by floor mapping inside the kernel, detector.py:175-181)."""
    if t < 1:
        raise ValueError("detection threshold must be >= 1")
    h, w = data.shape
    L = _dev.lib()
    t_ = _dev.torch()
    d = _dev.to_dev(data)
    out = _dev.empty((h, w), t_.uint8)
    if mask_bits is None:
        mptr, mw, mh = 0, 0, 0
    else:
        m = _dev.to_dev(np.ascontiguousarray(mask_bits, np.uint8))
        mptr, (mh, mw) = m.data_ptr(), mask_bits.shape
    _native.check(L.vf_score_map(d.data_ptr(), w, h, w, int(t), mptr, mw, mh, out.data_ptr(), w, _dev.stream()),
                  "vf_score_map")
    return out.cpu().numpy()


def detect_candidates(layer: GrayFrame, t: int, mask=None, layer_id: tuple[str, int] = ("octave", 0)
                      ) -> list[Candidate]:
    """detector.py:184-204: pixels with score >= t whose mapped mask entry is 1."""
    if t < 1:
        raise ValueError("detection threshold must be >= 1")
    smap = score_map(layer.data, int(t), None if mask is None else mask.bits)
    ys, xs = np.nonzero(smap)
    return [Candidate(int(x), int(y), layer_id, int(smap[y, x])) for y, x in zip(ys, xs)]


def ast_corner_score(layer: GrayFrame, x: int, y: int, arc_len: int = 9) -> int:
    """detector.py:58-71: largest integer t with arc_len contiguous circle
    pixels all > c + t or all < c - t (any arc length; vf_ast_corner_score)."""
    h, w = layer.data.shape
    if not (3 <= x < w - 3 and 3 <= y < h - 3):
        raise ValueError(f"({x}, {y}) is within 3 pixels of the layer border")
    return int(ast_corner_scores(layer, np.array([x]), np.array([y]), arc_len)[0])


def ast_corner_scores(layer: GrayFrame, xs, ys, arc_len: int = 9) -> np.ndarray:
    """ast_corner_score of many points in one launch (int32 array)."""
    h, w = layer.data.shape
    xs = np.ascontiguousarray(xs, np.int32)
    ys = np.ascontiguousarray(ys, np.int32)
    if xs.shape != ys.shape:
        raise ValueError("xs and ys must have the same shape")
    if xs.size and not (((xs >= 3) & (xs < w - 3) & (ys >= 3) & (ys < h - 3)).all()):
        bad = int(np.nonzero(~((xs >= 3) & (xs < w - 3) & (ys >= 3) & (ys < h - 3)))[0][0])
        raise ValueError(f"({int(xs[bad])}, {int(ys[bad])}) is within 3 pixels of the layer border")
    if int(arc_len) < 1:
        raise ValueError("zero-size array to reduction operation minimum which has no identity")
    if xs.size == 0:
        return np.zeros(0, np.int32)
    t_ = _dev.torch()
    d = _dev.to_dev(layer.data)
    out = _dev.empty(xs.shape, t_.int32)
    xd, yd = _dev.to_dev(xs), _dev.to_dev(ys)   # keep both alive until the launch is enqueued
    _native.check(_dev.lib().vf_ast_corner_score(d.data_ptr(), w, h, w, int(xs.size), xd.data_ptr(), yd.data_ptr(),
                                                 int(arc_len), out.data_ptr(), _dev.stream()), "vf_ast_corner_score")
    return out.cpu().numpy()


def nms_from_maps(maps: list[np.ndarray], width: int, height: int, n_octaves: int,
                  capacity: int | None = None) -> list[Keypoint]:
    """_nms_from_maps (detector.py:239-307) over uint8 score maps of every layer."""
    ws, hs, _ = layer_geometry(width, height, n_octaves)
    for i, m in enumerate(maps):
        if m.shape != (hs[i], ws[i]):
            raise ValueError(f"score map {i} has shape {m.shape}, expected {(hs[i], ws[i])}")
        if m.size:
            # numpy raises IndexError for smap[ys + 1, ...] past the last row/column (detector.py:260-262)
            if m[-1, :].any() or m[:, -1].any():
                raise IndexError("candidate on the last row/column of its layer")
    L = _dev.lib()
    t_ = _dev.torch()
    devs = [_dev.to_dev(np.ascontiguousarray(m, np.uint8)) for m in maps]
    ptrs = np.array([d.data_ptr() for d in devs], np.uint64)
    pitches = np.array([m.shape[1] for m in maps], np.int64)
    cap = capacity or max(1024, sum(int((m > 0).sum()) for m in maps))
    outs = [_dev.empty(cap, t_.float64) for _ in range(4)]
    n = ctypes.c_int32(0)
    _native.check(L.vf_nms_refine(ptrs.ctypes.data, pitches.ctypes.data, width, height, n_octaves, cap,
                                  outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(), outs[3].data_ptr(),
                                  ctypes.byref(n), _dev.stream()), "vf_nms_refine")
    k = int(n.value)
    x, y, s, v = (o[:k].cpu().numpy() for o in outs)
    return [Keypoint(float(x[i]), float(y[i]), float(s[i]), 0.0, float(v[i])) for i in range(k)]


def nms_and_refine(candidates: dict, pyramid: ScaleSpacePyramid) -> list[Keypoint]:
    """detector.py:310-324: rasterise candidates per layer, then NMS + refinement."""
    maps = [np.zeros(layer.frame.data.shape, np.int64) for layer in pyramid.layers]
    for i, layer in enumerate(pyramid.layers):
        for c in candidates.get((layer.kind, layer.level), []):
            maps[i][c.y, c.x] = c.score
    for m in maps:
        if m.size and (m.min() < 0 or m.max() > 255):
            raise ValueError("B200 score maps are uint8: candidate scores must lie in [0, 255]")
    f0 = pyramid.layers[0].frame
    return nms_from_maps([m.astype(np.uint8) for m in maps], f0.width, f0.height, pyramid.n_octaves)

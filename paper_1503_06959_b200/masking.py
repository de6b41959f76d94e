"""Detection masks and Eq. 1 feature propagation (drop-in for vidfeat.masking).

The per-element work (IDDM compare, histogram, block replication, mask bit
under each feature) runs on the GPU through the C-ABI; list splicing of the
Python Feature objects is host bookkeeping.  Reference: masking.py:1-192.
"""

from __future__ import annotations

import logging
from dataclasses import replace

import numpy as np

from . import _dev, _native
from .types import (DEFAULT_BINNING_GRID, DEFAULT_INTENSITY_THRESHOLD, DETECTED, PROPAGATED, DetectionMask,
                    Feature, GrayFrame, MaskConfig, SubsampledMask)

log = logging.getLogger(__name__)

__all__ = ["DetectionMask", "SubsampledMask", "Feature", "MaskConfig", "DETECTED", "PROPAGATED",
           "DEFAULT_INTENSITY_THRESHOLD", "DEFAULT_BINNING_GRID", "intensity_diff_mask", "binning_histogram",
           "keypoint_binning_mask", "upsample_mask", "mask_values", "merge_features"]


def intensity_diff_mask(prev_layer: GrayFrame, cur_layer: GrayFrame, t_i: float) -> SubsampledMask:
    """masking.py:84-93: cell = 1 iff |cur - prev| > t_i (strict)."""
    if prev_layer.data.shape != cur_layer.data.shape:
        raise ValueError(f"layer dimensions differ: {prev_layer.data.shape} vs {cur_layer.data.shape}")
    t = _dev.torch()
    a = _dev.to_dev(prev_layer.data)
    b = _dev.to_dev(cur_layer.data)
    out = _dev.empty(prev_layer.data.shape, t.uint8)
    _native.check(_dev.lib().vf_intensity_mask(a.data_ptr(), b.data_ptr(), a.numel(), float(t_i), out.data_ptr(),
                                               _dev.stream()), "vf_intensity_mask")
    return SubsampledMask(out.cpu().numpy())


def binning_histogram(features: list[Feature], frame_dims: tuple[int, int], grid: tuple[int, int]) -> np.ndarray:
    """masking.py:96-119: (rows, cols) histogram, ceil cells, clamped."""
    w, h = frame_dims
    rows, cols = grid
    t = _dev.torch()
    hist = _dev.zeros((rows, cols), t.int64)
    if not features:
        return hist.cpu().numpy()
    xs = np.array([f.kp.x for f in features])
    ys = np.array([f.kp.y for f in features])
    out_of_frame = int(((xs < 0) | (xs >= w) | (ys < 0) | (ys >= h)).sum())
    if out_of_frame:
        log.warning("%d features outside frame clamped to edge bins", out_of_frame)
    dx, dy = _dev.to_dev(xs), _dev.to_dev(ys)
    _native.check(_dev.lib().vf_binning_histogram(len(xs), dx.data_ptr(), dy.data_ptr(), w, h, rows, cols,
                                                  hist.data_ptr(), _dev.stream()), "vf_binning_histogram")
    return hist.cpu().numpy()


def keypoint_binning_mask(prev_features: list[Feature], frame_dims: tuple[int, int], grid: tuple[int, int],
                          t_h: int) -> SubsampledMask:
    """masking.py:122-136."""
    w, h = frame_dims
    rows, cols = grid
    hist = binning_histogram(prev_features, frame_dims, grid)
    return SubsampledMask((hist >= t_h).astype(np.uint8), cell_w=-(-w // cols), cell_h=-(-h // rows))


def upsample_mask(m: SubsampledMask, target: tuple[int, int]) -> DetectionMask:
    """masking.py:139-148: pixel (x, y) takes cell (x // cell_w, y // cell_h)."""
    w, h = target
    rows, cols = m.bits.shape
    cell_w = m.cell_w if m.cell_w is not None else -(-w // cols)
    cell_h = m.cell_h if m.cell_h is not None else -(-h // rows)
    if cell_w * cols < w or cell_h * rows < h:
        raise ValueError("mask cell geometry does not cover the target frame")
    t = _dev.torch()
    bits = _dev.to_dev(np.ascontiguousarray(m.bits, np.uint8))
    out = _dev.empty((h, w), t.uint8)
    _native.check(_dev.lib().vf_upsample_mask(bits.data_ptr(), rows, cols, cell_w, cell_h, w, h, out.data_ptr(),
                                              _dev.stream()), "vf_upsample_mask")
    return DetectionMask(out.cpu().numpy())


def mask_values(mask: DetectionMask, xs, ys) -> np.ndarray:
    """masking.py:157-165 _mask_values: bit under each rounded, clamped position."""
    n = len(xs)
    if n == 0:
        return np.zeros(0, np.uint8)
    t = _dev.torch()
    full = _dev.to_dev(np.ascontiguousarray(mask.bits, np.uint8))
    dx, dy = _dev.to_dev(np.asarray(xs, np.float64)), _dev.to_dev(np.asarray(ys, np.float64))
    out = _dev.empty(n, t.uint8)
    _native.check(_dev.lib().vf_mask_values(full.data_ptr(), mask.width, mask.height, n, dx.data_ptr(),
                                            dy.data_ptr(), out.data_ptr(), _dev.stream()), "vf_mask_values")
    return out.cpu().numpy()


def merge_features(detected: list[Feature], prev: list[Feature], mask: DetectionMask) -> list[Feature]:
    """masking.py:168-184 (Eq. 1): detected where the mask is 1, previous where it is 0."""
    dm = mask_values(mask, [f.kp.x for f in detected], [f.kp.y for f in detected])
    pm = mask_values(mask, [f.kp.x for f in prev], [f.kp.y for f in prev])
    out = [d for d, v in zip(detected, dm) if v == 1]
    out.extend(replace(p, origin=PROPAGATED, age=p.age + 1) for p, v in zip(prev, pm) if v == 0)
    return out

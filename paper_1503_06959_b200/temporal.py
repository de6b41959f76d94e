"""Temporal block-matching baseline on the GPU.

Mirrors /root/reference/pkg/src/vidfeat/temporal.py: ``GopConfig``,
``spiral_offsets`` (the search-order constants, built on the host like the
sampling pattern), ``spiral_search`` and ``baseline_step``.  The searches run
in the sm_100a kernel behind ``vf_block_match`` (csrc/vf_temporal.cuh, one
warp per feature); ``run_pipeline`` in ``temporal`` mode runs the whole
baseline inside FeatureEngine (full detection at GOP starts, block matching
in between, pipeline.py:281-345).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import replace

import numpy as np

from . import _dev, _native
from .types import PROPAGATED, Feature, GopConfig, GrayFrame

__all__ = ["GopConfig", "spiral_offsets", "spiral_search", "baseline_step", "block_match_device", "sad_block",
           "sad_blocks"]


def sad_block(a: np.ndarray, b: np.ndarray) -> int:
    """temporal.py:63-67: sum of absolute pixel differences of two equal-size patches."""
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        raise ValueError(f"patch dimensions differ: {a.shape} vs {b.shape}")
    return int(sad_blocks(a[None], b[None])[0])


def sad_blocks(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """sad_block of count pairs of uint8 patches [count, ...] in one launch (vf_sad_block)."""
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    if a.shape != b.shape:
        raise ValueError(f"patch dimensions differ: {a.shape} vs {b.shape}")
    count = a.shape[0]
    if count == 0:
        return np.zeros(0, np.int64)
    t_ = _dev.torch()
    out = _dev.empty((count,), t_.int64)
    n = int(np.prod(a.shape[1:]))
    ad, bd = _dev.to_dev(a), _dev.to_dev(b)   # keep both alive until the launch is enqueued
    _native.check(_dev.lib().vf_sad_block(ad.data_ptr(), bd.data_ptr(), n, count, out.data_ptr(), _dev.stream()),
                  "vf_sad_block")
    return out.cpu().numpy()


def spiral_offsets(radius: float, step: float) -> np.ndarray:
    """temporal.py:46-61: grid offsets within +/-radius at `step`, centre outward
    by Chebyshev ring, counterclockwise from +x within a ring."""
    n = int(math.floor(radius / step + 1e-9))
    vals = step * np.arange(-n, n + 1)
    ox, oy = np.meshgrid(vals, vals)
    ox, oy = ox.ravel(), oy.ravel()
    cheb = np.maximum(np.abs(ox), np.abs(oy))
    ang = np.arctan2(oy, ox)
    ang = np.where(ang < -1e-12, ang + 2.0 * np.pi, ang)
    order = np.lexsort((ang, cheb))
    return np.stack([ox[order], oy[order]], axis=1)


def _gop_struct(cfg: GopConfig):
    c = _native.VfConfig()
    c.gop_delta, c.gop_patch = int(cfg.delta), int(cfg.patch)
    c.gop_t_bm, c.gop_t_et = float(cfg.t_bm), float(cfg.t_et)
    c.gop_coarse_window, c.gop_coarse_step = float(cfg.coarse_window), float(cfg.coarse_step)
    c.gop_fine_window, c.gop_fine_step = float(cfg.fine_window), float(cfg.fine_step)
    return c


def block_match_device(prev, cur, x, y, cfg: GopConfig | None = None):
    """baseline_step's search for every feature (temporal.py:274-308) on CUDA
    tensors: prev / cur uint8 (h, w), x / y float64 (n,).  Returns (found bool,
    new x, new y, SAD) CUDA tensors."""
    t = _dev.torch()
    cfg = cfg or GopConfig()
    prev, cur = prev.contiguous(), cur.contiguous()
    if prev.shape != cur.shape or prev.dim() != 2:
        raise ValueError("previous and current frames must be 2-D and the same size")
    h, w = cur.shape
    n = int(x.numel())
    nx = t.empty(n, dtype=t.float64, device=cur.device)
    ny = t.empty(n, dtype=t.float64, device=cur.device)
    sad = t.empty(n, dtype=t.float64, device=cur.device)
    found = t.empty(n, dtype=t.uint8, device=cur.device)
    g = _gop_struct(cfg)
    x = x.to(t.float64).contiguous()
    y = y.to(t.float64).contiguous()
    _native.check(_native.lib().vf_block_match(prev.data_ptr(), cur.data_ptr(), w, h, w, n, x.data_ptr(),
                                               y.data_ptr(), ctypes.byref(g), nx.data_ptr(), ny.data_ptr(),
                                               sad.data_ptr(), found.data_ptr(), _dev.stream()), "vf_block_match")
    return found.bool(), nx, ny, sad


def spiral_search(prev_patch: np.ndarray, cur_frame: GrayFrame, center: tuple[float, float], cfg: GopConfig):
    """temporal.py:183-226: locate prev_patch in cur_frame around center.
    Returns ((x, y), sad) when the best SAD beats t_bm, else None.  The block
    at the rounded centre must lie inside the frame (as baseline_step ensures)."""
    ph, pw = prev_patch.shape
    if ph != cfg.patch or pw != cfg.patch:
        raise ValueError(f"patch dimensions differ: {prev_patch.shape} vs {(cfg.patch, cfg.patch)}")
    h, w = cur_frame.data.shape
    cxi = int(math.floor(center[0] + 0.5))
    cyi = int(math.floor(center[1] + 0.5))
    tlx, tly = cxi - pw // 2, cyi - ph // 2
    if tlx < 0 or tly < 0 or tlx + pw > w or tly + ph > h:
        raise ValueError("the block at the rounded centre leaves the frame")
    prev = np.zeros((h, w), np.uint8)
    prev[tly:tly + ph, tlx:tlx + pw] = prev_patch
    f, nx, ny, sad = block_match_device(_dev.to_dev(prev), _dev.to_dev(cur_frame.data),
                                        _dev.to_dev(np.array([center[0]], np.float64)),
                                        _dev.to_dev(np.array([center[1]], np.float64)), cfg)
    if not bool(f[0]):
        return None
    return (float(nx[0]), float(ny[0])), float(sad[0])


def baseline_step(prev_features: list[Feature], prev_frame: GrayFrame | None, cur_frame: GrayFrame,
                  frame_index: int, cfg: GopConfig, detector, descriptor) -> list[Feature]:
    """temporal.py:229-308: full detection at GOP starts, block matching
    elsewhere (unmatched features dropped; matched ones move, keeping
    descriptor, sigma and theta; origin propagated, age + 1)."""
    if frame_index % cfg.delta == 0 or prev_frame is None:
        return descriptor(cur_frame, detector(cur_frame))
    if not prev_features:
        return []
    xs = np.array([f.kp.x for f in prev_features], np.float64)
    ys = np.array([f.kp.y for f in prev_features], np.float64)
    found, nx, ny, _ = block_match_device(_dev.to_dev(prev_frame.data), _dev.to_dev(cur_frame.data),
                                          _dev.to_dev(xs), _dev.to_dev(ys), cfg)
    found, nx, ny = found.cpu().numpy(), nx.cpu().numpy(), ny.cpu().numpy()
    return [replace(f, kp=replace(f.kp, x=float(nx[i]), y=float(ny[i])), origin=PROPAGATED, age=f.age + 1)
            for i, f in enumerate(prev_features) if found[i]]

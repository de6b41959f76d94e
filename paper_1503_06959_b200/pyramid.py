"""Scale-space pyramid (drop-in for vidfeat.pyramid, pyramid.py:1-125).

build_pyramid runs k_pyramid (the same kernel as the pipeline) through the
C-ABI entry vf_build_pyramid.  Layer order o0, i0, o1, i1, ...; octave scale
2^-o, intra scale 2^-o / 1.5 (pyramid.py:118-124).
"""

from __future__ import annotations

import numpy as np

from . import _dev, _native
from .types import INTRA, OCTAVE, GrayFrame, PyramidLayer, ScaleSpacePyramid

__all__ = ["GrayFrame", "PyramidLayer", "ScaleSpacePyramid", "build_pyramid", "layer_geometry", "OCTAVE", "INTRA"]


def layer_geometry(width: int, height: int, n_octaves: int):
    """(ws, hs, scales) of the 2*O layers; raises the reference's ValueErrors (pyramid.py:103-109)."""
    if n_octaves < 1:
        raise ValueError("n_octaves must be >= 1")
    need = 1 << (n_octaves - 1)
    if width < need or height < need:
        raise ValueError(f"frame {width}x{height} too small for {n_octaves} octaves")
    ws, hs, sc = [], [], []
    ow, oh, iw, ih = width, height, (2 * width) // 3, (2 * height) // 3
    if iw < 1 or ih < 1:
        raise ValueError("dimension underflow in 2/3 resample")
    for o in range(n_octaves):
        if o > 0:
            ow, oh, iw, ih = ow // 2, oh // 2, iw // 2, ih // 2
            if min(ow, oh, iw, ih) < 1:
                raise ValueError("dimension underflow while halving")
        ws += [ow, iw]
        hs += [oh, ih]
        sc += [2.0 ** (-o), 2.0 ** (-o) / 1.5]
    return ws, hs, sc


def build_pyramid(frame: GrayFrame, n_octaves: int = 4) -> ScaleSpacePyramid:
    """pyramid.py:97-125 on the GPU; returns host layers like the reference."""
    H, W = frame.data.shape
    ws, hs, sc = layer_geometry(W, H, n_octaves)
    L = _dev.lib()
    t = _dev.torch()
    src = _dev.to_dev(frame.data)
    outs = [None] + [_dev.empty((hs[i], ws[i]), t.uint8) for i in range(1, 2 * n_octaves)]
    ptrs = np.array([0] + [o.data_ptr() for o in outs[1:]], np.uint64)
    pitches = np.array([W] + [ws[i] for i in range(1, 2 * n_octaves)], np.int64)
    _native.check(L.vf_build_pyramid(src.data_ptr(), W, H, W, n_octaves, ptrs.ctypes.data, pitches.ctypes.data,
                                     _dev.stream()), "vf_build_pyramid")
    layers = []
    for o in range(n_octaves):
        oframe = frame if o == 0 else GrayFrame(outs[2 * o].cpu().numpy(), frame.index)
        layers.append(PyramidLayer(oframe, sc[2 * o], OCTAVE, o))
        layers.append(PyramidLayer(GrayFrame(outs[2 * o + 1].cpu().numpy(), frame.index), sc[2 * o + 1], INTRA, o))
    return ScaleSpacePyramid(layers, n_octaves)

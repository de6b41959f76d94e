"""Descriptor radius matching on the GPU.

Mirrors /root/reference/pkg/src/vidfeat/matching.py:20-94: ``Match``,
``DEFAULT_MATCH_RADIUS``, ``hamming_matrix`` (pairwise Hamming distances of
packed descriptor rows, int32) and ``radius_match`` (every pair within t_m,
in np.nonzero order), with the reference's validation and error text.  The
distances come from the sm_100a kernels behind ``vf_hamming_matrix`` /
``vf_radius_match`` (csrc/vf_match.cu); there is no CPU path.

Device-resident variants (``hamming_matrix_device``, ``radius_match_device``)
take and return torch CUDA tensors, e.g. the packed descriptors that
``FeatureEngine.features_device`` exposes, so matching two frames' features
never leaves HBM.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _native
from .types import Feature

DEFAULT_MATCH_RADIUS = 102  # matching.py:20, Hamming threshold on 512-bit descriptors
_density = 0.0              # matches per pair seen by the last radius_match_device call


@dataclass(frozen=True, slots=True)
class Match:  # matching.py:25-29
    query_idx: int
    ref_idx: int
    distance: int


def _pack_descriptors(features: list[Feature]) -> np.ndarray:
    """matching.py:40-44: stacked 0/1 bits -> np.packbits rows."""
    bits = np.stack([f.desc for f in features])
    if bits.shape[1] % 8 != 0:
        raise ValueError("descriptor length must be a multiple of 8")
    return np.packbits(bits, axis=1)


def _as_rows(a):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    if a.ndim != 2:
        raise ValueError("packed descriptors must be a 2-D uint8 array (rows x bytes)")
    return a


def hamming_matrix_device(q, r):
    """Pairwise Hamming distances of packed rows q (nq x nb) and r (nr x nb),
    both uint8 CUDA tensors; returns an int32 (nq, nr) CUDA tensor."""
    t = _dev.torch()
    if q.dim() != 2 or r.dim() != 2 or q.shape[1] != r.shape[1]:
        raise ValueError("packed descriptor rows must be 2-D with equal widths")
    q = q.contiguous()
    r = r.contiguous()
    nq, nb = q.shape
    nr = r.shape[0]
    out = t.empty((nq, nr), dtype=t.int32, device=q.device)
    if nq and nr:
        _native.check(_native.lib().vf_hamming_matrix(q.data_ptr(), nq, r.data_ptr(), nr, nb, out.data_ptr(), nr,
                                                      _dev.stream()), "vf_hamming_matrix")
    return out


def hamming_matrix(q: np.ndarray, r: np.ndarray) -> np.ndarray:
    """matching.py:73-77: pairwise Hamming distances between packed descriptor rows."""
    q = _as_rows(q)
    r = _as_rows(r)
    if q.shape[1] != r.shape[1]:
        raise ValueError("packed descriptor rows have different widths")
    if q.shape[0] == 0 or r.shape[0] == 0:
        return np.empty((q.shape[0], r.shape[0]), np.int32)
    return hamming_matrix_device(_dev.to_dev(q), _dev.to_dev(r)).cpu().numpy()


def radius_match_device(q, r, t_m: int = DEFAULT_MATCH_RADIUS):
    """All (i, j) with Hamming(q_i, r_j) <= t_m on packed uint8 CUDA tensors.
    Returns (query_idx, ref_idx, distance) int32 CUDA tensors in np.nonzero
    order (query-major, then reference)."""
    import ctypes

    t = _dev.torch()
    if q.dim() != 2 or r.dim() != 2 or q.shape[1] != r.shape[1]:
        raise ValueError("packed descriptor rows must be 2-D with equal widths")
    q = q.contiguous()
    r = r.contiguous()
    nq, nb = q.shape
    nr = r.shape[0]
    L = _native.lib()
    global _density
    # size the output from the last observed match density (an overflow costs a recompute)
    cap = max(1 << 21, int(1.5 * _density * nq * nr) + 1024)
    while True:
        qi = t.empty(cap, dtype=t.int32, device=q.device)
        ri = t.empty(cap, dtype=t.int32, device=q.device)
        d = t.empty(cap, dtype=t.int32, device=q.device)
        n = ctypes.c_int64(0)
        rc = L.vf_radius_match(q.data_ptr(), nq, r.data_ptr(), nr, nb, int(t_m), qi.data_ptr(), ri.data_ptr(),
                               d.data_ptr(), cap, ctypes.byref(n), _dev.stream())
        if rc == -15:              # VF_ERR_MATCH_CAPACITY: n = the required size
            cap = int(n.value)
            continue
        _native.check(rc, "vf_radius_match")
        k = int(n.value)
        _density = max(_density * 0.5, k / max(1, nq * nr))
        return qi[:k], ri[:k], d[:k]


def radius_match(query: list[Feature], reference: list[Feature], t_m: int = DEFAULT_MATCH_RADIUS) -> list[Match]:
    """matching.py:80-94: every (query, reference) pair with Hamming distance <= t_m."""
    if not query or not reference:
        return []
    lengths = {f.desc.shape[0] for f in query} | {f.desc.shape[0] for f in reference}
    if len(lengths) != 1:
        raise ValueError(f"descriptors have mixed lengths: {sorted(lengths)}")
    qi, ri, d = radius_match_device(_dev.to_dev(_pack_descriptors(query)), _dev.to_dev(_pack_descriptors(reference)),
                                    t_m)
    qi, ri, d = qi.cpu().numpy(), ri.cpu().numpy(), d.cpu().numpy()
    return [Match(int(a), int(b), int(c)) for a, b, c in zip(qi, ri, d)]

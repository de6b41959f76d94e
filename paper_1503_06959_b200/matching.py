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


# ---------------------------------------------------------------------------
# Geometric verification: matching.py:97-220.  The
# RANSAC loop of every match set runs in csrc/vf_ransac.cu (vf_ransac_homography),
# many sets per launch; minimal samples follow np.random.default_rng(seed)
# draw for draw, so the chosen model matches the reference's.
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class MatchConfig:  # matching.py:32-37
    t_m: int = DEFAULT_MATCH_RADIUS
    iters: int = 1000
    reproj_tol: float = 3.0
    seed: int = 0


def project_points(h: np.ndarray, pts: np.ndarray) -> np.ndarray:
    """matching.py:149-154: points through a homography, |z| < 1e-12 -> 1e-12."""
    pts = np.asarray(pts, np.float64).reshape(-1, 2)
    ph = np.column_stack([pts, np.ones(len(pts))]) @ np.asarray(h, np.float64).T
    z = ph[:, 2]
    z = np.where(np.abs(z) < 1e-12, 1e-12, z)
    return ph[:, :2] / z[:, None]


def _check_seed(seed) -> int:
    seed = int(seed)
    if seed < 0:     # numpy's SeedSequence rejects negative entropy
        raise ValueError("expected non-negative integer")
    if seed >= 1 << 64:
        raise ValueError("seeds beyond 64 bits are not supported")
    return seed


def ransac_homography_device(src, dst, offsets, iters: int = 1000, reproj_tol: float = 3.0, seed: int = 0):
    """Batched ransac_homography on CUDA tensors.  src / dst: (N, 2) float64
    match coordinates (query / reference) of all problems, problem p owning
    rows [offsets[p], offsets[p+1]) (host ints).  Returns (H (P, 3, 3) float64,
    inlier (N,) bool, n_inliers (P,) int32; -1 where the reference returns
    (None, [])) as CUDA tensors."""
    import ctypes

    t = _dev.torch()
    off = np.ascontiguousarray(np.asarray(offsets, np.int64))
    P = off.size - 1
    if P < 0 or off[0] != 0 or np.any(np.diff(off) < 0):
        raise ValueError("offsets must start at 0 and be non-decreasing")
    if int(iters) < 0:
        raise ValueError("iters must be >= 0")
    dev = "cuda"
    src = src.to(device=dev, dtype=t.float64).contiguous().reshape(-1, 2)
    dst = dst.to(device=dev, dtype=t.float64).contiguous().reshape(-1, 2)
    if src.shape[0] != off[-1] or dst.shape[0] != off[-1]:
        raise ValueError("offsets do not cover the point arrays")
    H = t.empty((max(P, 0), 3, 3), dtype=t.float64, device=dev)
    inl = t.empty(int(off[-1]), dtype=t.uint8, device=dev)
    cnt = t.empty(max(P, 0), dtype=t.int32, device=dev)
    if P == 0:
        return H, inl.bool(), cnt
    _native.check(_native.lib().vf_ransac_homography(P, off.ctypes.data_as(ctypes.c_void_p), src.data_ptr(),
                                                     dst.data_ptr(), int(iters), float(reproj_tol),
                                                     _check_seed(seed), H.data_ptr(), inl.data_ptr(), cnt.data_ptr(),
                                                     _dev.stream()), "vf_ransac_homography")
    return H, inl.bool(), cnt


def ransac_homography_batch(problems, iters: int = 1000, reproj_tol: float = 3.0, seed: int = 0):
    """ransac_homography over many (src, dst) host point sets in one launch:
    returns [(H or None, inlier index list)] as the reference per problem."""
    srcs = [np.asarray(s, np.float64).reshape(-1, 2) for s, _ in problems]
    dsts = [np.asarray(d, np.float64).reshape(-1, 2) for _, d in problems]
    off = np.zeros(len(srcs) + 1, np.int64)
    off[1:] = np.cumsum([len(s) for s in srcs])
    if not srcs:
        return []
    src = _dev.to_dev(np.concatenate(srcs) if off[-1] else np.zeros((0, 2)))
    dst = _dev.to_dev(np.concatenate(dsts) if off[-1] else np.zeros((0, 2)))
    H, inl, cnt = ransac_homography_device(src, dst, off, iters, reproj_tol, seed)
    H, inl, cnt = H.cpu().numpy(), inl.cpu().numpy(), cnt.cpu().numpy()
    out = []
    for p in range(len(srcs)):
        if cnt[p] < 0:
            out.append((None, []))
        else:
            out.append((H[p].copy(), [int(i) for i in np.nonzero(inl[off[p]:off[p + 1]])[0]]))
    return out


def ransac_homography(matches: list[Match], query_kps, ref_kps, iters: int = 1000, reproj_tol: float = 3.0,
                      seed: int = 0):
    """matching.py:157-192: best-consensus homography mapping query points onto
    reference points, refit on the best consensus set.  Returns (H, inlier
    indices into matches); fewer than 4 matches or no usable model give
    (None, [])."""
    if len(matches) < 4:
        return None, []
    src = np.array([[query_kps[m.query_idx].x, query_kps[m.query_idx].y] for m in matches], np.float64)
    dst = np.array([[ref_kps[m.ref_idx].x, ref_kps[m.ref_idx].y] for m in matches], np.float64)
    return ransac_homography_batch([(src, dst)], iters, reproj_tol, seed)[0]


def match_and_verify(query: list[Feature], reference: list[Feature], cfg: MatchConfig):
    """matching.py:195-206: radius match + RANSAC; returns (H, inlier match list)."""
    return verify_batch([(query, reference)], cfg)[0]


def count_mpr(query: list[Feature], reference: list[Feature], t_m: int, ransac_cfg: MatchConfig) -> int:
    """matching.py:209-220: matches-post-RANSAC, the verified radius match's inlier count."""
    cfg = MatchConfig(t_m=t_m, iters=ransac_cfg.iters, reproj_tol=ransac_cfg.reproj_tol, seed=ransac_cfg.seed)
    return len(match_and_verify(query, reference, cfg)[1])


def verify_batch(pairs, cfg: MatchConfig):
    """match_and_verify for many (query, reference) feature-list pairs: each
    pair's radius match on the GPU, then ONE batched RANSAC launch over all
    pairs' match sets.  Returns [(H or None, inlier Match list)]."""
    sets, srcs, dsts = [], [], []
    for query, reference in pairs:
        ms = radius_match(query, reference, cfg.t_m)
        sets.append(ms)
        qi = np.fromiter((m.query_idx for m in ms), np.int64, len(ms))
        ri = np.fromiter((m.ref_idx for m in ms), np.int64, len(ms))
        qxy = np.array([[f.kp.x, f.kp.y] for f in query], np.float64).reshape(-1, 2)
        rxy = np.array([[f.kp.x, f.kp.y] for f in reference], np.float64).reshape(-1, 2)
        # fewer than 4 matches: (None, []) without a model (matching.py:166-167)
        srcs.append(qxy[qi] if len(ms) >= 4 else np.zeros((0, 2)))
        dsts.append(rxy[ri] if len(ms) >= 4 else np.zeros((0, 2)))
    res = ransac_homography_batch(list(zip(srcs, dsts)), cfg.iters, cfg.reproj_tol, cfg.seed)
    return [(h, [ms[i] for i in inl]) if h is not None else (None, []) for (h, inl), ms in zip(res, sets)]


def ransac_samples(seed: int, n: int, iters: int, device: bool = False) -> np.ndarray:
    """The (iters, 4) minimal-sample table ransac_homography draws for n
    matches: row k = the k-th default_rng(seed).choice(n, 4, replace=False).
    device=False runs the host generator (no GPU), True the CUDA one."""
    L = _native.lib()
    if device:
        t = _dev.torch()
        out = t.empty((max(int(iters), 0), 4), dtype=t.int32, device="cuda")
        _native.check(L.vf_ransac_samples(_check_seed(seed), int(n), int(iters), out.data_ptr(), _dev.stream()),
                      "vf_ransac_samples")
        return out.cpu().numpy()
    out = np.empty((max(int(iters), 0), 4), np.int32)
    _native.check(L.vf_ransac_samples_host(_check_seed(seed), int(n), int(iters), out.ctypes.data), "vf_ransac_samples")
    return out

"""Rotation-compensated 512-bit binary descriptors (drop-in for vidfeat.descriptor).

orientations_batch / describe_batch run the pipeline's warp-batched describe
kernel (vf_describe: strip SATs of the frame, per-lane sequential orientation
sums, __ballot_sync bit packing).  Reference: descriptor.py:1-285.
Serialization: 64 bytes, MSB-first (descriptor.py:271-285).
"""

from __future__ import annotations

import numpy as np

from . import _dev, _native
from .pattern import SamplingPattern, default_pattern
from .types import GrayFrame, Keypoint

DESCRIPTOR_BITS = 512
DESCRIPTOR_BYTES = 64

__all__ = ["FootprintError", "border_ok", "orientations_batch", "describe_batch", "describe_batch_packed",
           "estimate_orientation", "describe", "hamming", "pack_descriptor", "unpack_descriptor", "descriptor_hex",
           "DESCRIPTOR_BITS", "DESCRIPTOR_BYTES"]


class FootprintError(ValueError):
    """Keypoint too close to the layer border for descriptor sampling."""


def border_ok(layer: GrayFrame, kp: Keypoint) -> bool:
    """descriptor.py:183-191: the centre is at least 3*sigma from every border."""
    m = 3.0 * kp.sigma
    return kp.x >= m and kp.y >= m and kp.x <= layer.width - 1 - m and kp.y <= layer.height - 1 - m


def _check_pattern(pattern):
    if pattern is not None and pattern is not default_pattern():
        _native.ensure_pattern(pattern)


def _run(frame: np.ndarray, kx, ky, sg, theta=None, want_desc=True):
    H, W = frame.shape
    n = len(kx)
    t = _dev.torch()
    L = _dev.lib()
    if n == 0:
        return np.zeros(0), np.zeros((0, DESCRIPTOR_BYTES), np.uint8)
    f = _dev.to_dev(frame)
    dx = _dev.to_dev(np.asarray(kx, np.float64))
    dy = _dev.to_dev(np.asarray(ky, np.float64))
    ds = _dev.to_dev(np.asarray(sg, np.float64))
    dt = None if theta is None else _dev.to_dev(np.asarray(theta, np.float64))
    tho = _dev.empty(n, t.float64)
    desc = _dev.empty((n, DESCRIPTOR_BYTES), t.uint8) if want_desc else None
    _native.check(L.vf_describe(f.data_ptr(), W, H, W, n, dx.data_ptr(), dy.data_ptr(), ds.data_ptr(),
                                0 if dt is None else dt.data_ptr(), tho.data_ptr(),
                                0 if desc is None else desc.data_ptr(), _dev.stream()), "vf_describe")
    return tho.cpu().numpy(), (None if desc is None else desc.cpu().numpy())


def orientations_batch(layer: GrayFrame, kps: list[Keypoint], pattern: SamplingPattern | None = None,
                       sat=None) -> np.ndarray:
    """descriptor.py:194-209: orientation per keypoint (sequential long-pair sum, atan2)."""
    _check_pattern(pattern)
    th, _ = _run(layer.data, [k.x for k in kps], [k.y for k in kps], [k.sigma for k in kps], None, False)
    return th


def describe_batch_packed(layer: GrayFrame, kps: list[Keypoint], thetas, pattern: SamplingPattern | None = None
                          ) -> np.ndarray:
    """(n, 64) packed MSB-first descriptors at the given orientations."""
    _check_pattern(pattern)
    _, d = _run(layer.data, [k.x for k in kps], [k.y for k in kps], [k.sigma for k in kps],
                np.ascontiguousarray(thetas, np.float64), True)
    return d


def describe_batch(layer: GrayFrame, kps: list[Keypoint], thetas, pattern: SamplingPattern | None = None,
                   sat=None) -> np.ndarray:
    """descriptor.py:212-232: (n, 512) uint8 bit matrix."""
    d = describe_batch_packed(layer, kps, thetas, pattern)
    return np.unpackbits(d, axis=1) if len(d) else np.zeros((0, DESCRIPTOR_BITS), np.uint8)


def estimate_orientation(layer: GrayFrame, kp: Keypoint, pattern: SamplingPattern | None = None) -> float:
    """descriptor.py:235-244."""
    if not border_ok(layer, kp):
        raise FootprintError(f"keypoint ({kp.x:.1f}, {kp.y:.1f}, sigma={kp.sigma:.2f}) too close to border")
    return float(orientations_batch(layer, [kp], pattern)[0])


def describe(layer: GrayFrame, kp: Keypoint, theta: float, pattern: SamplingPattern | None = None) -> np.ndarray:
    """descriptor.py:247-259: 512-element 0/1 uint8 descriptor."""
    if not border_ok(layer, kp):
        raise FootprintError(f"keypoint ({kp.x:.1f}, {kp.y:.1f}, sigma={kp.sigma:.2f}) too close to border")
    return describe_batch(layer, [kp], np.array([theta]), pattern)[0]


def hamming(a: np.ndarray, b: np.ndarray) -> int:
    """descriptor.py:262-268 (a matching utility; host-side, outside the hot path)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        raise ValueError(f"descriptor length mismatch: {a.shape} vs {b.shape}")
    return int(np.count_nonzero(a != b))


def pack_descriptor(bits: np.ndarray) -> bytes:
    """64 bytes, MSB-first within each byte; bit 0 is the first byte's MSB."""
    if bits.shape != (DESCRIPTOR_BITS,):
        raise ValueError("descriptor must have exactly 512 bits")
    return np.packbits(bits.astype(np.uint8)).tobytes()


def unpack_descriptor(raw: bytes) -> np.ndarray:
    if len(raw) != DESCRIPTOR_BYTES:
        raise ValueError("packed descriptor must be exactly 64 bytes")
    return np.unpackbits(np.frombuffer(raw, np.uint8))


def descriptor_hex(bits: np.ndarray) -> str:
    return pack_descriptor(bits).hex()

"""Device-buffer helpers: numpy <-> torch CUDA tensors for the C-ABI calls.

PyTorch is the buffer carrier only (allocation, H2D/D2H, streams); every
computation is a call into the sm_100a library.
"""

from __future__ import annotations

import numpy as np

from . import _native


def torch():
    import torch as _t

    if not _t.cuda.is_available():
        raise RuntimeError("vidfeat-b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    return _t


def to_dev(a: np.ndarray):
    t = torch()
    return t.from_numpy(np.ascontiguousarray(a)).cuda()


def empty(shape, dtype):
    t = torch()
    return t.empty(shape, dtype=dtype, device="cuda")


def zeros(shape, dtype):
    t = torch()
    return t.zeros(shape, dtype=dtype, device="cuda")


def stream() -> int:
    return _native.stream_handle()


def sync():
    torch().cuda.current_stream().synchronize()


def lib():
    _native.ensure_pattern()
    return _native.lib()

"""FeatureEngine: one C-ABI context (vf_ctx) processing S independent streams.

This is the batched form of the reference's per-frame loop body
(pipeline.py:222-277): every call processes frame n of each stream with one
launch per stage over all streams.  Device memory, streams and the
torch.distributed plumbing belong to PyTorch; all compute is the sm_100a
library.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .types import MaskConfig, PipelineConfig


class _CudaArray:
    """Zero-copy __cuda_array_interface__ view of library-owned device memory."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {
            "shape": tuple(shape), "typestr": typestr, "data": (int(ptr), True), "version": 3, "strides": None,
        }


def _mode(mc: MaskConfig) -> int:
    return _native.MODES[mc.mode]


def gop_fields(gop) -> dict:
    """GopConfig -> the vf_config gop_* fields (None = reference defaults)."""
    from .types import GopConfig

    g = gop if gop is not None else GopConfig()
    return dict(gop_delta=int(g.delta), gop_patch=int(g.patch), gop_t_bm=float(g.t_bm), gop_t_et=float(g.t_et),
                gop_coarse_window=float(g.coarse_window), gop_coarse_step=float(g.coarse_step),
                gop_fine_window=float(g.fine_window), gop_fine_step=float(g.fine_step))


class FeatureEngine:
    def __init__(self, width: int, height: int, cfg: PipelineConfig | None = None, n_streams: int = 1,
                 kp_capacity: int = 0):
        cfg = cfg or PipelineConfig()
        mc = cfg.mask
        if cfg.threshold < 1:
            raise ValueError("detection threshold must be >= 1")
        c = _native.VfConfig(
            width=width, height=height, n_octaves=cfg.n_octaves, threshold=int(cfg.threshold),
            mask_mode=_mode(mc), t_i=float(mc.t_i), t_h=int(mc.t_h), grid_rows=int(mc.grid[0]),
            grid_cols=int(mc.grid[1]), octave_for_mask=-1 if mc.octave_for_mask is None else int(mc.octave_for_mask),
            per_layer=int(bool(mc.per_layer)), max_streams=int(n_streams), kp_capacity=int(kp_capacity),
            **gop_fields(getattr(cfg, "gop", None)))
        L = _native.lib()
        _native.ensure_pattern()
        h = ctypes.c_void_p()
        _native.check(L.vf_create(ctypes.byref(c), ctypes.byref(h)), "vf_create")
        self._h = h
        self.width, self.height, self.n_streams, self.cfg = width, height, n_streams, cfg
        n_layers = 2 * cfg.n_octaves
        ws = np.zeros(n_layers, np.int32)
        hs = np.zeros(n_layers, np.int32)
        sc = np.zeros(n_layers, np.float64)
        _native.check(L.vf_layer_geometry(self._h, ws.ctypes.data, hs.ctypes.data, sc.ctypes.data))
        self.layer_w, self.layer_h, self.layer_scale = ws, hs, sc

    # -- processing -----------------------------------------------------------
    def process(self, frames, stream=None, check: bool = False) -> None:
        """frames: CUDA uint8 tensor [S, H, W] (or [H, W] for S = 1), device-resident.

        check=True synchronizes after the step and, if a stream's features
        overflowed the capacity, grows it and replays the step from the saved
        state (vf_process_checked); the default leaves the step asynchronous
        and a capacity overflow is reported by report()/features calls."""
        import torch

        if frames.dim() == 2:
            frames = frames.unsqueeze(0)
        if frames.dtype != torch.uint8 or not frames.is_cuda:
            raise ValueError("frames must be a CUDA uint8 tensor")
        S, H, W = frames.shape
        if (H, W) != (self.height, self.width):
            raise ValueError(f"frame {W}x{H} does not match the engine's {self.width}x{self.height}")
        if frames.stride(2) != 1:
            frames = frames.contiguous()
        fn = _native.lib().vf_process_checked if check else _native.lib().vf_process
        _native.check(fn(self._h, frames.data_ptr(), frames.stride(0), frames.stride(1), S, _native.stream_handle(stream)),
                      "vf_process")

    @property
    def kp_capacity(self) -> int:
        n = ctypes.c_int32(0)
        _native.check(_native.lib().vf_get_capacity(self._h, ctypes.byref(n)))
        return int(n.value)

    def process_host(self, frames: np.ndarray, stream=None) -> None:
        """frames: host uint8 array [S, H, W]; the H2D copy is part of the call."""
        a = np.ascontiguousarray(frames)
        if a.ndim == 2:
            a = a[None]
        S, H, W = a.shape
        _native.check(_native.lib().vf_process_host(self._h, a.ctypes.data, H * W, W, S, _native.stream_handle(stream)),
                      "vf_process_host")

    def reset(self, stream=None) -> None:
        _native.check(_native.lib().vf_reset(self._h, _native.stream_handle(stream)))

    # -- results ----------------------------------------------------------------
    def report(self, s: int = 0, stream=None) -> _native.VfReport:
        r = _native.VfReport()
        _native.check(_native.lib().vf_get_report(self._h, s, ctypes.byref(r), _native.stream_handle(stream)),
                      "vf_get_report")
        return r

    def totals(self, s: int = 0, stream=None) -> np.ndarray:
        out = np.zeros(4, np.float64)
        _native.check(_native.lib().vf_get_totals(self._h, s, out.ctypes.data, _native.stream_handle(stream)))
        return out

    def features_device(self, s: int = 0, stream=None) -> dict:
        """Zero-copy torch views of stream s's current features (valid until the next process)."""
        import torch

        f = _native.VfFeatures()
        _native.check(_native.lib().vf_get_features(self._h, s, ctypes.byref(f), _native.stream_handle(stream)))
        n = int(f.n)
        out = {"n": n}
        if n == 0:
            dev = torch.device("cuda")
            for k, dt in (("x", torch.float64), ("y", torch.float64), ("sigma", torch.float64),
                          ("theta", torch.float64), ("score", torch.float64), ("origin", torch.uint8),
                          ("age", torch.int32)):
                out[k] = torch.zeros(0, dtype=dt, device=dev)
            out["desc"] = torch.zeros((0, 64), dtype=torch.uint8, device=dev)
            return out
        for k, ts in (("x", "<f8"), ("y", "<f8"), ("sigma", "<f8"), ("theta", "<f8"), ("score", "<f8"),
                      ("origin", "|u1"), ("age", "<i4")):
            out[k] = torch.as_tensor(_CudaArray(getattr(f, k), (n,), ts), device="cuda")
        out["desc"] = torch.as_tensor(_CudaArray(f.desc, (n, 64), "|u1"), device="cuda")
        return out

    def features_host(self, s: int = 0, stream=None) -> dict:
        """Copy stream s's current features into numpy arrays (synchronizes)."""
        f = _native.VfFeatures()
        L = _native.lib()
        _native.check(L.vf_get_features(self._h, s, ctypes.byref(f), _native.stream_handle(stream)))
        n = int(f.n)
        out = {k: np.zeros(n, np.float64) for k in ("x", "y", "sigma", "theta", "score")}
        out["origin"] = np.zeros(n, np.uint8)
        out["age"] = np.zeros(n, np.int32)
        out["desc"] = np.zeros((n, 64), np.uint8)
        got = ctypes.c_int32(0)
        _native.check(L.vf_copy_features(
            self._h, s, n, out["x"].ctypes.data, out["y"].ctypes.data, out["sigma"].ctypes.data,
            out["theta"].ctypes.data, out["score"].ctypes.data, out["origin"].ctypes.data, out["age"].ctypes.data,
            out["desc"].ctypes.data, ctypes.byref(got), _native.stream_handle(stream)), "vf_copy_features")
        out["n"] = n
        return out

    def fetch_all(self, out: dict | None = None, stream=None) -> dict:
        """Every stream's current features in one packed SoA (host arrays; pinned if `out` was
        made by alloc_host).  out["offsets"][s] .. [s+1] is stream s.  Synchronize before use."""
        if out is None:
            out = self.alloc_host(self.n_streams * 65536)
        n = ctypes.c_int64(len(out["x"]))
        _native.check(_native.lib().vf_fetch_features(
            self._h, self.n_streams, n, out["x"].ctypes.data, out["y"].ctypes.data, out["sigma"].ctypes.data,
            out["theta"].ctypes.data, out["score"].ctypes.data, out["origin"].ctypes.data, out["age"].ctypes.data,
            out["desc"].ctypes.data, out["offsets"].ctypes.data, _native.stream_handle(stream)), "vf_fetch_features")
        return out

    def submit(self, frames: np.ndarray) -> None:
        """Pipelined e2e API: enqueue host frames [S, H, W] (pinned for overlap) for one step."""
        a = np.ascontiguousarray(frames)
        if a.ndim == 2:
            a = a[None]
        S, H, W = a.shape
        self._keep = getattr(self, "_keep", [])[-2:] + [a]   # host memory must live until its copy ran (3 in flight)
        _native.check(_native.lib().vf_pipeline_submit(self._h, a.ctypes.data, H * W, W, S), "vf_pipeline_submit")

    def collect(self, out: dict) -> dict:
        """Features of the oldest submitted step (packed SoA, see fetch_all); blocks until copied."""
        n = ctypes.c_int64(len(out["x"]))
        _native.check(_native.lib().vf_pipeline_collect(
            self._h, n, out["x"].ctypes.data, out["y"].ctypes.data, out["sigma"].ctypes.data, out["theta"].ctypes.data,
            out["score"].ctypes.data, out["origin"].ctypes.data, out["age"].ctypes.data, out["desc"].ctypes.data,
            out["offsets"].ctypes.data), "vf_pipeline_collect")
        return out

    def set_delta(self, enable: bool = True) -> None:
        """Pipelined API: collect_delta returns new records + keep masks (see vf_pipeline_collect_delta)."""
        _native.check(_native.lib().vf_pipeline_set_delta(self._h, int(enable)), "vf_pipeline_set_delta")

    def collect_delta(self, out: dict) -> dict:
        """The oldest submitted step's result as a delta: out["x"..] detected records (packed over streams,
        out["offsets"]), out["keep"] keep-mask words (out["keep_offsets"]), out["counts"] [S, 3]."""
        n = ctypes.c_int64(len(out["x"]))
        _native.check(_native.lib().vf_pipeline_collect_delta(
            self._h, n, out["x"].ctypes.data, out["y"].ctypes.data, out["sigma"].ctypes.data, out["theta"].ctypes.data,
            out["score"].ctypes.data, out["desc"].ctypes.data, out["offsets"].ctypes.data, len(out["keep"]),
            out["keep"].ctypes.data, out["keep_offsets"].ctypes.data, out["counts"].ctypes.data),
            "vf_pipeline_collect_delta")
        return out

    def alloc_delta(self, cap: int, pinned: bool = True) -> dict:
        """Host buffers for collect_delta (pinned)."""
        import torch

        out = self.alloc_host(cap, pinned)
        kw = self.n_streams * (max(self.kp_capacity, cap) // 32 + 2)
        out["keep"] = torch.empty(kw, dtype=torch.int32, pin_memory=pinned).numpy().view(np.uint32)
        out["keep_offsets"] = np.zeros(self.n_streams + 1, np.int32)
        out["counts"] = np.zeros((self.n_streams, 3), np.int32)
        return out

    @staticmethod
    def delta_apply(prev: dict, delta: dict, s: int) -> dict:
        """Stream s's merged list from its previous list (SoA dict) and a collect_delta result."""
        a, b = int(delta["offsets"][s]), int(delta["offsets"][s + 1])
        ka, kb = int(delta["keep_offsets"][s]), int(delta["keep_offsets"][s + 1])
        nbits = int(delta["counts"][s][2])
        n_det = b - a
        cap = n_det + nbits
        out = {k: np.zeros(cap, np.float64) for k in ("x", "y", "sigma", "theta", "score")}
        out["origin"] = np.zeros(cap, np.uint8)
        out["age"] = np.zeros(cap, np.int32)
        out["desc"] = np.zeros((cap, 64), np.uint8)
        n_prev = len(prev["x"])
        pv = {k: np.ascontiguousarray(prev[k]) for k in ("x", "y", "sigma", "theta", "score", "origin", "age", "desc")}
        dv = {k: np.ascontiguousarray(delta[k][a:b]) for k in ("x", "y", "sigma", "theta", "score", "desc")}
        keep = np.ascontiguousarray(delta["keep"][ka:kb])
        n_out = ctypes.c_int32(0)
        _native.check(_native.lib().vf_delta_apply(
            n_prev, *(pv[k].ctypes.data for k in ("x", "y", "sigma", "theta", "score", "origin", "age", "desc")),
            n_det, *(dv[k].ctypes.data for k in ("x", "y", "sigma", "theta", "score", "desc")), nbits,
            keep.ctypes.data, cap, *(out[k].ctypes.data for k in ("x", "y", "sigma", "theta", "score", "origin", "age",
                                                                  "desc")), ctypes.byref(n_out)), "vf_delta_apply")
        n = int(n_out.value)
        res = {k: v[:n] for k, v in out.items()}
        res["n"] = n
        return res

    @staticmethod
    def alloc_host(cap: int, pinned: bool = True) -> dict:
        """Host SoA buffers for fetch_all (torch pinned memory viewed as numpy)."""
        import torch

        def arr(shape, dt):
            t = torch.empty(shape, dtype=dt, pin_memory=pinned)
            return t.numpy()

        out = {k: arr(cap, torch.float64) for k in ("x", "y", "sigma", "theta", "score")}
        out["origin"] = arr(cap, torch.uint8)
        out["age"] = arr(cap, torch.int32)
        out["desc"] = arr((cap, 64), torch.uint8)
        out["offsets"] = np.zeros(4096 + 1, np.int32)
        return out

    STAGES = ("binmask", "pyramid", "worklist", "fast", "nms", "sat", "describe", "propagate", "finalize")

    def set_history(self, hist=None) -> None:
        """Record every later frame's FrameReport row on the device into `hist`
        (a CUDA float64 tensor [n_streams, max_frames, 8]: n_detected,
        n_propagated, n_total, n_dropped, coverage, frame, n_survivors,
        n_candidates); None turns it off.  No host synchronization per frame."""
        import torch

        if hist is None:
            _native.check(_native.lib().vf_set_history(self._h, None, 0))
            self._hist = None
            return
        if (hist.dtype != torch.float64 or not hist.is_cuda or hist.dim() != 3 or hist.shape[0] != self.n_streams
                or hist.shape[2] != 8 or not hist.is_contiguous()):
            raise ValueError("history must be a contiguous CUDA float64 tensor [n_streams, max_frames, 8]")
        self._hist = hist   # keep the buffer alive while the library writes into it
        _native.check(_native.lib().vf_set_history(self._h, hist.data_ptr(), int(hist.shape[1])))

    def set_timing(self, enable: bool) -> None:
        _native.check(_native.lib().vf_set_timing(self._h, int(enable)))

    def stage_ms(self, stream=None) -> tuple[dict, int]:
        """Summed per-stage device ms since the last call, and the step count."""
        out = np.zeros(len(self.STAGES), np.float64)
        n = ctypes.c_int32(0)
        _native.check(_native.lib().vf_get_stage_ms(self._h, out.ctypes.data, ctypes.byref(n),
                                                    _native.stream_handle(stream)))
        return dict(zip(self.STAGES, out.tolist())), int(n.value)

    def diag(self, stream=None) -> dict:
        out = np.zeros(8, np.int64)
        _native.check(_native.lib().vf_get_diag(self._h, out.ctypes.data, _native.stream_handle(stream)))
        keys = ("fast_tiles_active", "fast_tiles", "sat_tiles_built", "sat_tiles", "dense_streams",
                "nms_candidates", "bands_per_stream", "kp_capacity")
        return dict(zip(keys, out.tolist()))

    def close(self) -> None:
        if getattr(self, "_h", None):
            _native.lib().vf_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

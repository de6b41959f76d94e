"""Per-frame orchestration (drop-in for vidfeat.pipeline.run_pipeline).

run_pipeline keeps the reference signature and outputs
(pipeline.py:207-278): list of per-frame Feature lists + FrameReports.  Each
frame is one FeatureEngine step (all stages on the GPU, one launch per
stage); FrameReport stage times come from CUDA events on the launch stream.

run_streams is the batched form for independent streams (BASELINE configs 3
and 5): one step processes frame n of every stream.  Its per-stream output
equals run_pipeline on that stream alone.
"""

from __future__ import annotations

import time

import numpy as np

from .engine import FeatureEngine
from .types import DETECTED, PROPAGATED, Feature, FrameReport, GrayFrame, Keypoint, MaskConfig, PipelineConfig

__all__ = ["PipelineConfig", "FrameReport", "run_pipeline", "run_pipeline_arrays", "run_streams", "features_from_arrays"]


def features_from_arrays(f: dict) -> list[Feature]:
    """SoA arrays (engine.features_host) -> reference Feature objects (512-bit unpacked desc)."""
    n = f["n"]
    if n == 0:
        return []
    bits = np.unpackbits(f["desc"], axis=1)
    x, y, s, t, v = (f[k].tolist() for k in ("x", "y", "sigma", "theta", "score"))
    org = f["origin"].tolist()
    age = f["age"].tolist()
    return [Feature(Keypoint(x[i], y[i], s[i], t[i], v[i]), bits[i], PROPAGATED if org[i] else DETECTED, age[i])
            for i in range(n)]


def _report(n, r, stage: dict, wall_ms: float) -> FrameReport:
    return FrameReport(
        frame=n, n_detected=r.n_detected, n_propagated=r.n_propagated, n_total=r.n_total, coverage=r.coverage,
        t_pyramid_ms=stage["pyramid"], t_mask_ms=stage["binmask"] + stage["worklist"],
        t_detect_ms=stage["fast"] + stage["nms"], t_describe_ms=stage["sat"] + stage["describe"] + stage["propagate"],
        t_total_ms=sum(stage.values()), t_wall_ms=wall_ms, n_dropped=r.n_dropped)


def run_pipeline_arrays(frames: list[GrayFrame], cfg: PipelineConfig):
    """run_pipeline with SoA outputs (no per-feature Python objects)."""
    import torch

    if not frames:
        raise ValueError("empty frame sequence")
    H, W = frames[0].data.shape
    eng = FeatureEngine(W, H, cfg, n_streams=1)
    eng.set_timing(True)
    outs, reports = [], []
    try:
        for n, fr in enumerate(frames):
            if fr.data.shape != (H, W):
                raise ValueError("all frames of a sequence must have the same size")
            wall0 = time.perf_counter_ns()
            dev = torch.from_numpy(np.ascontiguousarray(fr.data)).cuda(non_blocking=False)
            eng.process(dev, check=True)
            r = eng.report(0)
            stage, _ = eng.stage_ms()
            f = eng.features_host(0)
            outs.append(f)
            reports.append(_report(n, r, stage, (time.perf_counter_ns() - wall0) / 1e6))
    finally:
        eng.close()
    return outs, reports


def run_pipeline(frames: list[GrayFrame], cfg: PipelineConfig) -> tuple[list[list[Feature]], list[FrameReport]]:
    """Extract features from every frame under the configured mode (pipeline.py:207-278)."""
    outs, reports = run_pipeline_arrays(frames, cfg)
    return [features_from_arrays(f) for f in outs], reports


def run_streams(frames, cfg: PipelineConfig, collect: bool = True):
    """frames: uint8 [S, N, H, W] (numpy, or torch CUDA tensor kept on device).

    Returns (per-stream list of per-frame SoA dicts (if collect), per-stream
    list of FrameReports).  Stream s's results equal run_pipeline(frames[s]).
    """
    import torch

    if isinstance(frames, np.ndarray):
        frames_t = torch.from_numpy(np.ascontiguousarray(frames))
    else:
        frames_t = frames
    S, N, H, W = frames_t.shape
    if N == 0:
        raise ValueError("empty frame sequence")
    eng = FeatureEngine(W, H, cfg, n_streams=S)
    feats = [[] for _ in range(S)]
    reps = [[] for _ in range(S)]
    try:
        for n in range(N):
            batch = frames_t[:, n]
            if not batch.is_cuda:
                batch = batch.cuda()
            eng.process(batch.contiguous(), check=True)
            for s in range(S):
                r = eng.report(s)
                reps[s].append(FrameReport(frame=n, n_detected=r.n_detected, n_propagated=r.n_propagated,
                                           n_total=r.n_total, coverage=r.coverage, t_pyramid_ms=0.0, t_mask_ms=0.0,
                                           t_detect_ms=0.0, t_describe_ms=0.0, t_total_ms=0.0, n_dropped=r.n_dropped))
                if collect:
                    feats[s].append(eng.features_host(s))
    finally:
        eng.close()
    return feats, reps

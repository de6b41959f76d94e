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
from dataclasses import dataclass, replace

import numpy as np

from .engine import FeatureEngine
from .types import DETECTED, PROPAGATED, Feature, FrameReport, GrayFrame, Keypoint, MaskConfig, PipelineConfig

__all__ = ["PipelineConfig", "FrameReport", "DivergenceStat", "run_pipeline", "run_pipeline_arrays", "run_streams",
           "features_from_arrays", "divergence_report", "divergence_from_arrays"]


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


# ---------------------------------------------------------------------------
# divergence_report (pipeline.py:348-398): masked vs full detection, paired
# keypoints.  Both runs are GPU pipelines; the greedy pairing is host code
# over the two SoA lists (it is sequential by definition: each masked
# keypoint takes the nearest unused full keypoint in list order).
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class DivergenceStat:
    """pipeline.py:74-85."""

    frame: int
    only_masked: int
    only_full: int
    common: int

    @property
    def preserved(self) -> float:
        """Fraction of full-detection keypoints present in the masked run."""
        denom = self.common + self.only_full
        return 1.0 if denom == 0 else self.common / denom


def _match_keypoint_sets(masked: dict, full: dict, pos_tol: float = 1.0, scale_ratio_tol: float = 1.2):
    """pipeline.py:348-381 on SoA dicts (x, y, sigma): greedy pairing within
    pos_tol (Euclidean, <=) and scale ratio <= scale_ratio_tol, candidates
    scanned cell by cell (integer-truncated positions, cells within
    ceil(pos_tol)) and, inside a cell, in full-list order; a later candidate
    at an equal distance replaces the earlier one (the reference's <=).
    Returns (common, only_masked, only_full)."""
    nm, nf = len(masked["x"]), len(full["x"])
    if nm == 0 or nf == 0:
        return 0, nm, nf
    fx, fy, fs = full["x"], full["y"], full["sigma"]
    cx_f = fx.astype(np.int64)   # int(f.kp.x): truncation toward zero
    cy_f = fy.astype(np.int64)
    order = np.lexsort((np.arange(nf), cx_f, cy_f))
    keys = cy_f[order] * (1 << 32) + cx_f[order]
    used = np.zeros(nf, bool)
    reach = int(np.ceil(pos_tol))
    mx, my, ms = masked["x"].tolist(), masked["y"].tolist(), masked["sigma"].tolist()
    common = 0
    for i in range(nm):
        x, y, sg = mx[i], my[i], ms[i]
        cx, cy = int(x), int(y)
        best_j, best_d = -1, pos_tol
        for gy in range(cy - reach, cy + reach + 1):
            for gx in range(cx - reach, cx + reach + 1):
                k = gy * (1 << 32) + gx
                a = np.searchsorted(keys, k, "left")
                b = np.searchsorted(keys, k, "right")
                for j in order[a:b]:
                    if used[j]:
                        continue
                    d = float(np.hypot(fx[j] - x, fy[j] - y))
                    ratio = max(fs[j], sg) / min(fs[j], sg)
                    if d <= best_d and ratio <= scale_ratio_tol:
                        best_d, best_j = d, j
        if best_j >= 0:
            used[best_j] = True
            common += 1
    return common, nm - common, nf - common


def divergence_from_arrays(masked_frames: list[dict], full_frames: list[dict]) -> list[DivergenceStat]:
    out = []
    for n, (m, f) in enumerate(zip(masked_frames, full_frames)):
        common, only_m, only_f = _match_keypoint_sets(m, f)
        out.append(DivergenceStat(n, only_m, only_f, common))
    return out


def divergence_report(frames: list[GrayFrame], cfg: PipelineConfig) -> list[DivergenceStat]:
    """pipeline.py:384-398: run the masked and the full (mode none) pipelines
    on the GPU side by side and diff their outputs (1 px / 1.2x pairing)."""
    full_cfg = replace(cfg, mask=replace(cfg.mask, mode="none"))
    masked, _ = run_pipeline_arrays(frames, cfg)
    full, _ = run_pipeline_arrays(frames, full_cfg)
    return divergence_from_arrays(masked, full)

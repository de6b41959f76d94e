"""GPU parity at the BASELINE.json configs' real frame sizes (seeded scenes),
against the pinned CPU oracle on frame prefixes, plus size-independent
properties at full size (determinism, all-ones-mask identity, batch = single).

Prefixes keep the CPU oracle to seconds (SURVEY.md 8(d) parity coverage):
config 3: 8 streams x 3 frames; config 4: 3 frames of 4K fresh noise; config 5:
6 streams (static / pan / objects) x 3 frames, all three modes."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_batch(frames, mode, **kw):
    import torch

    from paper_1503_06959_b200.engine import FeatureEngine
    from paper_1503_06959_b200.types import MaskConfig, PipelineConfig

    S, N, H, W = frames.shape
    eng = FeatureEngine(W, H, PipelineConfig(mask=MaskConfig(mode=mode, **kw)), n_streams=S)
    dev = torch.from_numpy(np.ascontiguousarray(frames.transpose(1, 0, 2, 3))).cuda()
    outs = [[None] * N for _ in range(S)]
    reps = [[None] * N for _ in range(S)]
    for n in range(N):
        eng.process(dev[n])
        for s in range(S):
            reps[s][n] = eng.report(s)
            outs[s][n] = eng.features_host(s)
    eng.close()
    return outs, reps


def _check_vs_oracle(frames, mode, label, **kw):
    from oracle import oracle
    from paper_1503_06959_b200.pattern import default_pattern

    outs, reps = _run_batch(frames, mode, **kw)
    for s in range(frames.shape[0]):
        ref = oracle.run_sequence(list(frames[s]), default_pattern(), mode=mode, **kw)
        for n, e in enumerate(ref):
            o, r = outs[s][n], reps[s][n]
            where = f"{label} stream {s} frame {n}"
            assert r.n_total == e.n_total and r.n_detected == e.n_detected, where
            assert r.n_dropped == e.n_dropped and r.coverage == e.coverage, where
            for k in ("x", "y", "score", "origin", "age", "desc"):
                assert np.array_equal(o[k], getattr(e, k)), f"{where}: {k}"
            assert np.abs(o["sigma"] - e.sigma).max(initial=0) <= 1e-4, where
            assert np.abs(o["theta"] - e.theta).max(initial=0) <= 1e-4, where


def test_config3_batch_of_8_1080p():
    from paper_1503_06959_b200 import scenes

    frames = scenes.generate(scenes.CONFIGS[3], 3).numpy()
    _check_vs_oracle(frames, "intensity", "config3")


def test_config4_4k_fresh_noise():
    from paper_1503_06959_b200 import scenes

    frames = scenes.generate(scenes.CONFIGS[4], 3).numpy()
    _check_vs_oracle(frames, "intensity", "config4")


@pytest.mark.parametrize("mode", ["intensity", "binning", "none"])
def test_config5_mixed_streams(mode):
    from paper_1503_06959_b200 import scenes

    frames = scenes.generate(scenes.CONFIGS[5], 3, streams=range(6)).numpy()
    _check_vs_oracle(frames, mode, f"config5/{mode}")


def test_config4_full_coverage_every_frame():
    """Config 4's scene must select every top-octave cell after frame 0 (BASELINE.json)."""
    from paper_1503_06959_b200 import scenes

    frames = scenes.generate(scenes.CONFIGS[4], 4).numpy()
    _, reps = _run_batch(frames, "intensity")
    assert all(r.coverage == 1.0 for r in reps[0][1:])


def test_config2_coverage_range():
    """Config 2 (panning 720p): per-frame active fraction within BASELINE.json's 10-60% band
    (median inside it, no frame above it; a sub-pixel pan step can give a quieter frame)."""
    from paper_1503_06959_b200 import scenes

    frames = scenes.generate(scenes.CONFIGS[2], 12).numpy()
    _, reps = _run_batch(frames, "intensity")
    cov = [r.coverage for r in reps[0][1:]]
    assert 0.10 <= float(np.median(cov)) <= 0.60 and max(cov) <= 0.60, cov


def test_full_size_determinism_and_gating_identity():
    """1080p batch: repeated runs identical; an all-ones mask (t_i = -1) equals mode none (c01)."""
    from paper_1503_06959_b200 import scenes

    frames = scenes.generate(scenes.CONFIGS[5], 4, streams=range(3)).numpy()
    a, _ = _run_batch(frames, "intensity")
    b, _ = _run_batch(frames, "intensity")
    c, rc = _run_batch(frames, "none")
    d, rd = _run_batch(frames, "intensity", t_i=-1.0)
    for s in range(3):
        for n in range(4):
            for k in ("x", "y", "sigma", "theta", "score", "origin", "age", "desc"):
                assert np.array_equal(a[s][n][k], b[s][n][k])
                assert np.array_equal(c[s][n][k], d[s][n][k])
            assert rd[s][n].coverage == 1.0


@pytest.mark.parametrize("cfg_id,mode,n_frames,streams", [(5, "intensity", 6, range(6)), (5, "none", 3, range(3)),
                                                           (4, "intensity", 3, None), (2, "intensity", 10, None)])
def test_early_sat_marks_cover_every_kept_footprint(cfg_id, mode, n_frames, streams, monkeypatch):
    """Early SAT (k_fast marks SAT tiles from footprint bounds of its candidates, k_sat runs beside the
    NMS): with VF_SAT_CHECK=1 k_nms_test asserts on the device that every tile a kept keypoint's
    descriptor reads was marked (a miss sets a sticky error bit and the fetch raises); the features
    must equal the oracle's, and those of the late arrangement (VF_SAT_EARLY=0), bit for bit."""
    from paper_1503_06959_b200 import scenes

    kw = {"streams": streams} if streams is not None else {}
    frames = scenes.generate(scenes.CONFIGS[cfg_id], n_frames, **kw).numpy()
    monkeypatch.setenv("VF_SAT_EARLY", "1")
    monkeypatch.setenv("VF_SAT_CHECK", "1")
    _check_vs_oracle(frames, mode, f"config{cfg_id}/{mode}/early-sat")
    early, _ = _run_batch(frames, mode)
    monkeypatch.setenv("VF_SAT_EARLY", "0")
    late, _ = _run_batch(frames, mode)
    for s in range(frames.shape[0]):
        for n in range(n_frames):
            for k in ("x", "y", "sigma", "theta", "score", "origin", "age", "desc"):
                assert np.array_equal(early[s][n][k], late[s][n][k]), (s, n, k)

"""GPU parity at the SURVEY.md 8(d) coverage lengths, frame by frame in lock
step with the CPU oracle (oracle/vf_oracle.c, pinned to the reference's
golden vectors in test_oracle_golden.py):

  config 1  640x480, all 100 frames, modes intensity / binning / none
  config 2  1280x720 pan, all 300 frames (intensity)
  config 3  all 8 1080p streams x 50 frames, plus stream 0 at its full 200 frames
  config 4  3840x2160 fresh noise, 20 frames (dense: every cell active)
  config 5  all 64 1080p streams x 10 frames, plus 8 full-length 300-frame
            streams across the three scene kinds
  bench     the bench's CUDA-generated config-5 frames 0-24 (a stream sample)

The temporal state accumulates (pipeline.py:276-277: the merged list feeds
the next frame), so every run starts at frame 0 and every frame is compared:
counts, coverage, order, origin, age, x, y, score and packed descriptors
exactly; sigma and theta within abs 1e-4 (north_star).  Frames are generated
on the fly (CPU scene generator) and never stored for the whole run."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _threads():
    import os

    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return os.cpu_count() or 1


def _compare(o, e, where):
    assert o["n"] == e.n_total, f"{where}: n_total {o['n']} vs {e.n_total}"
    for k in ("x", "y", "score", "origin", "age"):
        assert np.array_equal(o[k], getattr(e, k)), f"{where}: {k}"
    bad = np.nonzero((o["desc"] != e.desc).any(1))[0]
    assert bad.size == 0, f"{where}: {bad.size} descriptors differ (first {bad[:5]})"
    for k in ("sigma", "theta"):
        d = np.abs(o[k] - getattr(e, k))
        assert d.size == 0 or d.max() <= TOL, f"{where}: {k} max diff {d.max()}"


def lockstep(cfg, streams, n_frames, mode="intensity", source=None, kp_capacity=0):
    """Run `streams` of scene config `cfg` for n_frames through the engine (one
    batch) and the oracle (one pipeline per stream, host threads), comparing
    every frame.  source(n) -> uint8 [S, H, W] overrides the CPU generator."""
    import torch

    from oracle import oracle
    from paper_1503_06959_b200 import scenes
    from paper_1503_06959_b200.engine import FeatureEngine
    from paper_1503_06959_b200.pattern import default_pattern
    from paper_1503_06959_b200.types import MaskConfig, PipelineConfig

    S, W, H = len(streams), cfg.width, cfg.height
    pat = default_pattern()
    pool = ThreadPoolExecutor(max_workers=min(S, _threads()))
    gens = None if source is not None else list(pool.map(lambda s: scenes.SceneStream(cfg, s, "cpu"), streams))
    pipes = [oracle.OraclePipeline(W, H, pat, mode=mode) for _ in streams]
    eng = FeatureEngine(W, H, PipelineConfig(mask=MaskConfig(mode=mode)), n_streams=S, kp_capacity=kp_capacity)
    out = eng.alloc_host(S * max(65536, W * H // 8))
    checked = 0
    try:
        for n in range(n_frames):
            if source is None:
                host = np.stack(list(pool.map(lambda g: g.next_frame().numpy(), gens)))
            else:
                host = np.ascontiguousarray(source(n))
            eng.process(torch.from_numpy(host).cuda(), check=True)
            ref = list(pool.map(lambda i: pipes[i].process(host[i]), range(S)))
            eng.fetch_all(out)
            torch.cuda.synchronize()
            off = out["offsets"]
            for i in range(S):
                a, b = int(off[i]), int(off[i + 1])
                o = {k: out[k][a:b] for k in ("x", "y", "sigma", "theta", "score", "origin", "age", "desc")}
                o["n"] = b - a
                r, e = eng.report(i), ref[i]
                where = f"{mode} stream {streams[i]} frame {n}"
                assert (r.n_detected, r.n_propagated, r.n_total, r.n_dropped) == (
                    e.n_detected, e.n_propagated, e.n_total, e.n_dropped), where
                assert r.coverage == e.coverage, where
                _compare(o, e, where)
                checked += 1
    finally:
        eng.close()
        for p in pipes:
            p.close()
        pool.shutdown()
    return checked


def _cfg(c):
    from paper_1503_06959_b200 import scenes

    return scenes.CONFIGS[c]


@pytest.mark.parametrize("mode", ["intensity", "binning", "none"])
def test_config1_all_100_frames(mode):
    assert lockstep(_cfg(1), [0], 100, mode) == 100


def test_config2_all_300_frames():
    assert lockstep(_cfg(2), [0], 300) == 300


def test_config3_8_streams_50_frames():
    assert lockstep(_cfg(3), list(range(8)), 50) == 400


def test_config3_stream0_full_200_frames():
    assert lockstep(_cfg(3), [0], 200) == 200


def test_config4_dense_4k_20_frames():
    assert lockstep(_cfg(4), [0], 20) == 20


def test_config5_all_64_streams_10_frames():
    assert lockstep(_cfg(5), list(range(64)), 10) == 640


def test_config5_one_full_length_stream_per_kind():
    """Full 300 frames of a static, a pan and an objects stream (kind = s mod 3)."""
    assert lockstep(_cfg(5), [0, 1, 2], 300) == 900


def test_config5_eight_full_length_streams():
    assert lockstep(_cfg(5), [3, 10, 17, 24, 31, 38, 45, 52], 300) == 2400


def test_bench_cuda_generated_frames():
    """The CUDA scene generator's config-5 frames 0-24 (bench.py --gen cuda):
    six streams (two of each kind) downloaded and checked like the rest."""
    import torch

    from paper_1503_06959_b200 import scenes

    cfg = _cfg(5)
    streams = [0, 1, 2, 33, 34, 35]
    gens = [scenes.SceneStream(cfg, s, torch.device("cuda")) for s in streams]
    assert lockstep(cfg, streams, 25, source=lambda n: torch.stack([g.next_frame() for g in gens]).cpu().numpy()) \
        == 150


@pytest.mark.parametrize("mode", ["intensity", "none"])
def test_small_capacity_grows_and_matches(mode):
    """A tiny kp_capacity (4096, a fraction of a 1080p frame's ~20k features)
    overflows on the first frames; the engine grows the capacity and replays
    the frame from the saved state, so results still equal the oracle's."""
    assert lockstep(_cfg(5), [1, 2], 6, mode, kp_capacity=4096) == 12


def test_capacity_grows_in_place():
    """The capacity after the retries is large enough for a 1080p frame and
    the engine keeps using it (no further overflow on later frames)."""
    import torch

    from paper_1503_06959_b200 import scenes
    from paper_1503_06959_b200.engine import FeatureEngine
    from paper_1503_06959_b200.types import MaskConfig, PipelineConfig

    cfg = _cfg(5)
    fr = scenes.generate(cfg, 3, streams=[2]).numpy()[:, :]          # [1, 3, H, W]
    eng = FeatureEngine(cfg.width, cfg.height, PipelineConfig(mask=MaskConfig(mode="intensity")), n_streams=1,
                        kp_capacity=1024)
    try:
        for n in range(3):
            eng.process(torch.from_numpy(fr[:, n]).cuda(), check=True)
            r = eng.report(0)
            assert r.n_total <= eng.kp_capacity
        assert eng.kp_capacity >= r.n_total > 1024
    finally:
        eng.close()


@pytest.mark.parametrize("mode", ["intensity", "binning", "none"])
def test_delta_results_rebuild_the_lists(mode):
    """vf_pipeline_collect_delta (new records + Eq. 1 keep masks of the previous
    lists) rebuilt on the host with vf_delta_apply gives exactly the oracle's
    merged lists, frame after frame (6 config-5 streams x 8 frames)."""
    from oracle import oracle
    from paper_1503_06959_b200 import scenes
    from paper_1503_06959_b200.engine import FeatureEngine
    from paper_1503_06959_b200.pattern import default_pattern
    from paper_1503_06959_b200.types import MaskConfig, PipelineConfig

    cfg = scenes.CONFIGS[5]
    S, N = 6, 8
    fr = scenes.generate(cfg, N, streams=range(S)).numpy()              # [S, N, H, W]
    eng = FeatureEngine(cfg.width, cfg.height, PipelineConfig(mask=MaskConfig(mode=mode)), n_streams=S)
    eng.set_delta(True)
    out = eng.alloc_delta(S * 65536)
    pipes = [oracle.OraclePipeline(cfg.width, cfg.height, default_pattern(), mode=mode) for _ in range(S)]
    empty = {k: np.zeros(0, np.float64) for k in ("x", "y", "sigma", "theta", "score")}
    empty.update(origin=np.zeros(0, np.uint8), age=np.zeros(0, np.int32), desc=np.zeros((0, 64), np.uint8))
    lists = [empty] * S
    d2h = 0
    try:
        for n in range(N):
            eng.submit(np.ascontiguousarray(fr[:, n]))
            eng.collect_delta(out)
            d2h += int(out["offsets"][S]) * 104 + 4 * int(out["keep_offsets"][S])
            for s in range(S):
                lists[s] = {k: (v.copy() if k != "n" else v) for k, v in FeatureEngine.delta_apply(lists[s], out, s).items()}
                e = pipes[s].process(fr[s, n])
                assert int(out["counts"][s][0]) == e.n_detected and int(out["counts"][s][1]) == e.n_propagated
                _compare(lists[s], e, f"delta {mode} stream {s} frame {n}")
    finally:
        eng.close()
        for p in pipes:
            p.close()
    assert d2h > 0

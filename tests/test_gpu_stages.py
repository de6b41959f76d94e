"""GPU parity of the per-stage drop-ins (through the C-ABI) against the
reference's golden vectors, plus the reference's own unit-test cases
(tests/test_{pyramid,detector,descriptor,masking}.py in the reference)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _gf(a):
    from paper_1503_06959_b200.types import GrayFrame

    return GrayFrame(np.ascontiguousarray(a, np.uint8))


# ---- pyramid (reference tests/test_pyramid.py) ------------------------------
@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_pyramid_golden(tag):
    from paper_1503_06959_b200.pyramid import build_pyramid

    g = golden("pyramid.npz")
    pyr = build_pyramid(_gf(g[f"{tag}_frame"]), int(g[f"{tag}_O"]))
    for i, layer in enumerate(pyr.layers):
        assert np.array_equal(layer.frame.data, g[f"{tag}_layer{i}"]), i
        assert layer.scale == float(g[f"{tag}_scale{i}"])


def test_pyramid_sizes_vga_and_errors():
    from paper_1503_06959_b200.pyramid import build_pyramid

    pyr = build_pyramid(_gf(np.full((480, 640), 137, np.uint8)), 4)
    assert [(l.frame.width, l.frame.height) for l in pyr.layers] == [
        (640, 480), (426, 320), (320, 240), (213, 160), (160, 120), (106, 80), (80, 60), (53, 40)]
    assert all(np.all(l.frame.data == 137) for l in pyr.layers)
    with pytest.raises(ValueError):
        build_pyramid(_gf(np.zeros((4, 64), np.uint8)), 4)
    with pytest.raises(ValueError):
        build_pyramid(_gf(np.zeros((8, 8), np.uint8)), 4)
    with pytest.raises(ValueError):
        build_pyramid(_gf(np.zeros((64, 64), np.uint8)), 0)


# ---- segment test (reference tests/test_detector.py, c04) -------------------
def test_score_maps_golden():
    from paper_1503_06959_b200.detector import score_map

    g = golden("score_maps.npz")
    for k in range(int(g["n"])):
        got = score_map(g[f"data{k}"], int(g[f"t{k}"]), g[f"mask{k}"])
        assert np.array_equal(got, g[f"score{k}"]), k


def test_ast_kats():
    from paper_1503_06959_b200.detector import ast_corner_score

    g = golden("score_maps.npz")
    for d, s in zip(g["kat_data"], g["kat_score"]):
        assert ast_corner_score(_gf(d), 8, 8) == int(s)
    with pytest.raises(ValueError):
        ast_corner_score(_gf(g["kat_data"][0]), 2, 8)


def test_detect_candidates_semantics():
    from paper_1503_06959_b200.detector import detect_candidates
    from paper_1503_06959_b200.types import DetectionMask

    rng = np.random.default_rng(12345)
    layer = _gf(rng.integers(0, 256, (64, 64), dtype=np.uint8))
    assert detect_candidates(layer, 10, DetectionMask(np.zeros((64, 64), np.uint8))) == []
    assert detect_candidates(layer, 10, DetectionMask(np.ones((64, 64), np.uint8))) == detect_candidates(layer, 10)
    low = {(c.x, c.y) for c in detect_candidates(layer, 12)}
    high = {(c.x, c.y) for c in detect_candidates(layer, 35)}
    assert high <= low
    with pytest.raises(ValueError):
        detect_candidates(layer, 0)


def test_c04_score_maps_vs_oracle_many():
    """Acceptance c04 scale: 100 random 64x64 layers x t in {10, 30, 55}, vs the pinned oracle."""
    from oracle import oracle
    from paper_1503_06959_b200.detector import score_map

    rng = np.random.default_rng(7)
    for _ in range(100):
        data = rng.integers(0, 256, (64, 64), dtype=np.uint8)
        for t in (10, 30, 55):
            assert np.array_equal(score_map(data, t).astype(np.int32), oracle.score_map(data, t))


# ---- NMS + refinement --------------------------------------------------------
@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_nms_golden(tag):
    from paper_1503_06959_b200.detector import nms_from_maps

    g = golden("nms.npz")
    O = int(g[f"{tag}_O"])
    f = g[f"{tag}_frame"]
    kps = nms_from_maps([g[f"{tag}_map{i}"] for i in range(2 * O)], f.shape[1], f.shape[0], O)
    got = np.array([[k.x, k.y, k.score] for k in kps]).reshape(-1, 3)
    exp = np.stack([g[f"{tag}_x"], g[f"{tag}_y"], g[f"{tag}_score"]], 1)
    assert got.shape == exp.shape
    assert np.array_equal(got, exp)
    assert np.allclose([k.sigma for k in kps], g[f"{tag}_sigma"], rtol=0, atol=1e-12)


def test_nms_reference_cases():
    from paper_1503_06959_b200.detector import nms_and_refine
    from paper_1503_06959_b200.pyramid import build_pyramid
    from paper_1503_06959_b200.types import Candidate

    g = golden("nms.npz")
    pyr = build_pyramid(_gf(np.zeros((64, 64), np.uint8)), 2)
    for ci in range(int(g["n_cases"])):
        cands = {}
        for li, x, y, s in g[f"case{ci}_cands"]:
            lid = (pyr.layers[li].kind, pyr.layers[li].level)
            cands.setdefault(lid, []).append(Candidate(int(x), int(y), lid, int(s)))
        kps = nms_and_refine(cands, pyr)
        got = np.array([[k.x, k.y, k.sigma, k.score] for k in kps]).reshape(-1, 4)
        exp = g[f"case{ci}_kps"]
        assert got.shape == exp.shape and np.allclose(got, exp, atol=1e-12), ci


# ---- descriptor (reference tests/test_descriptor.py) -------------------------
def test_describe_golden():
    from paper_1503_06959_b200 import descriptor
    from paper_1503_06959_b200.types import Keypoint

    g = golden("describe.npz")
    frame = _gf(g["data"])
    kps = [Keypoint(float(a), float(b), float(c)) for a, b, c in zip(g["kx"], g["ky"], g["sigma"])]
    th = descriptor.orientations_batch(frame, kps)
    assert np.allclose(th, g["orient"], rtol=0, atol=1e-9)
    assert np.array_equal(descriptor.describe_batch_packed(frame, kps, g["theta_in"]), g["desc_theta_in"])
    assert np.array_equal(descriptor.describe_batch_packed(frame, kps, g["orient"]), g["desc_orient"])
    for f, o, d in zip(g["kat_frames"], g["kat_orient"], g["kat_desc"]):
        kp = Keypoint(32.0, 32.0, 1.0)
        assert abs(descriptor.estimate_orientation(_gf(f), kp) - o) <= 1e-12
        assert np.array_equal(np.packbits(descriptor.describe(_gf(f), kp, 0.0)), d)


def test_describe_footprint_errors():
    from paper_1503_06959_b200 import descriptor
    from paper_1503_06959_b200.types import Keypoint

    layer = _gf(np.clip(np.arange(64)[None, :].repeat(64, 0) * 3, 0, 255))
    with pytest.raises(descriptor.FootprintError):
        descriptor.describe(layer, Keypoint(62.0, 32.0, 2.0), 0.0)
    with pytest.raises(descriptor.FootprintError):
        descriptor.estimate_orientation(layer, Keypoint(1.0, 32.0, 1.0))


# ---- masks (reference tests/test_masking.py) ---------------------------------
def test_masks_golden():
    from paper_1503_06959_b200 import masking
    from paper_1503_06959_b200.types import Feature, Keypoint, SubsampledMask

    g = golden("masks.npz")
    for t_i in (-1.0, 0.0, 19.5, 20.0, 30.0):
        got = masking.intensity_diff_mask(_gf(g["idm_a"]), _gf(g["idm_b"]), t_i).bits
        assert np.array_equal(got, g[f"idm_{t_i}"])
    feats = [Feature(Keypoint(float(x), float(y), 1.0), np.zeros(512, np.uint8)) for x, y in zip(g["bin_x"], g["bin_y"])]
    assert np.array_equal(masking.binning_histogram(feats, (640, 480), (16, 16)), g["bin_hist_16"])
    assert np.array_equal(masking.binning_histogram(feats, (640, 480), (3, 5)), g["bin_hist_3x5"])
    up = masking.upsample_mask(SubsampledMask(g["up_bits"], cell_w=9, cell_h=9), (70, 50)).bits
    assert np.array_equal(up, g["up_full"])
    with pytest.raises(ValueError):
        masking.upsample_mask(SubsampledMask(np.ones((2, 2), np.uint8), cell_w=4, cell_h=4), (64, 48))


def test_merge_features_rule():
    from paper_1503_06959_b200 import masking
    from paper_1503_06959_b200.types import DETECTED, PROPAGATED, DetectionMask, Feature, Keypoint

    rng = np.random.default_rng(3)
    bits = rng.integers(0, 2, (48, 64)).astype(np.uint8)
    mask = DetectionMask(bits)
    det = [Feature(Keypoint(float(rng.uniform(0, 63)), float(rng.uniform(0, 47)), 1.0), np.zeros(512, np.uint8))
           for _ in range(25)]
    prev = [Feature(Keypoint(float(rng.uniform(0, 63)), float(rng.uniform(0, 47)), 1.0), np.zeros(512, np.uint8),
                    DETECTED, 2) for _ in range(40)]
    out = masking.merge_features(det, prev, mask)
    exp = [d for d in det if bits[min(int(np.floor(d.kp.y + .5)), 47), min(int(np.floor(d.kp.x + .5)), 63)] == 1]
    exp += [p for p in prev if bits[min(int(np.floor(p.kp.y + .5)), 47), min(int(np.floor(p.kp.x + .5)), 63)] == 0]
    assert [(f.kp.x, f.kp.y) for f in out] == [(f.kp.x, f.kp.y) for f in exp]
    n_det = sum(1 for f in out if f.origin == DETECTED)
    assert all(f.origin == PROPAGATED and f.age == 3 for f in out[n_det:])


# ---- drop-in run_pipeline (reference tests/test_pipeline.py, c01, c02) --------
def test_run_pipeline_objects_match_golden():
    from paper_1503_06959_b200.pipeline import run_pipeline
    from paper_1503_06959_b200.types import GrayFrame, MaskConfig, PipelineConfig

    g = golden("pipeline_small_intensity.npz")
    frames = [GrayFrame(f, i) for i, f in enumerate(g["frames"])]
    feats, reports = run_pipeline(frames, PipelineConfig(threshold=25, mask=MaskConfig(mode="intensity", t_i=15)))
    offs = g["offsets"]
    for n, fs in enumerate(feats):
        a, b = offs[n], offs[n + 1]
        assert len(fs) == b - a
        assert [f.kp.x for f in fs] == g["x"][a:b].tolist()
        assert [f.kp.y for f in fs] == g["y"][a:b].tolist()
        assert np.array_equal(np.array([np.packbits(f.desc) for f in fs]).reshape(-1, 64), g["desc"][a:b])
        assert [f.origin == "propagated" for f in fs] == g["origin"][a:b].astype(bool).tolist()
        r = reports[n]
        assert (r.n_detected, r.n_propagated, r.n_total, r.n_dropped) == (
            g["r_n_detected"][n], g["r_n_propagated"][n], g["offsets"][n + 1] - g["offsets"][n], g["r_n_dropped"][n])
        assert r.coverage == g["r_coverage"][n]
        assert min(r.t_pyramid_ms, r.t_mask_ms, r.t_detect_ms, r.t_describe_ms, r.t_total_ms) >= 0.0


def test_c01_gating_identity():
    """All-ones mask (t_i = -1) is bit-identical to no mask (acceptance c01)."""
    from paper_1503_06959_b200.pipeline import run_pipeline_arrays
    from paper_1503_06959_b200.types import GrayFrame, MaskConfig, PipelineConfig

    rng = np.random.default_rng(42)
    frames = [GrayFrame(rng.integers(0, 256, (480, 640), dtype=np.uint8), i) for i in range(6)]
    plain, _ = run_pipeline_arrays(frames, PipelineConfig(mask=MaskConfig(mode="none")))
    forced, reps = run_pipeline_arrays(frames, PipelineConfig(mask=MaskConfig(mode="intensity", t_i=-1.0)))
    assert all(r.coverage == 1.0 for r in reps)
    for a, b in zip(plain, forced):
        for k in ("x", "y", "sigma", "theta", "score", "origin", "desc"):
            assert np.array_equal(a[k], b[k]), k


def test_c02_static_fixpoint():
    from paper_1503_06959_b200.pipeline import run_pipeline_arrays
    from paper_1503_06959_b200.types import GrayFrame, MaskConfig, PipelineConfig

    g = golden("pipeline_static_intensity.npz")
    frames = [GrayFrame(f, i) for i, f in enumerate(g["frames"])]
    outs, reps = run_pipeline_arrays(frames, PipelineConfig(threshold=25, mask=MaskConfig(mode="intensity", t_i=5)))
    assert all(r.coverage == 0.0 for r in reps[1:])
    for n in range(1, len(outs)):
        for k in ("x", "y", "sigma", "theta", "score", "desc"):
            assert np.array_equal(outs[n][k], outs[0][k])
        assert set(outs[n]["age"].tolist()) == {n}


def test_run_streams_equals_per_stream():
    """Batched streams (config 3/5 path) equal independent single-stream runs."""
    from oracle import oracle
    from paper_1503_06959_b200 import scenes
    from paper_1503_06959_b200.pattern import default_pattern
    from paper_1503_06959_b200.pipeline import run_streams
    from paper_1503_06959_b200.types import MaskConfig, PipelineConfig

    cfg = scenes.SceneConfig(640, 480, 6, 3, "mixed", (3, 6), (0.0, 4.0), (0.5, 2.0), noise_sigma=2.0,
                             block_contrast=120.0, seed=77)
    frames = scenes.generate(cfg).numpy()
    for mode in ("intensity", "binning"):
        feats, reps = run_streams(frames, PipelineConfig(mask=MaskConfig(mode=mode)))
        for s in range(frames.shape[0]):
            ref = oracle.run_sequence(list(frames[s]), default_pattern(), mode=mode)
            for n, (o, e) in enumerate(zip(feats[s], ref)):
                assert o["n"] == e.n_total, (mode, s, n)
                assert np.array_equal(o["x"], e.x) and np.array_equal(o["desc"], e.desc), (mode, s, n)
                assert reps[s][n].coverage == e.coverage


def test_packed_and_pipelined_outputs_match_per_stream():
    """vf_fetch_features (packed, all streams) and the pipelined submit/collect
    e2e API return exactly the per-stream feature lists."""
    import torch

    from paper_1503_06959_b200 import scenes
    from paper_1503_06959_b200.engine import FeatureEngine
    from paper_1503_06959_b200.types import MaskConfig, PipelineConfig

    cfg = scenes.SceneConfig(640, 480, 5, 3, "mixed", (3, 6), (0.0, 4.0), (0.5, 2.0), noise_sigma=2.0,
                             block_contrast=120.0, seed=91)
    frames = scenes.generate(cfg).numpy()  # [S, N, H, W]
    S, N = frames.shape[:2]
    pcfg = PipelineConfig(mask=MaskConfig(mode="intensity"))
    ref = FeatureEngine(640, 480, pcfg, n_streams=S)
    pipe = FeatureEngine(640, 480, pcfg, n_streams=S)
    out_fetch = ref.alloc_host(S * 20000, pinned=False)
    out_pipe = pipe.alloc_host(S * 20000)
    dev = torch.from_numpy(np.ascontiguousarray(frames.transpose(1, 0, 2, 3))).cuda()
    host = [np.ascontiguousarray(frames[:, n]) for n in range(N)]
    pipe.submit(host[0])
    for n in range(N):
        ref.process(dev[n])
        per = [ref.features_host(s) for s in range(S)]
        ref.fetch_all(out_fetch)
        torch.cuda.synchronize()
        if n + 1 < N:
            pipe.submit(host[n + 1])
        pipe.collect(out_pipe)
        for out in (out_fetch, out_pipe):
            offs = out["offsets"]
            for s in range(S):
                a, b = int(offs[s]), int(offs[s + 1])
                assert b - a == per[s]["n"], (n, s)
                for k in ("x", "y", "sigma", "theta", "score", "origin", "age", "desc"):
                    assert np.array_equal(out[k][a:b], per[s][k]), (n, s, k)
    ref.close()
    pipe.close()


@pytest.mark.parametrize("d2h_kernel", ["1", "0"])
def test_pipelined_api_three_steps_in_flight(d2h_kernel):
    """vf_pipeline_submit keeps up to three steps in flight (a fourth submit is refused) and
    collect / collect_delta return them oldest first, identical to step-by-step processing --
    with the results delivered by one k_copy_out launch (small results into pinned arrays) or by
    the per-field copies (VF_D2H_KERNEL=0), into pinned and into pageable arrays."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    child = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_1503_06959_b200 import scenes
from paper_1503_06959_b200.engine import FeatureEngine
from paper_1503_06959_b200.types import MaskConfig, PipelineConfig
cfg = scenes.SceneConfig(320, 240, 9, 2, "mixed", (3, 6), (0.0, 4.0), (0.5, 2.0), noise_sigma=2.0,
                         block_contrast=120.0, seed=17)
frames = scenes.generate(cfg).numpy()
S, N = frames.shape[:2]
pcfg = PipelineConfig(mask=MaskConfig(mode="intensity"))
ref = FeatureEngine(320, 240, pcfg, n_streams=S)
dev = torch.from_numpy(np.ascontiguousarray(frames.transpose(1, 0, 2, 3))).cuda()
want = []
for n in range(N):
    ref.process(dev[n])
    want.append([ref.features_host(s) for s in range(S)])
ref.close()
host = [np.ascontiguousarray(frames[:, n]) for n in range(N)]
keys = ("x", "y", "sigma", "theta", "score", "origin", "age", "desc")
for pinned in (True, False):
    pipe = FeatureEngine(320, 240, pcfg, n_streams=S)
    out = pipe.alloc_host(S * 20000, pinned=pinned)
    pipe.submit(host[0]); pipe.submit(host[1]); pipe.submit(host[2])
    try:
        pipe.submit(host[3])
        raise SystemExit("a fourth step in flight was accepted")
    except (RuntimeError, ValueError):
        pass
    for n in range(N):
        pipe.collect(out)
        if n + 3 < N:
            pipe.submit(host[n + 3])
        offs = out["offsets"]
        for s in range(S):
            a, b = int(offs[s]), int(offs[s + 1])
            assert b - a == want[n][s]["n"], (pinned, n, s)
            for k in keys:
                assert np.array_equal(out[k][a:b], want[n][s][k]), (pinned, n, s, k)
    pipe.close()
    # delta delivery, three in flight: rebuild every merged list on the host
    pipe = FeatureEngine(320, 240, pcfg, n_streams=S)
    out = pipe.alloc_delta(S * 20000, pinned=pinned)
    pipe.set_delta(True)
    empty = {k: np.zeros(0, np.float64) for k in ("x", "y", "sigma", "theta", "score")}
    empty.update(origin=np.zeros(0, np.uint8), age=np.zeros(0, np.int32), desc=np.zeros((0, 64), np.uint8))
    prev = [empty] * S
    for n in range(min(3, N)):
        pipe.submit(host[n])
    for n in range(N):
        pipe.collect_delta(out)
        if n + 3 < N:
            pipe.submit(host[n + 3])
        for s in range(S):
            cur = FeatureEngine.delta_apply(prev[s], out, s)
            assert cur["n"] == want[n][s]["n"], (pinned, n, s)
            for k in keys:
                assert np.array_equal(cur[k], want[n][s][k]), (pinned, n, s, k)
            prev[s] = {k: (v.copy() if k != "n" else v) for k, v in cur.items()}
    pipe.close()
print("ok")
"""
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, VF_D2H_KERNEL=d2h_kernel)   # read once per process
    r = subprocess.run([sys.executable, "-c", child, str(root)], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), (r.stdout[-500:], r.stderr[-2000:])

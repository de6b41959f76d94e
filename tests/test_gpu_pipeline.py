"""GPU parity: the sm_100a pipeline (through the C-ABI) vs the reference's
golden vectors and vs the pinned CPU oracle.

Tolerances (north_star): bit-exact for masks/coverage, counts, order, origin,
age, scores and packed descriptors; fp64 x, y, sigma, theta, score within
abs 1e-4 (expected identical up to ulp-level libm differences)."""

import numpy as np
import pytest

from conftest import GOLDEN, golden

pytestmark = pytest.mark.gpu

PIPELINES = sorted(p.stem[len("pipeline_"):] for p in GOLDEN.glob("pipeline_*.npz") if not p.stem.endswith("_temporal"))
TOL = 1e-4


def run_engine(frames, **cfgkw):
    import torch
    from paper_1503_06959_b200.engine import FeatureEngine
    from paper_1503_06959_b200.types import MaskConfig, PipelineConfig

    mc = MaskConfig(**{k: v for k, v in cfgkw.items() if k in ("mode", "t_i", "t_h", "grid", "octave_for_mask", "per_layer")})
    cfg = PipelineConfig(threshold=cfgkw.get("threshold", 55), n_octaves=cfgkw.get("n_octaves", 4), mask=mc)
    H, W = frames[0].shape
    eng = FeatureEngine(W, H, cfg, n_streams=1)
    dev = torch.from_numpy(np.ascontiguousarray(np.stack(frames))).cuda()
    outs = []
    for n in range(len(frames)):
        eng.process(dev[n:n + 1])
        r = eng.report(0)
        f = eng.features_host(0)
        f["report"] = r
        outs.append(f)
    eng.close()
    return outs


def compare(outs, ref, label):
    """ref: list of dicts with x,y,sigma,theta,score,origin,age,desc + counts."""
    for n, (o, e) in enumerate(zip(outs, ref)):
        r = o["report"]
        where = f"{label} frame {n}"
        assert r.n_total == len(e["x"]), f"{where}: n_total {r.n_total} vs {len(e['x'])}"
        assert r.n_detected == e["n_detected"], where
        assert r.n_propagated == e["n_propagated"], where
        assert r.n_dropped == e["n_dropped"], where
        assert r.coverage == e["coverage"], where
        assert np.array_equal(o["origin"], e["origin"]), where
        assert np.array_equal(o["age"], e["age"]), where
        for k in ("x", "y", "sigma", "theta", "score"):
            d = np.abs(o[k] - e[k])
            assert d.size == 0 or d.max() <= TOL, f"{where}: {k} max diff {d.max()}"
        assert np.array_equal(o["x"], e["x"]), f"{where}: x not bit-identical"
        assert np.array_equal(o["y"], e["y"]), f"{where}: y not bit-identical"
        assert np.array_equal(o["score"], e["score"]), f"{where}: score not bit-identical"
        bad = np.nonzero((o["desc"] != e["desc"]).any(1))[0]
        assert bad.size == 0, f"{where}: {bad.size} descriptors differ (first {bad[:5]})"


def golden_frames(g):
    offs = g["offsets"]
    out = []
    for n in range(len(offs) - 1):
        a, b = offs[n], offs[n + 1]
        out.append({k: g[k][a:b] for k in ("x", "y", "sigma", "theta", "score", "origin", "age", "desc")} | {
            "n_detected": int(g["r_n_detected"][n]), "n_propagated": int(g["r_n_propagated"][n]),
            "n_dropped": int(g["r_n_dropped"][n]), "coverage": float(g["r_coverage"][n])})
    return out


@pytest.mark.parametrize("name", PIPELINES)
def test_pipeline_vs_reference_goldens(name):
    g = golden(f"pipeline_{name}.npz")
    ofm = int(g["octave_for_mask"])
    outs = run_engine(list(g["frames"]), threshold=int(g["threshold"]), n_octaves=int(g["n_octaves"]),
                      mode=str(g["mode"]), t_i=float(g["t_i"]), t_h=int(g["t_h"]),
                      grid=tuple(int(v) for v in g["grid"]), octave_for_mask=None if ofm < 0 else ofm,
                      per_layer=bool(g["per_layer"]))
    compare(outs, golden_frames(g), name)


def oracle_frames(frames, **cfg):
    from oracle import oracle
    from paper_1503_06959_b200.pattern import default_pattern

    res = oracle.run_sequence(list(frames), default_pattern(), **cfg)
    return [dict(x=r.x, y=r.y, sigma=r.sigma, theta=r.theta, score=r.score, origin=r.origin, age=r.age,
                 desc=r.desc, n_detected=r.n_detected, n_propagated=r.n_propagated, n_dropped=r.n_dropped,
                 coverage=r.coverage) for r in res]


@pytest.mark.parametrize("mode", ["intensity", "binning", "none"])
def test_config1_vs_oracle(mode):
    """BASELINE config 1 (640x480, seeded objects scene), 12-frame prefix."""
    from paper_1503_06959_b200 import scenes

    frames = scenes.generate(scenes.CONFIGS[1], 12, streams=[0])[0].numpy()
    outs = run_engine(list(frames), mode=mode)
    compare(outs, oracle_frames(frames, mode=mode), f"config1/{mode}")


def test_config2_vs_oracle():
    """BASELINE config 2 (1280x720 panning scene, intensity), 8-frame prefix."""
    from paper_1503_06959_b200 import scenes

    frames = scenes.generate(scenes.CONFIGS[2], 8, streams=[0])[0].numpy()
    outs = run_engine(list(frames), mode="intensity")
    compare(outs, oracle_frames(frames, mode="intensity"), "config2")

"""GPU parity of the temporal block-matching baseline
through the C ABI (vf_block_match, FeatureEngine mode 3) against the
reference's own outputs (tests/golden/temporal.npz, pipeline_*_temporal.npz)
and the pinned CPU oracle: exact positions, SADs, counts, order, descriptors."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _gop(gp):
    from paper_1503_06959_b200.types import GopConfig

    return GopConfig(delta=int(gp[0]), patch=int(gp[1]), t_bm=float(gp[2]), t_et=float(gp[3]),
                     coarse_window=float(gp[4]), coarse_step=float(gp[5]), fine_window=float(gp[6]),
                     fine_step=float(gp[7]))


def _bm(prev, cur, x, y, cfg):
    import torch

    from paper_1503_06959_b200.temporal import block_match_device

    f, nx, ny, sd = block_match_device(torch.from_numpy(prev).cuda(), torch.from_numpy(cur).cuda(),
                                       torch.from_numpy(np.asarray(x, np.float64)).cuda(),
                                       torch.from_numpy(np.asarray(y, np.float64)).cuda(), cfg)
    return f.cpu().numpy(), nx.cpu().numpy(), ny.cpu().numpy(), sd.cpu().numpy()


def test_block_match_golden():
    """vf_block_match == the reference's spiral_search on every golden case
    (coarse early exits, quarter-pixel refinements, rejections, border blocks)."""
    g = golden("temporal.npz")
    for ci in range(int(g["n_bm"])):
        for gi in range(3):
            k = f"bm{ci}_{gi}"
            f, nx, ny, sd = _bm(g[f"bm{ci}_prev"], g[f"bm{ci}_cur"], g[f"bm{ci}_x"], g[f"bm{ci}_y"],
                                _gop(g[f"{k}_gop"]))
            exp = g[f"{k}_found"]
            assert np.array_equal(f, exp), k
            assert np.array_equal(nx[exp], g[f"{k}_nx"][exp]) and np.array_equal(ny[exp], g[f"{k}_ny"][exp]), k
            assert np.array_equal(sd[exp], g[f"{k}_sad"][exp]), k


@pytest.mark.parametrize("kw", [dict(fine_step=0.3, fine_window=1.5),             # non-dyadic: fp64 path
                                dict(coarse_step=1.5, coarse_window=6.0),         # truncated coarse offsets
                                dict(patch=6, t_bm=400.0, t_et=100.0),            # patch % 4 != 0
                                dict(t_et=5000.0),                                # early exits everywhere
                                dict(t_et=1.0, t_bm=1e9, coarse_window=4.0)])     # full fine search
def test_block_match_configs_vs_oracle(kw):
    from oracle import oracle
    from paper_1503_06959_b200.types import GopConfig

    g = golden("temporal.npz")
    cfg = GopConfig(**kw)
    okw = dict(patch=cfg.patch, t_bm=cfg.t_bm, t_et=cfg.t_et, coarse_window=cfg.coarse_window,
               coarse_step=cfg.coarse_step, fine_window=cfg.fine_window, fine_step=cfg.fine_step)
    for ci in range(int(g["n_bm"])):
        prev, cur, x, y = g[f"bm{ci}_prev"], g[f"bm{ci}_cur"], g[f"bm{ci}_x"], g[f"bm{ci}_y"]
        f, nx, ny, sd = _bm(prev, cur, x, y, cfg)
        ef, enx, eny, esd = oracle.block_match(prev, cur, x, y, **okw)
        assert np.array_equal(f, ef), (kw, ci)
        assert np.array_equal(nx[ef], enx[ef]) and np.array_equal(ny[ef], eny[ef]), (kw, ci)
        assert np.array_equal(sd[ef], esd[ef]), (kw, ci)


def _check_frames(outs, reps, exp_frames, where):
    for n, (o, r, e) in enumerate(zip(outs, reps, exp_frames)):
        assert (r.n_detected, r.n_propagated, r.n_total, r.n_dropped) == \
            (e.n_detected, e.n_propagated, e.n_total, e.n_dropped), (where, n)
        assert r.coverage == e.coverage, (where, n)
        for k in ("x", "y", "score", "origin", "age", "desc"):
            assert np.array_equal(o[k], getattr(e, k)), (where, n, k)
        assert np.abs(o["sigma"] - e.sigma).max(initial=0) <= 1e-12, (where, n)
        assert np.abs(o["theta"] - e.theta).max(initial=0) <= 1e-4, (where, n)


@pytest.mark.parametrize("name", ["small_temporal", "scene_temporal"])
def test_temporal_pipeline_golden(name):
    """run_pipeline(mode='temporal') == the reference (pipeline.py:281-345)."""
    from types import SimpleNamespace

    from paper_1503_06959_b200.pipeline import run_pipeline_arrays
    from paper_1503_06959_b200.types import GrayFrame, MaskConfig, PipelineConfig

    g = golden(f"pipeline_{name}.npz")
    cfg = PipelineConfig(threshold=int(g["threshold"]), n_octaves=int(g["n_octaves"]),
                         mask=MaskConfig(mode="temporal"), gop=_gop(g["gop"]))
    outs, reps = run_pipeline_arrays([GrayFrame(f, i) for i, f in enumerate(g["frames"])], cfg)
    off = g["offsets"]
    exp = [SimpleNamespace(**{k: g[k][off[n]:off[n + 1]] for k in ("x", "y", "sigma", "theta", "score", "origin",
                                                                   "age", "desc")},
                           n_detected=int(g["r_n_detected"][n]), n_propagated=int(g["r_n_propagated"][n]),
                           n_total=int(g["r_n_total"][n]), n_dropped=int(g["r_n_dropped"][n]),
                           coverage=float(g["r_coverage"][n])) for n in range(len(g["frames"]))]
    _check_frames(outs, reps, exp, name)


def test_temporal_streams_1080p_vs_oracle():
    """Three 1080p config-5 streams (static / pan / objects), GOP length 3,
    batched in one engine: every frame equals the oracle's run of the stream."""
    import torch

    from oracle import oracle
    from paper_1503_06959_b200 import scenes
    from paper_1503_06959_b200.engine import FeatureEngine
    from paper_1503_06959_b200.pattern import default_pattern
    from paper_1503_06959_b200.types import GopConfig, MaskConfig, PipelineConfig

    frames = scenes.generate(scenes.CONFIGS[5], 5, streams=range(3)).numpy()
    cfg = PipelineConfig(mask=MaskConfig(mode="temporal"), gop=GopConfig(delta=3))
    eng = FeatureEngine(1920, 1080, cfg, n_streams=3)
    dev = torch.from_numpy(np.ascontiguousarray(frames.transpose(1, 0, 2, 3))).cuda()
    outs = [[] for _ in range(3)]
    reps = [[] for _ in range(3)]
    for n in range(5):
        eng.process(dev[n])
        for s in range(3):
            outs[s].append(eng.features_host(s))
            reps[s].append(eng.report(s))
    eng.close()
    for s in range(3):
        ref = oracle.run_sequence(list(frames[s]), default_pattern(), mode="temporal", gop=dict(delta=3))
        _check_frames(outs[s], reps[s], ref, f"stream {s}")
        assert any(r.n_propagated > 0 for r in reps[s][1:3])


def test_gop_errors_through_c_abi():
    """GopConfig errors from the C side carry the reference's messages (temporal.py:33-43)."""
    import torch

    from paper_1503_06959_b200 import _native
    from paper_1503_06959_b200.temporal import _gop_struct

    L = _native.lib()
    z = torch.zeros((32, 32), dtype=torch.uint8, device="cuda")
    for field, val, msg in [("gop_delta", 0, "GOP length"), ("gop_patch", 7, "patch side")]:
        c = _gop_struct(__import__("paper_1503_06959_b200.types", fromlist=["GopConfig"]).GopConfig())
        setattr(c, field, val)
        rc = L.vf_block_match(z.data_ptr(), z.data_ptr(), 32, 32, 32, 0, 0, 0, __import__("ctypes").byref(c),
                              0, 0, 0, 0, 0)
        with pytest.raises(ValueError, match=msg):
            _native.check(rc)

"""The CPU oracle (oracle/vf_oracle.c) against golden vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only.

This pins the oracle: everything the GPU parity tests compare against is
first shown here to reproduce the reference bit-for-bit (sigma to 1 ulp,
see test_pipeline_goldens)."""

import numpy as np
import pytest

from conftest import GOLDEN, golden
from oracle import oracle
from paper_1503_06959_b200.pattern import build_default_pattern

PIPELINES = sorted(p.stem[len("pipeline_"):] for p in GOLDEN.glob("pipeline_*.npz") if not p.stem.endswith("_temporal"))


def test_pattern_matches_reference_builder():
    g = golden("pattern_v1.npz")
    p = build_default_pattern()
    for k in ("points", "radii", "short_pairs", "long_pairs"):
        assert np.array_equal(getattr(p, k), g[k]), k
    assert p.long_pairs.shape[0] == 393


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_pyramid(tag):
    g = golden("pyramid.npz")
    O = int(g[f"{tag}_O"])
    layers = oracle.build_pyramid(g[f"{tag}_frame"], O)
    _, _, sc = oracle.layer_dims(g[f"{tag}_frame"].shape[1], g[f"{tag}_frame"].shape[0], O)
    for i, l in enumerate(layers):
        assert np.array_equal(l, g[f"{tag}_layer{i}"]), i
        assert sc[i] == float(g[f"{tag}_scale{i}"])


def test_score_maps():
    g = golden("score_maps.npz")
    for k in range(int(g["n"])):
        got = oracle.score_map(g[f"data{k}"], int(g[f"t{k}"]), g[f"mask{k}"])
        assert np.array_equal(got.astype(np.uint8), g[f"score{k}"]), k
    for d, s in zip(g["kat_data"], g["kat_score"]):
        m = oracle.score_map(d, 1)
        assert max(int(m[8, 8]) , 0) == int(s) or (s == 0 and m[8, 8] == 0)


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_nms(tag):
    g = golden("nms.npz")
    O = int(g[f"{tag}_O"])
    f = g[f"{tag}_frame"]
    _, _, sc = oracle.layer_dims(f.shape[1], f.shape[0], O)
    maps = [g[f"{tag}_map{i}"].astype(np.int32) for i in range(2 * O)]
    k = oracle.nms(maps, sc, f.shape[1], f.shape[0])
    assert np.array_equal(k["x"], g[f"{tag}_x"])
    assert np.array_equal(k["y"], g[f"{tag}_y"])
    assert np.array_equal(k["score"], g[f"{tag}_score"])
    assert np.allclose(k["sigma"], g[f"{tag}_sigma"], rtol=0, atol=1e-12)


def test_nms_reference_cases():
    g = golden("nms.npz")
    _, _, sc = oracle.layer_dims(64, 64, 2)
    ws, hs, _ = oracle.layer_dims(64, 64, 2)
    for ci in range(int(g["n_cases"])):
        maps = [np.zeros((hs[i], ws[i]), np.int32) for i in range(4)]
        for li, x, y, s in g[f"case{ci}_cands"]:
            maps[li][y, x] = s
        k = oracle.nms(maps, sc, 64, 64)
        exp = g[f"case{ci}_kps"]
        got = np.stack([k["x"], k["y"], k["sigma"], k["score"]], 1) if len(k["x"]) else np.zeros((0, 4))
        assert got.shape == exp.shape and np.allclose(got, exp, atol=1e-12), ci


def test_describe():
    g = golden("describe.npz")
    p = build_default_pattern()
    th = oracle.orientations(g["data"], g["kx"], g["ky"], g["sigma"], p)
    assert np.allclose(th, g["orient"], rtol=0, atol=1e-9)
    assert np.array_equal(oracle.describe(g["data"], g["kx"], g["ky"], g["sigma"], g["theta_in"], p),
                          g["desc_theta_in"])
    assert np.array_equal(oracle.describe(g["data"], g["kx"], g["ky"], g["sigma"], g["orient"], p),
                          g["desc_orient"])
    for f, o, d in zip(g["kat_frames"], g["kat_orient"], g["kat_desc"]):
        assert abs(oracle.orientations(f, [32.0], [32.0], [1.0], p)[0] - o) <= 1e-12
        assert np.array_equal(oracle.describe(f, [32.0], [32.0], [1.0], [0.0], p)[0], d)


def test_masks():
    g = golden("masks.npz")
    for t_i in (-1.0, 0.0, 19.5, 20.0, 30.0):
        assert np.array_equal(oracle.intensity_mask(g["idm_a"], g["idm_b"], t_i), g[f"idm_{t_i}"])
    assert np.array_equal(oracle.binning_hist(g["bin_x"], g["bin_y"], 640, 480, 16, 16), g["bin_hist_16"])
    assert np.array_equal(oracle.binning_hist(g["bin_x"], g["bin_y"], 640, 480, 3, 5), g["bin_hist_3x5"])
    assert np.array_equal(oracle.upsample(g["up_bits"], 9, 9, 70, 50), g["up_full"])


def compare_frames(outs, g, sigma_atol=1e-12):
    offs = g["offsets"]
    for n, o in enumerate(outs):
        a, b = offs[n], offs[n + 1]
        assert o.n_total == b - a, n
        assert o.n_detected == g["r_n_detected"][n]
        assert o.n_propagated == g["r_n_propagated"][n]
        assert o.n_dropped == g["r_n_dropped"][n]
        assert o.coverage == g["r_coverage"][n]
        assert np.array_equal(o.x, g["x"][a:b]), n
        assert np.array_equal(o.y, g["y"][a:b]), n
        assert np.array_equal(o.score, g["score"][a:b]), n
        assert np.array_equal(o.origin, g["origin"][a:b]), n
        assert np.array_equal(o.age, g["age"][a:b]), n
        assert np.array_equal(o.desc, g["desc"][a:b]), n
        # numpy's SIMD power (AVX-512 SVML) and glibc pow differ by <= 1 ulp
        assert np.allclose(o.sigma, g["sigma"][a:b], rtol=0, atol=sigma_atol), n
        assert np.allclose(o.theta, g["theta"][a:b], rtol=0, atol=1e-9), n


@pytest.mark.parametrize("name", PIPELINES)
def test_pipeline_goldens(name):
    g = golden(f"pipeline_{name}.npz")
    p = build_default_pattern()
    ofm = int(g["octave_for_mask"])
    outs = oracle.run_sequence(
        list(g["frames"]), p, threshold=int(g["threshold"]), n_octaves=int(g["n_octaves"]),
        mode=str(g["mode"]), t_i=float(g["t_i"]), t_h=int(g["t_h"]), grid=tuple(int(v) for v in g["grid"]),
        octave_for_mask=None if ofm < 0 else ofm, per_layer=bool(g["per_layer"]))
    compare_frames(outs, g)


def test_oracle_hamming_matrix_golden():
    """vfo_hamming_matrix == the reference's hamming_matrix (matching.py:73-77)."""
    from oracle import oracle

    g = golden("matching.npz")
    for tag in "abcd":
        assert np.array_equal(oracle.hamming_matrix(g[f"{tag}_q"], g[f"{tag}_r"]), g[f"{tag}_d"]), tag


def test_oracle_radius_match_golden():
    """Oracle radius match == the reference's radius_match (matching.py:80-94),
    planted distances 0..200 around t_m in {0, 50, 102, 260} and 56-bit rows."""
    from oracle import oracle

    g = golden("matching.npz")
    q = np.packbits(g["plant_q_bits"], axis=1)
    r = np.packbits(g["plant_r_bits"], axis=1)
    for t_m in (0, 50, 102, 260):
        qi, ri, d = oracle.radius_match(q, r, t_m)
        assert np.array_equal(np.stack([qi, ri, d], 1).reshape(-1, 3), g[f"plant_{t_m}"]), t_m
    qi, ri, d = oracle.radius_match(np.packbits(g["w56_q_bits"], axis=1), np.packbits(g["w56_r_bits"], axis=1), 24)
    assert np.array_equal(np.stack([qi, ri, d], 1).reshape(-1, 3), g["w56_24"])
    assert int(g["default_radius"]) == 102


def _gop_kw(gp):
    return dict(delta=int(gp[0]), patch=int(gp[1]), t_bm=float(gp[2]), t_et=float(gp[3]),
                coarse_window=float(gp[4]), coarse_step=float(gp[5]), fine_window=float(gp[6]),
                fine_step=float(gp[7]))


def test_spiral_offsets_golden():
    """temporal.py:46-61 order: the oracle's and the product's host constants."""
    from oracle import oracle
    from paper_1503_06959_b200.temporal import spiral_offsets

    g = golden("temporal.npz")
    for key, (r, st) in {"coarse_12_2": (12.0, 2.0), "fine_175_025": (1.75, 0.25), "odd_5_1": (5.0, 1.0)}.items():
        assert np.array_equal(oracle.spiral_offsets(r, st), g[key])
        assert np.array_equal(spiral_offsets(r, st), g[key])


def test_oracle_block_match_golden():
    """Oracle spiral search == the reference's spiral_search (temporal.py:183-226) on
    integer / quarter-pixel shifts, noise, border centres and three GopConfigs."""
    from oracle import oracle

    g = golden("temporal.npz")
    for ci in range(int(g["n_bm"])):
        for gi in range(3):
            k = f"bm{ci}_{gi}"
            f, nx, ny, sd = oracle.block_match(g[f"bm{ci}_prev"], g[f"bm{ci}_cur"], g[f"bm{ci}_x"], g[f"bm{ci}_y"],
                                               **_gop_kw(g[f"{k}_gop"]))
            assert np.array_equal(f, g[f"{k}_found"]), k
            assert np.array_equal(nx, g[f"{k}_nx"]) and np.array_equal(ny, g[f"{k}_ny"]), k
            assert np.array_equal(sd, g[f"{k}_sad"]), k


@pytest.mark.parametrize("name", ["small_temporal", "scene_temporal"])
def test_oracle_temporal_pipeline_golden(name):
    """Oracle run_pipeline(mode='temporal') == the reference (pipeline.py:281-345)."""
    from oracle import oracle
    from paper_1503_06959_b200.pattern import default_pattern

    g = golden(f"pipeline_{name}.npz")
    ref = oracle.run_sequence(list(g["frames"]), default_pattern(), threshold=int(g["threshold"]),
                              n_octaves=int(g["n_octaves"]), mode="temporal", gop=_gop_kw(g["gop"]))
    off = g["offsets"]
    for n, e in enumerate(ref):
        a, b = off[n], off[n + 1]
        for k in ("x", "y", "score", "origin", "age", "desc"):
            assert np.array_equal(getattr(e, k), g[k][a:b]), (n, k)
        assert np.abs(e.sigma - g["sigma"][a:b]).max(initial=0) <= 1e-12
        assert np.abs(e.theta - g["theta"][a:b]).max(initial=0) <= 1e-9
        assert (e.n_detected, e.n_total, e.n_dropped) == (g["r_n_detected"][n], g["r_n_total"][n], g["r_n_dropped"][n])
        assert e.coverage == g["r_coverage"][n]


def test_gop_config_validation():
    from paper_1503_06959_b200.types import GopConfig

    for kw, msg in [({"delta": 0}, "GOP length"), ({"patch": 15}, "patch side"), ({"fine_step": 3.0}, "fine_step"),
                    ({"t_et": 0.0}, "SAD thresholds")]:
        with pytest.raises(ValueError, match=msg):
            GopConfig(**kw)


def test_divergence_report_matches_reference():
    """pipeline.divergence_from_arrays (the host pairing of divergence_report,
    pipeline.py:348-398) applied to the oracle's masked and full runs equals
    the reference's DivergenceStat counts on its c03 trend scene (half size)."""
    from oracle import oracle
    from paper_1503_06959_b200.pattern import default_pattern
    from paper_1503_06959_b200.pipeline import divergence_from_arrays

    g = golden("divergence.npz")
    frames = list(g["frames"])
    kw = dict(threshold=int(g["threshold"]), t_i=float(g["t_i"]))
    m = oracle.run_sequence(frames, default_pattern(), mode="intensity", **kw)
    f = oracle.run_sequence(frames, default_pattern(), mode="none", **kw)
    soa = lambda r: {"x": r.x, "y": r.y, "sigma": r.sigma}  # noqa: E731
    stats = divergence_from_arrays([soa(r) for r in m], [soa(r) for r in f])
    assert [s.common for s in stats] == g["common"].tolist()
    assert [s.only_masked for s in stats] == g["only_masked"].tolist()
    assert [s.only_full for s in stats] == g["only_full"].tolist()
    assert np.allclose([s.preserved for s in stats], g["preserved"])

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

PIPELINES = sorted(p.stem[len("pipeline_"):] for p in GOLDEN.glob("pipeline_*.npz"))


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

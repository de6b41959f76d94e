"""Output formats and sequence loading: byte-identical
to files written by the reference itself (tests/golden/formats.npz, made by
tests/golden/make_golden.py from report.dump_features / emit_report /
write_sweep_summary / io.load_sequence).  Host-side code, CPU tests; the
feature lines come from the library's native formatter (vf_format_features)."""

import json

import numpy as np
import pytest

from conftest import golden


def _frames_from_golden():
    g = golden("pipeline_scene_intensity.npz")
    off = g["offsets"]
    soa = []
    for n in range(len(off) - 1):
        a, b = off[n], off[n + 1]
        soa.append({k: g[k][a:b] for k in ("x", "y", "sigma", "theta", "origin", "desc")})
    return soa


def _edge_features():
    from paper_1503_06959_b200.types import Feature, Keypoint

    return [Feature(Keypoint(-0.0, 0.00005, 1.00005, -0.0000005), np.zeros(512, np.uint8), "detected", 0),
            Feature(Keypoint(1919.99995, 1079.12345, 12.0, 3.14159265), np.ones(512, np.uint8), "propagated", 3),
            Feature(Keypoint(0.125, 2.5e-5, 7.75, -3.1415926535), (np.arange(512) % 2).astype(np.uint8), "detected",
                    0)]


def test_dump_features_byte_identical(tmp_path):
    """SoA frames (engine layout) + Feature objects + an empty frame -> the reference's features.txt."""
    from paper_1503_06959_b200.report import dump_features

    fm = golden("formats.npz")
    frames = _frames_from_golden() + [_edge_features(), []]
    dump_features(frames, tmp_path / "features.txt")
    assert (tmp_path / "features.txt").read_bytes() == fm["features_txt"].tobytes()


def test_parse_features_round_trip(tmp_path):
    from paper_1503_06959_b200.report import dump_features, parse_features

    frames = _frames_from_golden()[:2]
    dump_features(frames, tmp_path / "f.txt")
    back = parse_features(tmp_path / "f.txt")
    for soa, fs in zip(frames, back):
        assert len(fs) == len(soa["x"])
        assert np.array_equal(np.stack([np.packbits(f.desc) for f in fs]), soa["desc"])
        assert np.allclose([f.kp.x for f in fs], soa["x"], atol=5e-5)
        assert [f.origin for f in fs] == ["propagated" if o else "detected" for o in soa["origin"]]
    (tmp_path / "bad.txt").write_text("frames 0 1\n")
    with pytest.raises(ValueError):
        parse_features(tmp_path / "bad.txt")


def test_report_csv_json_byte_identical(tmp_path):
    from paper_1503_06959_b200.report import CSV_COLUMNS, emit_report, summarize, write_sweep_summary
    from paper_1503_06959_b200.types import FrameReport

    fm = golden("formats.npz")
    n = len(fm["rep_frame"])
    reps = [FrameReport(int(fm["rep_frame"][i]), int(fm["rep_n_detected"][i]), int(fm["rep_n_propagated"][i]),
                        int(fm["rep_n_total"][i]), float(fm["rep_coverage"][i]), float(fm["rep_t_pyramid_ms"][i]),
                        float(fm["rep_t_mask_ms"][i]), float(fm["rep_t_detect_ms"][i]),
                        float(fm["rep_t_describe_ms"][i]), float(fm["rep_t_total_ms"][i]),
                        n_dropped=int(fm["rep_n_dropped"][i]),
                        accuracy=None if np.isnan(fm["rep_accuracy"][i]) else float(fm["rep_accuracy"][i]))
            for i in range(n)]
    c, j = emit_report(reps, tmp_path, prefix="frames")
    assert c.read_bytes() == fm["frames_csv"].tobytes()
    assert j.read_bytes() == fm["frames_json"].tobytes()
    p = write_sweep_summary([{"t": 10, "mpr": 12.5}, {"t": 20, "mpr": None}], tmp_path)
    assert p.read_bytes() == fm["sweep_json"].tobytes()
    assert CSV_COLUMNS[0] == "frame" and CSV_COLUMNS[-1] == "accuracy"
    assert summarize([]) == {"frames": 0}
    assert json.loads(j.read_text())["frames"] == n


def test_load_sequence_matches_reference(tmp_path):
    """Numeric filename order, names without digits last, RGB -> L, PGM + PNG, other files ignored."""
    from paper_1503_06959_b200.io import load_sequence

    fm = golden("formats.npz")
    fs = golden("formats_seq.npz")
    for i, name in enumerate(fs["names"]):
        (tmp_path / str(name)).write_bytes(fs[f"seqfile_{i}"].tobytes())
    got = load_sequence(tmp_path)
    assert np.array_equal(np.stack([f.data for f in got]), fm["seq_loaded"])
    assert [f.index for f in got] == fm["seq_index"].tolist()
    with pytest.raises(ValueError):
        load_sequence(tmp_path / "missing")
    (tmp_path / "empty").mkdir()
    with pytest.raises(ValueError):
        load_sequence(tmp_path / "empty")


def test_format_capacity_and_empty():
    import ctypes

    from paper_1503_06959_b200 import _native
    from paper_1503_06959_b200.report import format_features

    L = _native.lib()
    need = ctypes.c_int64(-1)
    assert L.vf_format_features(0, 0, 0, 0, 0, 0, 0, 0, 0, ctypes.byref(need)) == 0 and need.value == 0
    assert format_features({"x": np.zeros(0), "y": np.zeros(0), "sigma": np.zeros(0), "theta": np.zeros(0),
                            "origin": np.zeros(0, np.uint8), "desc": np.zeros((0, 64), np.uint8)}) == b""
    one = {"x": np.array([1.0]), "y": np.array([2.0]), "sigma": np.array([3.0]), "theta": np.array([0.5]),
           "origin": np.array([1], np.uint8), "desc": np.full((1, 64), 0xAB, np.uint8)}
    assert format_features(one) == b"1.0000 2.0000 3.0000 0.500000 propagated " + b"ab" * 64 + b"\n"


def test_fixed_point_formatter_matches_python():
    """The native exact %.4f / %.6f (128-bit, round half to even) equals Python's
    formatting on random, tiny, huge, negative-zero and exact-halfway values."""
    from paper_1503_06959_b200.report import format_features

    rng = np.random.default_rng(1)
    n = 20000
    vals = np.concatenate([rng.uniform(-3000, 3000, n), rng.uniform(-1, 1, n) * 10.0 ** rng.integers(-12, 4, n),
                           np.round(rng.uniform(-100, 100, n) * 20000) / 20000,
                           np.round(rng.uniform(-4, 4, n) * 2e6) / 2e6,
                           [0.0, -0.0, 0.5e-4, -0.5e-4, 1.5e-4, 2.5e-4, 1e11, -1e11, 5e-7, -5e-7, 2.5e-6, 1e13,
                            float("nan"), float("inf"), -float("inf")]])
    m = len(vals)
    f = {"x": vals, "y": vals[::-1].copy(), "sigma": np.abs(vals), "theta": vals,
         "origin": np.zeros(m, np.uint8), "desc": np.zeros((m, 64), np.uint8)}
    got = format_features(f).decode().splitlines()
    for i in range(m):
        exp = f"{f['x'][i]:.4f} {f['y'][i]:.4f} {f['sigma'][i]:.4f} {f['theta'][i]:.6f} detected "
        assert got[i].startswith(exp), (got[i][:70], exp)

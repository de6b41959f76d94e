"""Geometric verification + evaluation, CPU side:
the oracle's RANSAC against the reference's own outputs
(tests/golden/ransac.npz, made by make_golden.py from
matching.ransac_homography), the minimal-sample stream (the product's host
generator and the oracle's) against numpy's default_rng itself, and the
host-side evaluation protocols (evaluation.py) against the reference's
outputs and its tests/test_evaluation.py semantics."""

import numpy as np
import pytest

from conftest import golden

H_RTOL = 1e-9   # model entries, relative to max |H| (rounding of a different SVD path)


def test_sample_tables_vs_numpy():
    from oracle import oracle
    from paper_1503_06959_b200.matching import ransac_samples

    g = golden("ransac.npz")
    for i in range(int(g["n_samples"])):
        seed, n, tab = int(g[f"s{i}_seed"]), int(g[f"s{i}_n"]), g[f"s{i}_tab"]
        assert np.array_equal(ransac_samples(seed, n, len(tab)), tab), (seed, n)
        assert np.array_equal(oracle.ransac_samples(seed, n, len(tab)), tab), (seed, n)
    rng = np.random.default_rng(0)
    for _ in range(20):   # fresh draws from numpy itself, seeds across the 32/64-bit word boundary
        seed = int(rng.integers(0, 2**63)) >> int(rng.integers(0, 63))
        n = int(rng.integers(4, 100000))
        r = np.random.default_rng(seed)
        ref = np.array([r.choice(n, 4, replace=False) for _ in range(64)])
        assert np.array_equal(ransac_samples(seed, n, 64), ref), (seed, n)


def test_sampler_errors():
    from paper_1503_06959_b200.matching import ransac_samples

    with pytest.raises(ValueError):
        ransac_samples(-1, 10, 4)
    with pytest.raises(ValueError):
        ransac_samples(0, 3, 4)


def test_oracle_ransac_golden():
    from oracle import oracle

    g = golden("ransac.npz")
    for i in range(int(g["n_ransac"])):
        iters, tol, _ = g[f"r{i}_par"]
        h, inl = oracle.ransac_homography(g[f"r{i}_src"], g[f"r{i}_dst"], int(iters), float(tol), int(g[f"r{i}_seed"]))
        H = g[f"r{i}_H"]
        if np.isnan(H).any():
            assert h is None and inl == [], i
            continue
        assert np.abs(h - H).max() <= H_RTOL * np.abs(H).max(), i
        assert inl == list(g[f"r{i}_inl"]), i


def test_project_points():
    from paper_1503_06959_b200.matching import project_points

    h = np.array([[2.0, 0.0, 1.0], [0.0, 3.0, -1.0], [0.0, 0.0, 1.0]])
    assert np.allclose(project_points(h, np.array([[1.0, 2.0]])), [[3.0, 5.0]])
    z0 = np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [1.0, 0.0, -1.0]])   # z = x - 1 = 0 at x = 1
    assert np.allclose(project_points(z0, np.array([[1.0, 4.0]])), [[1e12, 4e12]])


def test_average_precision_golden_and_cases():
    from paper_1503_06959_b200.evaluation import RankedList, average_precision

    g = golden("ransac.npz")
    for rel, tot, ap in zip(g["ap_rel"], g["ap_tot"], g["ap_val"]):
        rel = rel[rel >= 0]
        assert average_precision(RankedList(list(range(rel.size)), rel, int(tot))) == ap

    def ranked(r, total=None):
        r = np.asarray(r)
        return RankedList(list(range(r.size)), r, int(r.sum()) if total is None else total)

    assert average_precision(ranked([1, 1, 1, 0, 0])) == 1.0
    assert abs(average_precision(ranked([1, 0, 1], total=2)) - 5.0 / 6.0) < 1e-12
    assert average_precision(ranked([0, 0, 0], total=3)) == 0.0
    assert average_precision(ranked([], total=1)) == 0.0
    assert average_precision(ranked([1, 0, 1], total=2)) > average_precision(ranked([0, 1, 1], total=2))
    with pytest.raises(ValueError):
        average_precision(ranked([0, 0], total=0))


def test_sequence_and_map():
    from paper_1503_06959_b200.evaluation import mean_average_precision, sequence_ap

    assert sequence_ap([0.5, 1.0]) == 0.75
    assert mean_average_precision([0.2, 0.4, 0.9]) == pytest.approx(0.5)
    for f in (sequence_ap, mean_average_precision):
        with pytest.raises(ValueError):
            f([])


def test_tracking_accuracy_and_files(tmp_path):
    from paper_1503_06959_b200.evaluation import (GroundTruthRecord, ObjectEstimate, corner_geometry,
                                                  load_ground_truth, load_relevance, save_ground_truth,
                                                  tracking_accuracy)

    def est(oid, cx, cy):
        return ObjectEstimate(oid, np.array([[cx - 5, cy - 5], [cx + 5, cy - 5], [cx + 5, cy + 5], [cx - 5, cy + 5]]))

    truth = [GroundTruthRecord(0, 1, 100.0, 80.0)]
    assert tracking_accuracy({0: est(1, 110.0, 80.0)}, truth) == 1.0     # boundary inclusive
    assert tracking_accuracy({0: est(1, 110.5, 80.0)}, truth) == 0.0
    assert tracking_accuracy({0: est(2, 100.0, 80.0)}, truth) == 0.0
    two = truth + [GroundTruthRecord(1, 1, 102.0, 81.0)]
    assert tracking_accuracy({0: est(1, 100.0, 80.0), 1: None}, two) == 0.5
    with pytest.raises(ValueError):
        tracking_accuracy({}, [])
    assert np.allclose(est(0, 50.0, 60.0).centroid, [50.0, 60.0])
    assert np.array_equal(corner_geometry(200, 100), [[0, 0], [199, 0], [199, 99], [0, 99]])
    recs = [GroundTruthRecord(0, 2, 100.5, 200.25), GroundTruthRecord(1, 2, 103.5, 202.25)]
    save_ground_truth(recs, tmp_path / "t.txt")
    assert (tmp_path / "t.txt").read_text() == "0 2 100.5000 200.2500\n1 2 103.5000 202.2500\n"
    assert load_ground_truth(tmp_path / "t.txt") == recs
    (tmp_path / "bad.txt").write_text("0 1 2\n")
    with pytest.raises(ValueError):
        load_ground_truth(tmp_path / "bad.txt")
    (tmp_path / "rel.txt").write_text("# comment\nq0 a b c\nq1 d\nq2\n")
    assert load_relevance(tmp_path / "rel.txt") == {"q0": {"a", "b", "c"}, "q1": {"d"}, "q2": set()}

"""GPU parity of descriptor matching through the C ABI
(vf_hamming_matrix / vf_radius_match) against the reference's own outputs
(tests/golden/matching.npz) and the pinned CPU oracle, plus the reference's
radius-match unit cases (tests/test_matching.py:30-64) and size-independent
properties at frame-feature scale."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def feats(bits):
    from paper_1503_06959_b200.types import Feature, Keypoint

    return [Feature(Keypoint(0.0, 0.0, 1.0), np.asarray(b, np.uint8)) for b in bits]


def as_rows(ms):
    return np.array([[m.query_idx, m.ref_idx, m.distance] for m in ms], np.int64).reshape(-1, 3)


def test_hamming_matrix_golden():
    from paper_1503_06959_b200.matching import hamming_matrix

    g = golden("matching.npz")
    for tag in "abcd":   # 64-, 7- and 32-byte rows, ragged tile edges
        assert np.array_equal(hamming_matrix(g[f"{tag}_q"], g[f"{tag}_r"]), g[f"{tag}_d"]), tag


def test_radius_match_golden():
    from paper_1503_06959_b200.matching import radius_match

    g = golden("matching.npz")
    for t_m in (0, 50, 102, 260):   # 7419 matches at 260: the dense path
        assert np.array_equal(as_rows(radius_match(feats(g["plant_q_bits"]), feats(g["plant_r_bits"]), t_m)),
                              g[f"plant_{t_m}"]), t_m
    assert np.array_equal(as_rows(radius_match(feats(g["w56_q_bits"]), feats(g["w56_r_bits"]), 24)), g["w56_24"])


def test_reference_unit_cases():
    """tests/test_matching.py:30-64 semantics."""
    from paper_1503_06959_b200.matching import DEFAULT_MATCH_RADIUS, radius_match

    rng = np.random.default_rng(3)
    assert DEFAULT_MATCH_RADIUS == 102
    f8 = feats(rng.integers(0, 2, (8, 512)))
    self_pairs = {(m.query_idx, m.ref_idx) for m in radius_match(f8, f8, 102) if m.distance == 0}
    assert {(i, i) for i in range(8)} <= self_pairs
    base = rng.integers(0, 2, 512).astype(np.uint8)

    def flip(k):
        b = base.copy()
        b[rng.choice(512, k, replace=False)] ^= 1
        return b

    assert len(radius_match(feats([base]), feats([flip(102)]), 102)) == 1
    assert len(radius_match(feats([base]), feats([flip(103)]), 102)) == 0
    assert len(radius_match(feats([base]), feats([flip(0), flip(10), flip(50)]), 102)) == 3
    # one query, many references: np.nonzero order is reference order
    refs = feats([flip(k) for k in (0, 90, 10, 200, 50, 3, 101, 7)])
    got = [(m.ref_idx, m.distance) for m in radius_match(feats([base]), refs, 102)]
    assert got == [(0, 0), (1, 90), (2, 10), (4, 50), (5, 3), (6, 101), (7, 7)]
    q, r = feats(rng.integers(0, 2, (6, 512))), feats(rng.integers(0, 2, (6, 512)))
    fwd = {(m.query_idx, m.ref_idx) for m in radius_match(q, r, 260)}
    rev = {(m.ref_idx, m.query_idx) for m in radius_match(r, q, 260)}
    assert fwd == rev
    assert radius_match([], q, 102) == [] and radius_match(q, [], 102) == []
    with pytest.raises(ValueError):
        radius_match(feats([base]), feats([base[:256]]), 102)


def test_large_random_vs_oracle_and_capacity_retry():
    """3000 x 2500 rows vs the oracle; t_m = 512 returns every pair (7.5 M
    matches, far past the first buffer) through the capacity retry."""
    import torch

    from oracle import oracle
    from paper_1503_06959_b200.matching import hamming_matrix_device, radius_match_device

    rng = np.random.default_rng(11)
    q = rng.integers(0, 256, (3000, 64), dtype=np.uint8)
    r = rng.integers(0, 256, (2500, 64), dtype=np.uint8)
    ref = oracle.hamming_matrix(q, r)
    qd, rd = torch.from_numpy(q).cuda(), torch.from_numpy(r).cuda()
    assert np.array_equal(hamming_matrix_device(qd, rd).cpu().numpy(), ref)
    for t_m in (230, 512):
        qi, ri, d = radius_match_device(qd, rd, t_m)
        eq, er, ed = oracle.radius_match(q, r, t_m)
        assert np.array_equal(qi.cpu().numpy(), eq) and np.array_equal(ri.cpu().numpy(), er)
        assert np.array_equal(d.cpu().numpy(), ed)


def test_frame_features_properties():
    """Packed descriptors of two consecutive 1080p frames of a config-5 stream
    (device-resident, from the engine): the GPU matrix equals the oracle's on
    a row sample, is symmetric (H(a, b) = H(b, a)^T), self-distances are 0,
    and radius_match agrees with the matrix."""
    import torch

    from oracle import oracle
    from paper_1503_06959_b200 import scenes
    from paper_1503_06959_b200.engine import FeatureEngine
    from paper_1503_06959_b200.matching import hamming_matrix_device, radius_match_device
    from paper_1503_06959_b200.types import MaskConfig, PipelineConfig

    fr = scenes.generate(scenes.CONFIGS[5], 2, streams=[2]).numpy()[0]
    eng = FeatureEngine(1920, 1080, PipelineConfig(mask=MaskConfig(mode="intensity")), n_streams=1)
    dev = torch.from_numpy(fr).cuda()
    descs = []
    for n in range(2):
        eng.process(dev[n:n + 1])
        descs.append(torch.from_numpy(eng.features_host(0)["desc"]).cuda())
    eng.close()
    a, b = descs
    assert a.shape[0] > 1000 and b.shape[0] > 1000
    hab = hamming_matrix_device(a, b)
    hba = hamming_matrix_device(b, a)
    assert torch.equal(hab, hba.t())
    assert int(hamming_matrix_device(a, a).diagonal().abs().sum()) == 0
    rows = np.random.default_rng(0).choice(a.shape[0], 200, replace=False)
    assert np.array_equal(hab.cpu().numpy()[rows], oracle.hamming_matrix(a.cpu().numpy()[rows], b.cpu().numpy()))
    qi, ri, d = radius_match_device(a, b, 102)
    m = (hab <= 102).nonzero()
    assert torch.equal(qi.long(), m[:, 0]) and torch.equal(ri.long(), m[:, 1])
    assert torch.equal(d, hab[m[:, 0], m[:, 1]])
    assert qi.numel() > 0            # propagated features re-match across frames


def test_unaligned_rows_take_popc_path():
    """Rows at an odd byte address (4-byte alignment fails) use the POPC kernels: same distances."""
    import torch

    from oracle import oracle
    from paper_1503_06959_b200.matching import hamming_matrix_device, radius_match_device

    rng = np.random.default_rng(5)
    q = rng.integers(0, 256, (300, 64), dtype=np.uint8)
    r = rng.integers(0, 256, (257, 64), dtype=np.uint8)
    buf = torch.zeros(300 * 64 + 1, dtype=torch.uint8, device="cuda")
    buf[1:] = torch.from_numpy(q.reshape(-1)).cuda()
    qd = buf[1:].view(300, 64)                     # data_ptr % 4 == 1
    assert qd.data_ptr() % 4 == 1
    rd = torch.from_numpy(r).cuda()
    assert np.array_equal(hamming_matrix_device(qd, rd).cpu().numpy(), oracle.hamming_matrix(q, r))
    qi, ri, d = radius_match_device(qd, rd, 240)
    eq, er, ed = oracle.radius_match(q, r, 240)
    assert np.array_equal(qi.cpu().numpy(), eq) and np.array_equal(ri.cpu().numpy(), er)
    assert np.array_equal(d.cpu().numpy(), ed)

"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch dir (the mount is read-only and
misses ``data/sampling_pattern_v1.npz``), regenerates the pattern asset with
the reference's own ``python -m vidfeat.pattern`` code path, imports
``vidfeat`` from there (numba path, the reference default, accel.py:33) and
writes small ``.npz`` fixtures next to this script.  The fixtures hold the
inputs too, so tests never need the reference at run time.
"""

from __future__ import annotations

import os
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg")


def import_reference():
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    os.environ.setdefault("NUMBA_CACHE_DIR", str(Path(tempfile.gettempdir()) / "vidfeat_numba_cache"))
    sys.dont_write_bytecode = True
    scratch = Path(tempfile.gettempdir()) / "vidfeat_ref_copy"
    if not (scratch / "src" / "vidfeat" / "data" / "sampling_pattern_v1.npz").exists():
        if scratch.exists():
            shutil.rmtree(scratch)
        shutil.copytree(REF, scratch)
        sys.path.insert(0, str(scratch / "src"))
        import vidfeat.pattern as vp  # noqa: E402

        vp._regenerate()
    else:
        sys.path.insert(0, str(scratch / "src"))
    import vidfeat  # noqa: F401

    return vidfeat


def feats_to_arrays(per_frame):
    """list[list[Feature]] -> flat SoA + frame offsets (packed descriptors)."""
    offs = [0]
    cols = {k: [] for k in ("x", "y", "sigma", "theta", "score", "origin", "age", "desc")}
    for fs in per_frame:
        for f in fs:
            cols["x"].append(f.kp.x)
            cols["y"].append(f.kp.y)
            cols["sigma"].append(f.kp.sigma)
            cols["theta"].append(f.kp.theta)
            cols["score"].append(f.kp.score)
            cols["origin"].append(0 if f.origin == "detected" else 1)
            cols["age"].append(f.age)
            cols["desc"].append(np.packbits(f.desc))
        offs.append(offs[-1] + len(fs))
    out = {
        "offsets": np.array(offs, np.int64),
        "x": np.array(cols["x"], np.float64),
        "y": np.array(cols["y"], np.float64),
        "sigma": np.array(cols["sigma"], np.float64),
        "theta": np.array(cols["theta"], np.float64),
        "score": np.array(cols["score"], np.float64),
        "origin": np.array(cols["origin"], np.uint8),
        "age": np.array(cols["age"], np.int32),
        "desc": np.array(cols["desc"], np.uint8).reshape(-1, 64),
    }
    return out


def reports_to_arrays(reports):
    return {
        "r_n_detected": np.array([r.n_detected for r in reports], np.int64),
        "r_n_propagated": np.array([r.n_propagated for r in reports], np.int64),
        "r_n_total": np.array([r.n_total for r in reports], np.int64),
        "r_n_dropped": np.array([r.n_dropped for r in reports], np.int64),
        "r_coverage": np.array([r.coverage for r in reports], np.float64),
    }


def main():
    vf = import_reference()
    from vidfeat import detector, descriptor, masking, pattern, pipeline, pyramid, synth
    from vidfeat.masking import MaskConfig
    from vidfeat.pipeline import PipelineConfig, run_pipeline
    from vidfeat.pyramid import GrayFrame

    assert vf.accel.USE_NUMBA, "golden vectors come from the reference's default (numba) path"

    # 1. pattern (pattern.py:49-72) -----------------------------------------
    p = pattern.default_pattern()
    np.savez_compressed(HERE / "pattern_v1.npz", points=p.points, radii=p.radii,
                        short_pairs=p.short_pairs, long_pairs=p.long_pairs)

    # 2. pyramid (pyramid.py:97-125) ---------------------------------------
    rng = np.random.default_rng(12345)
    pyr_out = {}
    for tag, (w, h, O) in {"a": (200, 150, 4), "b": (97, 61, 3), "c": (64, 64, 4)}.items():
        f = rng.integers(0, 256, (h, w), dtype=np.uint8)
        pyr = pyramid.build_pyramid(GrayFrame(f), O)
        pyr_out[f"{tag}_frame"] = f
        pyr_out[f"{tag}_O"] = np.array(O)
        for i, layer in enumerate(pyr.layers):
            pyr_out[f"{tag}_layer{i}"] = layer.frame.data
            pyr_out[f"{tag}_scale{i}"] = np.array(layer.scale)
    np.savez_compressed(HERE / "pyramid.npz", **pyr_out)

    # 3. score maps (detector.py:107-172) incl. gating and KATs --------------
    sm = {}
    rng = np.random.default_rng(7)
    k = 0
    for trial in range(8):
        h, w = (64, 64) if trial < 6 else (40, 71)
        data = rng.integers(0, 256, (h, w), dtype=np.uint8)
        mask = (rng.random((h, w)) < 0.7).astype(np.uint8) if trial % 2 else None
        for t in (1, 10, 30, 55, 200):
            smap = detector._score_map(data, t, mask)
            sm[f"data{k}"] = data
            sm[f"mask{k}"] = np.ones((h, w), np.uint8) if mask is None else mask
            sm[f"t{k}"] = np.array(t)
            sm[f"score{k}"] = smap.astype(np.uint8)
            assert smap.max() < 256
            k += 1
    sm["n"] = np.array(k)
    # KATs from tests/test_detector.py:48-73 (ring patterns around (8, 8))
    rings = [[200] * 12 + [100] * 4, [141] * 9 + [100] * 7, [141] * 8 + [100] * 8,
             [30] * 10 + [200] * 6, [255] * 5 + [100] * 7 + [255] * 4]
    centers = [100, 100, 100, 200, 100]
    kat = []
    for ring, c in zip(rings, centers):
        d = np.full((16, 16), c, np.uint8)
        for (dx, dy), v in zip(detector.CIRCLE, ring):
            d[8 + dy, 8 + dx] = v
        kat.append((d, detector.ast_corner_score(GrayFrame(d), 8, 8)))
    sm["kat_data"] = np.stack([d for d, _ in kat])
    sm["kat_score"] = np.array([s for _, s in kat], np.int64)
    np.savez_compressed(HERE / "score_maps.npz", **sm)

    # 4. NMS + refinement (detector.py:239-324) ----------------------------
    nm = {}
    rng = np.random.default_rng(99)
    for tag, (w, h, O, t) in {"a": (128, 128, 3, 20), "b": (160, 120, 4, 30), "c": (97, 75, 2, 15)}.items():
        f = rng.integers(0, 256, (h, w), dtype=np.uint8)
        pyr = pyramid.build_pyramid(GrayFrame(f), O)
        maps = [detector._score_map(l.frame.data, t, None) for l in pyr.layers]
        kps = detector._nms_from_maps(maps, pyr)
        nm[f"{tag}_frame"] = f
        nm[f"{tag}_O"] = np.array(O)
        nm[f"{tag}_t"] = np.array(t)
        for i, m in enumerate(maps):
            nm[f"{tag}_map{i}"] = m.astype(np.uint8)
        nm[f"{tag}_x"] = np.array([q.x for q in kps])
        nm[f"{tag}_y"] = np.array([q.y for q in kps])
        nm[f"{tag}_sigma"] = np.array([q.sigma for q in kps])
        nm[f"{tag}_score"] = np.array([q.score for q in kps])
    # the reference's own NMS unit cases (tests/test_detector.py:126-181)
    pyr = pyramid.build_pyramid(GrayFrame(np.zeros((64, 64), np.uint8)), 2)
    C = detector.Candidate
    cases = [
        {("octave", 0): [C(20, 24, ("octave", 0), 50)]},
        {("octave", 0): [C(20, 24, ("octave", 0), 10), C(21, 24, ("octave", 0), 12)]},
        {("octave", 0): [C(20, 24, ("octave", 0), 10), C(21, 24, ("octave", 0), 10)]},
        {("octave", 0): [C(20, 24, ("octave", 0), 10)], ("intra", 0): [C(13, 16, ("intra", 0), 50)]},
        {("intra", 1): [C(10, 10, ("intra", 1), 30)]},
    ]
    for ci, cands in enumerate(cases):
        kps = detector.nms_and_refine(cands, pyr)
        nm[f"case{ci}_cands"] = np.array(
            [[next(i for i, l in enumerate(pyr.layers) if (l.kind, l.level) == lid), c.x, c.y, c.score]
             for lid, cl in cands.items() for c in cl], np.int64).reshape(-1, 4)
        nm[f"case{ci}_kps"] = np.array([[q.x, q.y, q.sigma, q.score] for q in kps]).reshape(-1, 4)
    nm["n_cases"] = np.array(len(cases))
    np.savez_compressed(HERE / "nms.npz", **nm)

    # 5. orientation + descriptor (descriptor.py:85-232) -------------------
    de = {}
    rng = np.random.default_rng(2024)
    data = rng.integers(0, 256, (96, 96), dtype=np.uint8)
    n = 64
    kx = rng.uniform(30, 66, n)
    ky = rng.uniform(30, 66, n)
    sg = rng.choice([1.0, 1.5, 2.0, 2.5], n) * rng.uniform(0.9, 1.1, n)
    th = rng.uniform(-3.1, 3.1, n)
    frame = GrayFrame(data)
    kps = [detector.Keypoint(float(a), float(b), float(c)) for a, b, c in zip(kx, ky, sg)]
    de["data"] = data
    de["kx"], de["ky"], de["sigma"], de["theta_in"] = kx, ky, sg, th
    de["orient"] = descriptor.orientations_batch(frame, kps, p)
    de["desc_theta_in"] = np.packbits(descriptor.describe_batch(frame, kps, th, p), axis=1)
    de["desc_orient"] = np.packbits(descriptor.describe_batch(frame, kps, de["orient"], p), axis=1)
    # KATs (tests/test_descriptor.py:63-81): constant, x-ramp, y-ramp, edge
    xs, ys = np.meshgrid(np.arange(64), np.arange(64))
    kat_frames = [np.full((64, 64), 90, np.uint8), np.clip(xs * 3, 0, 255).astype(np.uint8),
                  np.clip(ys * 3, 0, 255).astype(np.uint8)]
    edge = np.full((64, 64), 50, np.uint8)
    edge[:, :32] = 200
    kat_frames.append(edge)
    de["kat_frames"] = np.stack(kat_frames)
    de["kat_orient"] = np.array([descriptor.estimate_orientation(GrayFrame(f), detector.Keypoint(32.0, 32.0, 1.0), p)
                                 for f in kat_frames])
    de["kat_desc"] = np.stack([np.packbits(descriptor.describe(GrayFrame(f), detector.Keypoint(32.0, 32.0, 1.0), 0.0, p))
                               for f in kat_frames])
    np.savez_compressed(HERE / "describe.npz", **de)

    # 6. masks (masking.py:84-184) -----------------------------------------
    mk = {}
    rng = np.random.default_rng(5)
    a = rng.integers(0, 256, (60, 80), dtype=np.uint8)
    b = np.clip(a.astype(np.int16) + rng.integers(-40, 41, (60, 80)), 0, 255).astype(np.uint8)
    mk["idm_a"], mk["idm_b"] = a, b
    for t_i in (-1.0, 0.0, 19.5, 20.0, 30.0):
        mk[f"idm_{t_i}"] = masking.intensity_diff_mask(GrayFrame(a), GrayFrame(b), t_i).bits
    xs_ = np.concatenate([rng.uniform(0, 640, 300), [639.0, 0.0, 639.999999]])
    ys_ = np.concatenate([rng.uniform(0, 480, 300), [479.0, 0.0, 479.999999]])
    F = masking.Feature
    feats = [F(detector.Keypoint(float(x), float(y), 1.0), np.zeros(512, np.uint8)) for x, y in zip(xs_, ys_)]
    mk["bin_x"], mk["bin_y"] = xs_, ys_
    mk["bin_hist_16"] = masking.binning_histogram(feats, (640, 480), (16, 16))
    mk["bin_hist_3x5"] = masking.binning_histogram(feats, (640, 480), (3, 5))
    bits = rng.integers(0, 2, (6, 8)).astype(np.uint8)
    mk["up_bits"] = bits
    mk["up_full"] = masking.upsample_mask(masking.SubsampledMask(bits, cell_w=9, cell_h=9), (70, 50)).bits
    np.savez_compressed(HERE / "masks.npz", **mk)

    # 7. whole-pipeline sequences (pipeline.py:207-278) ---------------------
    small, _ = synth.synth_sequence(
        synth.moving_object_scene((128, 96), object_frac=0.2, velocity=(3.0, 0.0), seed=6), 6, (128, 96), seed=6)
    static, _ = synth.synth_sequence(synth.static_scene(seed=8), 6, (128, 96), seed=8)
    rng = np.random.default_rng(42)
    rnd = [GrayFrame(rng.integers(0, 256, (240, 320), dtype=np.uint8), index=i) for i in range(3)]
    sys.path.insert(0, str(HERE.parents[1]))
    from paper_1503_06959_b200 import scenes  # our seeded BASELINE config-1 scene generator

    cfg1 = scenes.SceneConfig(320, 240, 5, 1, "objects", (3, 3), (1.0, 3.0), noise_sigma=2.0, seed=11)
    scn = [GrayFrame(f, i) for i, f in enumerate(scenes.generate(cfg1)[0].numpy())]
    runs = {
        "small_none": (small, PipelineConfig(threshold=25, mask=MaskConfig(mode="none"))),
        "small_intensity": (small, PipelineConfig(threshold=25, mask=MaskConfig(mode="intensity", t_i=15))),
        "small_binning": (small, PipelineConfig(threshold=25, mask=MaskConfig(mode="binning", t_h=1, grid=(8, 8)))),
        "small_perlayer": (small, PipelineConfig(threshold=25, mask=MaskConfig(mode="intensity", t_i=15, per_layer=True))),
        "small_octave1": (small, PipelineConfig(threshold=25, n_octaves=3, mask=MaskConfig(mode="intensity", t_i=10, octave_for_mask=1))),
        "static_intensity": (static, PipelineConfig(threshold=25, mask=MaskConfig(mode="intensity", t_i=5))),
        "random_forced": (rnd, PipelineConfig(mask=MaskConfig(mode="intensity", t_i=-1.0))),
        "random_none": (rnd, PipelineConfig(mask=MaskConfig(mode="none"))),
        "scene_intensity": (scn, PipelineConfig(mask=MaskConfig(mode="intensity"))),
        "scene_binning": (scn, PipelineConfig(mask=MaskConfig(mode="binning"))),
    }
    for name, (frames, cfg) in runs.items():
        feats, reports = run_pipeline(frames, cfg)
        mc = cfg.mask
        np.savez_compressed(
            HERE / f"pipeline_{name}.npz",
            frames=np.stack([f.data for f in frames]),
            threshold=np.array(cfg.threshold), n_octaves=np.array(cfg.n_octaves),
            mode=np.array(mc.mode), t_i=np.array(mc.t_i), t_h=np.array(mc.t_h), grid=np.array(mc.grid),
            octave_for_mask=np.array(-1 if mc.octave_for_mask is None else mc.octave_for_mask),
            per_layer=np.array(mc.per_layer),
            **feats_to_arrays(feats), **reports_to_arrays(reports))
        print(name, [len(f) for f in feats])


def make_matching():
    """8. descriptor matching (matching.py:47-94), SURVEY.md 8(f) rank 1."""
    import_reference()
    from vidfeat import matching
    from vidfeat.detector import Keypoint
    from vidfeat.masking import Feature

    mt = {}
    rng = np.random.default_rng(31)
    # tests/test_kernel_equivalence.py:74-79 shapes, plus a larger random pair
    for tag, (nq, nr, nb) in {"a": (17, 23, 64), "b": (150, 133, 64), "c": (9, 11, 7), "d": (33, 5, 32)}.items():
        q = rng.integers(0, 256, (nq, nb), dtype=np.uint8)
        r = rng.integers(0, 256, (nr, nb), dtype=np.uint8)
        mt[f"{tag}_q"], mt[f"{tag}_r"] = q, r
        mt[f"{tag}_d"] = matching.hamming_matrix(q, r)
    # planted near-duplicates (tests/test_matching.py:30-64 style): distances
    # 0, 10, 50, 101, 102, 103, 200 from each query, shuffled into the refs
    base = rng.integers(0, 2, (40, 512)).astype(np.uint8)
    refs = []
    for i in range(40):
        for k in (0, 10, 50, 101, 102, 103, 200):
            b = base[i].copy()
            b[rng.choice(512, k, replace=False)] ^= 1
            refs.append(b)
    refs = np.stack(refs)[rng.permutation(len(refs))]

    def feats(bits):
        return [Feature(Keypoint(0.0, 0.0, 1.0), b.astype(np.uint8), "detected", 0) for b in bits]

    mt["plant_q_bits"], mt["plant_r_bits"] = base, refs
    for t_m in (0, 50, 102, 260):
        ms = matching.radius_match(feats(base), feats(refs), t_m)
        mt[f"plant_{t_m}"] = np.array([[m.query_idx, m.ref_idx, m.distance] for m in ms], np.int64).reshape(-1, 3)
    # 56-bit descriptors (7 packed bytes)
    q56 = rng.integers(0, 2, (12, 56)).astype(np.uint8)
    r56 = rng.integers(0, 2, (15, 56)).astype(np.uint8)
    mt["w56_q_bits"], mt["w56_r_bits"] = q56, r56
    ms = matching.radius_match(feats(q56), feats(r56), 24)
    mt["w56_24"] = np.array([[m.query_idx, m.ref_idx, m.distance] for m in ms], np.int64).reshape(-1, 3)
    mt["default_radius"] = np.array(matching.DEFAULT_MATCH_RADIUS)
    np.savez_compressed(HERE / "matching.npz", **mt)
    print("matching", {k: v.shape for k, v in mt.items() if k.startswith("plant_") and v.ndim == 2})


def make_temporal():
    """9. temporal block-matching baseline (temporal.py, pipeline.py:281-345), SURVEY.md 8(f) rank 2."""
    import_reference()
    import math

    from vidfeat import synth, temporal
    from vidfeat.masking import MaskConfig
    from vidfeat.pipeline import PipelineConfig, run_pipeline
    from vidfeat.pyramid import GrayFrame

    tm = {}
    tm["coarse_12_2"] = temporal.spiral_offsets(12.0, 2.0)
    tm["fine_175_025"] = temporal.spiral_offsets(1.75, 0.25)
    tm["odd_5_1"] = temporal.spiral_offsets(5.0, 1.0)
    # per-feature searches: prev = smooth texture, cur = prev shifted (integer
    # and quarter-pixel bilinear) + noise; centres include border cases
    rng = np.random.default_rng(77)
    H, W = 120, 160
    base = rng.integers(0, 256, (H + 8, W + 8)).astype(np.float64)
    k = np.ones(5) / 5
    base = np.apply_along_axis(lambda r: np.convolve(r, k, "same"), 0, base)
    base = np.apply_along_axis(lambda r: np.convolve(r, k, "same"), 1, base)
    prev = np.clip(base[4:4 + H, 4:4 + W] * 1.6 - 60, 0, 255).astype(np.uint8)
    cases = []
    for ci, (sx, sy, noise) in enumerate([(3.0, -2.0, 0.0), (1.25, 0.5, 2.0), (-5.5, 4.75, 4.0), (9.0, 9.0, 8.0),
                                          (0.0, 0.0, 30.0)]):
        yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
        srcx, srcy = np.clip(xx - sx, 0, W - 1.001), np.clip(yy - sy, 0, H - 1.001)
        x0, y0 = np.floor(srcx).astype(int), np.floor(srcy).astype(int)
        ax, ay = srcx - x0, srcy - y0
        pf = prev.astype(np.float64)
        cur = ((1 - ax) * (1 - ay) * pf[y0, x0] + ax * (1 - ay) * pf[y0, x0 + 1] + (1 - ax) * ay * pf[y0 + 1, x0]
               + ax * ay * pf[y0 + 1, x0 + 1])
        cur = np.clip(np.rint(cur + rng.normal(0, noise, cur.shape)), 0, 255).astype(np.uint8)
        xs = np.concatenate([rng.uniform(0, W, 60), [7.5, 8.0, W - 8.5, W - 8.0, 152.4]])
        ys = np.concatenate([rng.uniform(0, H, 60), [7.5, 8.0, H - 8.5, H - 8.0, 3.0]])
        for gi, g in enumerate([temporal.GopConfig(), temporal.GopConfig(t_et=50.0, t_bm=2500.0),
                                temporal.GopConfig(t_et=1.0, t_bm=900.0, coarse_window=6.0)]):
            found, nx, ny, sad = [], [], [], []
            half = g.patch // 2
            for x, y in zip(xs, ys):
                cxi, cyi = int(math.floor(x + 0.5)), int(math.floor(y + 0.5))
                tlx, tly = cxi - half, cyi - half
                ok = not (tlx < 0 or tly < 0 or tlx + g.patch > W or tly + g.patch > H)
                res = (temporal.spiral_search(prev[tly:tly + g.patch, tlx:tlx + g.patch], GrayFrame(cur),
                                              (float(x), float(y)), g) if ok else None)
                found.append(res is not None)
                nx.append(res[0][0] if res else 0.0)
                ny.append(res[0][1] if res else 0.0)
                sad.append(res[1] if res else 0.0)
            key = f"bm{ci}_{gi}"
            tm[f"{key}_found"] = np.array(found)
            tm[f"{key}_nx"], tm[f"{key}_ny"], tm[f"{key}_sad"] = np.array(nx), np.array(ny), np.array(sad)
            tm[f"{key}_gop"] = np.array([g.delta, g.patch, g.t_bm, g.t_et, g.coarse_window, g.coarse_step,
                                         g.fine_window, g.fine_step])
        tm[f"bm{ci}_prev"], tm[f"bm{ci}_cur"], tm[f"bm{ci}_x"], tm[f"bm{ci}_y"] = prev, cur, xs, ys
    tm["n_bm"] = np.array(5)
    np.savez_compressed(HERE / "temporal.npz", **tm)
    # whole temporal pipeline runs (pipeline.py:281-345)
    small, _ = synth.synth_sequence(
        synth.moving_object_scene((128, 96), object_frac=0.2, velocity=(3.0, 0.0), seed=6), 7, (128, 96), seed=6)
    sys.path.insert(0, str(HERE.parents[1]))
    from paper_1503_06959_b200 import scenes

    cfg1 = scenes.SceneConfig(320, 240, 7, 1, "objects", (3, 3), (1.0, 3.0), noise_sigma=2.0, seed=11)
    scn = [GrayFrame(f, i) for i, f in enumerate(scenes.generate(cfg1)[0].numpy())]
    runs = {
        "small_temporal": (small, PipelineConfig(threshold=25, mask=MaskConfig(mode="temporal"),
                                                 gop=temporal.GopConfig(delta=3))),
        "scene_temporal": (scn, PipelineConfig(mask=MaskConfig(mode="temporal"), gop=temporal.GopConfig(delta=4))),
    }
    for name, (frames, cfg) in runs.items():
        feats, reports = run_pipeline(frames, cfg)
        g = cfg.gop
        np.savez_compressed(
            HERE / f"pipeline_{name}.npz",
            frames=np.stack([f.data for f in frames]), threshold=np.array(cfg.threshold),
            n_octaves=np.array(cfg.n_octaves), mode=np.array("temporal"),
            gop=np.array([g.delta, g.patch, g.t_bm, g.t_et, g.coarse_window, g.coarse_step, g.fine_window,
                          g.fine_step]),
            **feats_to_arrays(feats), **reports_to_arrays(reports))
        print(name, [len(f) for f in feats])


def make_formats():
    """10. output formats + sequence loading (report.py, io.py), SURVEY.md 8(f) rank 3."""
    import_reference()
    from vidfeat import io as vio
    from vidfeat import report as vrep
    from vidfeat.detector import Keypoint
    from vidfeat.masking import Feature
    from vidfeat.pipeline import FrameReport

    g = np.load(HERE / "pipeline_scene_intensity.npz")
    off = g["offsets"]
    frames = []
    for n in range(len(off) - 1):
        a, b = off[n], off[n + 1]
        fs = [Feature(Keypoint(float(g["x"][i]), float(g["y"][i]), float(g["sigma"][i]), float(g["theta"][i]),
                               float(g["score"][i])), np.unpackbits(g["desc"][i]),
                      "propagated" if g["origin"][i] else "detected", int(g["age"][i])) for i in range(a, b)]
        frames.append(fs)
    # edge values: -0.0, halfway cases, large coordinates, 1e-5 theta
    edge = [Feature(Keypoint(-0.0, 0.00005, 1.00005, -0.0000005), np.zeros(512, np.uint8), "detected", 0),
            Feature(Keypoint(1919.99995, 1079.12345, 12.0, 3.14159265), np.ones(512, np.uint8), "propagated", 3),
            Feature(Keypoint(0.125, 2.5e-5, 7.75, -3.1415926535), np.arange(512) % 2, "detected", 0)]
    frames.append(edge)
    frames.append([])
    tmp = Path(tempfile.mkdtemp())
    vrep.dump_features(frames, tmp / "features.txt")
    reps = [FrameReport(n, int(g["r_n_detected"][n]), int(g["r_n_propagated"][n]), int(g["r_n_total"][n]),
                        float(g["r_coverage"][n]), 1.234567 * n, 0.1 * n + 0.00005, 2.0 / 3.0, 12.5, 100.0 / 7.0,
                        n_dropped=int(g["r_n_dropped"][n]), accuracy=None if n % 2 else 0.123456789 * n)
            for n in range(len(off) - 1)]
    vrep.emit_report(reps, tmp, prefix="frames")
    vrep.write_sweep_summary([{"t": 10, "mpr": 12.5}, {"t": 20, "mpr": None}], tmp)
    fm = {"features_txt": np.frombuffer((tmp / "features.txt").read_bytes(), np.uint8),
          "frames_csv": np.frombuffer((tmp / "frames.csv").read_bytes(), np.uint8),
          "frames_json": np.frombuffer((tmp / "frames_summary.json").read_bytes(), np.uint8),
          "sweep_json": np.frombuffer((tmp / "sweep_summary.json").read_bytes(), np.uint8)}
    for k in ("frame", "n_detected", "n_propagated", "n_total", "n_dropped"):
        fm[f"rep_{k}"] = np.array([getattr(r, k) for r in reps])
    for k in ("coverage", "t_pyramid_ms", "t_mask_ms", "t_detect_ms", "t_describe_ms", "t_total_ms"):
        fm[f"rep_{k}"] = np.array([getattr(r, k) for r in reps])
    fm["rep_accuracy"] = np.array([np.nan if r.accuracy is None else r.accuracy for r in reps])
    # sequence loading: numeric order, no-digit names last, colour -> L, PGM + PNG
    rng = np.random.default_rng(8)
    seq = tmp / "seq"
    seq.mkdir()
    names = ["f_10.png", "f_2.pgm", "f_1.png", "zz.png", "f_003.pgm"]
    for k, nm in enumerate(names):
        vio.write_frame(seq / nm, rng.integers(0, 256, (24, 32), dtype=np.uint8))
    from PIL import Image
    Image.fromarray(rng.integers(0, 256, (24, 32, 3), dtype=np.uint8), mode="RGB").save(seq / "f_7.png")
    (seq / "notes.txt").write_text("ignored")
    loaded = vio.load_sequence(seq)
    fm["seq_files"] = np.array(sorted(p.name for p in seq.iterdir()))
    fm["seq_file_bytes"] = np.array([np.frombuffer((seq / nm).read_bytes(), np.uint8) for nm in fm["seq_files"]],
                                    dtype=object)
    fm["seq_loaded"] = np.stack([fr.data for fr in loaded])
    fm["seq_index"] = np.array([fr.index for fr in loaded])
    np.savez_compressed(HERE / "formats.npz", **{k: v for k, v in fm.items() if k != "seq_file_bytes"})
    # file bytes as separate entries (object arrays are not allowed without pickle)
    extra = {f"seqfile_{i}": b for i, b in enumerate(fm["seq_file_bytes"])}
    np.savez_compressed(HERE / "formats_seq.npz", names=fm["seq_files"], **extra)
    shutil.rmtree(tmp)
    print("formats", len(fm["features_txt"]), "bytes of dump")


def make_ransac():
    """9. geometric verification + evaluation (matching.py:97-220,
    evaluation.py:60-171), SURVEY.md 8(f) rank 4."""
    import_reference()
    from vidfeat import evaluation, matching
    from vidfeat.detector import Keypoint
    from vidfeat.masking import Feature

    rng = np.random.default_rng(57)
    out = {}

    def proj(h, p):
        ph = np.column_stack([p, np.ones(len(p))]) @ h.T
        return ph[:, :2] / ph[:, 2:]

    def scene(h, n_in, n_out, noise=0.0, w=640, hgt=480, tol=3.0):
        src = rng.uniform([40, 40], [w - 40, hgt - 40], (n_in, 2))
        dst = proj(h, src) + (rng.normal(0.0, noise, (n_in, 2)) if noise else 0.0)
        os_, od = [], []
        while len(os_) < n_out:
            a = rng.uniform([0, 0], [w, hgt], 2)
            b = rng.uniform([0, 0], [w, hgt], 2)
            if np.linalg.norm(proj(h, a[None])[0] - b) > 4.0 * tol:
                os_.append(a)
                od.append(b)
        src = np.vstack([src, np.array(os_).reshape(-1, 2)])
        dst = np.vstack([dst, np.array(od).reshape(-1, 2)])
        perm = rng.permutation(len(src))
        return src[perm], dst[perm]

    persp = np.array([[0.92, 0.11, 35.0], [-0.07, 1.05, -12.0], [1.2e-4, -8e-5, 1.0]])
    cases = []
    pts = rng.uniform(50, 400, (8, 2))
    cases.append((pts, pts.copy(), 200, 3.0, 1))                                     # identity, exact
    cases.append((*scene(np.array([[1.02, 0.03, 8.0], [-0.02, 0.98, -5.0], [1e-5, -2e-5, 1.0]]), 70, 30), 1000, 3.0, 3))
    cases.append((*scene(np.array([[0.9, 0.05, 20.0], [0.02, 1.1, -8.0], [0.0, 0.0, 1.0]]), 40, 20), 500, 3.0, 5))
    cases.append((*scene(np.array([[1.0, 0.0, 12.0], [0.0, 1.0, 7.0], [0.0, 0.0, 1.0]]), 30, 30), 300, 3.0, 7))
    line = np.array([[i * 10.0, 0.0] for i in range(8)])
    cases.append((line, line.copy(), 50, 3.0, 0))                                    # collinear -> None
    tri = np.array([[i * 10.0, i * 5.0] for i in range(3)])
    cases.append((tri, tri.copy(), 1000, 3.0, 0))                                    # < 4 matches -> None
    cases.append((*scene(persp, 300, 700, noise=0.7, w=1280, hgt=720), 1000, 3.0, 11))  # 30 % inliers, noisy
    cases.append((*scene(persp, 1200, 1800, noise=0.5, w=1920, hgt=1080), 1000, 3.0, 2**33 + 1))
    cases.append((rng.uniform(0, 640, (50, 2)), rng.uniform(0, 480, (50, 2)), 200, 3.0, 4))   # all outliers
    q4 = rng.uniform(60, 500, (4, 2))
    cases.append((q4, proj(persp, q4), 10, 3.0, 2))                                  # n == 4
    dup = np.vstack([np.repeat(rng.uniform(100, 300, (1, 2)), 6, 0), rng.uniform(50, 500, (6, 2))])
    cases.append((dup, proj(persp, dup), 100, 3.0, 9))                               # coincident samples
    cases.append((*scene(persp, 20, 10), 0, 3.0, 0))                                 # iters = 0 -> None
    cases.append((*scene(persp, 150, 150, noise=0.4), 800, 1.0, 12))                # tight tolerance
    for i, (src, dst, iters, tol, seed) in enumerate(cases):
        kq = [Keypoint(float(x), float(y), 1.0) for x, y in src]
        kr = [Keypoint(float(x), float(y), 1.0) for x, y in dst]
        ms = [matching.Match(j, j, 0) for j in range(len(src))]
        h, inl = matching.ransac_homography(ms, kq, kr, iters=iters, reproj_tol=tol, seed=seed)
        out[f"r{i}_src"], out[f"r{i}_dst"] = np.asarray(src, np.float64), np.asarray(dst, np.float64)
        out[f"r{i}_par"] = np.array([iters, tol, seed], np.float64)
        out[f"r{i}_seed"] = np.array(seed, np.uint64)
        out[f"r{i}_H"] = np.full((3, 3), np.nan) if h is None else h
        out[f"r{i}_inl"] = np.array(inl, np.int64)
    out["n_ransac"] = np.array(len(cases))

    # sample tables straight from numpy (the RNG the reference seeds)
    for i, (seed, n) in enumerate([(0, 4), (0, 100), (3, 70), (2**33 + 1, 3000), (7, 2**31 - 1)]):
        r = np.random.default_rng(seed)
        out[f"s{i}_seed"], out[f"s{i}_n"] = np.array(seed, np.uint64), np.array(n)
        out[f"s{i}_tab"] = np.array([r.choice(n, 4, replace=False) for _ in range(400)], np.int32)
    out["n_samples"] = np.array(5)

    def feat(bits, x, y):
        return Feature(Keypoint(float(x), float(y), 1.0), bits.astype(np.uint8), "detected", 0)

    # match_and_verify / count_mpr on features (tests/test_matching.py:153-170 style)
    descs = rng.integers(0, 2, (60, 512)).astype(np.uint8)
    src = rng.uniform(60, 600, (60, 2))
    dst = proj(persp, src)
    dst[45:] = rng.uniform(0, 640, (15, 2))                       # 15 displaced: outliers
    noise_r = rng.integers(0, 2, (40, 512)).astype(np.uint8)
    q = [feat(d, *p) for d, p in zip(descs, src)]
    r = [feat(d, *p) for d, p in zip(np.vstack([descs, noise_r]), np.vstack([dst, rng.uniform(0, 640, (40, 2))]))]
    out["mv_q_bits"], out["mv_q_xy"] = descs, src
    out["mv_r_bits"] = np.vstack([descs, noise_r])
    out["mv_r_xy"] = np.array([[f.kp.x, f.kp.y] for f in r])
    cfg = matching.MatchConfig(t_m=102, iters=1000, reproj_tol=3.0, seed=0)
    h, ms = matching.match_and_verify(q, r, cfg)
    out["mv_H"] = h
    out["mv_matches"] = np.array([[m.query_idx, m.ref_idx, m.distance] for m in ms], np.int64).reshape(-1, 3)
    out["mv_mpr"] = np.array([matching.count_mpr(q, r, t, cfg) for t in (0, 102, 200)])
    out["mv_mpr_disjoint"] = np.array(matching.count_mpr(q[:20], [feat(b, 0, 0) for b in noise_r[:20]], 102, cfg))

    # locate_object over a 3-object database (evaluation.py:95-121)
    objs, frame = [], []
    hs = [np.array([[1.0, 0.0, 300.0], [0.0, 1.0, 120.0], [0.0, 0.0, 1.0]]), persp,
          np.array([[0.8, -0.1, 500.0], [0.1, 0.8, 300.0], [0.0, 0.0, 1.0]])]
    n_vis = [25, 0, 40]
    for oid in range(3):
        bits = rng.integers(0, 2, (50, 512)).astype(np.uint8)
        xy = rng.uniform(0, 200, (50, 2))
        objs.append((oid, bits, xy))
        k = n_vis[oid]
        if k:
            fx = proj(hs[oid], xy[:k]) + rng.normal(0.0, 0.3, (k, 2))
            frame += [feat(b, *p) for b, p in zip(bits[:k], fx)]
    fb = rng.integers(0, 2, (60, 512)).astype(np.uint8)
    frame += [feat(b, *p) for b, p in zip(fb, rng.uniform(0, 1280, (60, 2)))]
    db = [evaluation.ObjectModel(oid, [feat(b, *p) for b, p in zip(bits, xy)], evaluation.corner_geometry(200, 200))
          for oid, bits, xy in objs]
    est = evaluation.locate_object(frame, db, cfg)
    for oid, bits, xy in objs:
        out[f"lo_obj{oid}_bits"], out[f"lo_obj{oid}_xy"] = bits, xy
    out["lo_frame_bits"] = np.stack([f.desc for f in frame])
    out["lo_frame_xy"] = np.array([[f.kp.x, f.kp.y] for f in frame])
    out["lo_id"] = np.array(est.object_id)
    out["lo_corners"] = est.corners
    out["lo_mpr"] = np.array(est.mpr)

    # average precision on random ranked lists (evaluation.py:60-68)
    aps, rels, tots = [], [], []
    for _ in range(60):
        z = int(rng.integers(1, 40))
        rel = (rng.random(z) < 0.3).astype(np.int64)
        tot = int(rel.sum() + rng.integers(0, 3))
        if tot == 0:
            continue
        rels.append(np.pad(rel, (0, 40 - z), constant_values=-1))
        tots.append(tot)
        aps.append(evaluation.average_precision(evaluation.RankedList(list(range(z)), rel, tot)))
    out["ap_rel"], out["ap_tot"], out["ap_val"] = np.array(rels), np.array(tots), np.array(aps)
    np.savez_compressed(HERE / "ransac.npz", **out)
    print("ransac", [(i, int(np.isnan(out[f"r{i}_H"]).any()), len(out[f"r{i}_inl"])) for i in range(len(cases))],
          "mpr", out["mv_mpr"], "locate", int(est.object_id), int(est.mpr))


def make_divergence():
    """divergence_report (pipeline.py:348-398) on the first 6 frames of the
    reference's acceptance-c03 trend scene (test_acceptance.py:57-73: a
    textured object covering 25% of the VGA frame sweeping over a static
    textured background), threshold 40, t_i = 20; plus ast_corner_score at
    several arc lengths (detector.py:58-71) and sad_block (temporal.py:63-67)."""
    import_reference()
    from vidfeat import detector, temporal
    from vidfeat.masking import MaskConfig
    from vidfeat.pipeline import PipelineConfig, divergence_report
    from vidfeat.pyramid import GrayFrame
    from vidfeat.synth import SceneObject, SceneSpec, synth_sequence

    w, h = 640, 480
    obj = SceneObject(object_id=0, size=(w // 2, h // 2), start=(32.0, 24.0), velocity=(8.0, 0.0), texture_seed=7,
                      block=8, block_parity=True)
    scene = SceneSpec(background_seed=0, detail=60, blob_cell=16, objects=(obj,))
    frames, _ = synth_sequence(scene, 6, (w, h), seed=1)
    cfg = PipelineConfig(threshold=40, mask=MaskConfig(mode="intensity", t_i=20))
    stats = divergence_report(frames, cfg)
    out = {"frames": np.stack([f.data for f in frames]), "threshold": np.array(40), "t_i": np.array(20.0),
           "only_masked": np.array([s.only_masked for s in stats]), "only_full": np.array([s.only_full for s in stats]),
           "common": np.array([s.common for s in stats]), "preserved": np.array([s.preserved for s in stats])}
    rng = np.random.default_rng(99)
    layer = rng.integers(0, 256, (48, 64), dtype=np.uint8)
    layer[20:28, 30:38] = 250   # bright blocks give long arcs
    xs = rng.integers(3, 61, 200)
    ys = rng.integers(3, 45, 200)
    arcs = (1, 2, 5, 9, 12, 16, 20)
    out["ast_layer"], out["ast_x"], out["ast_y"], out["ast_arcs"] = layer, xs, ys, np.array(arcs)
    out["ast_scores"] = np.array([[detector.ast_corner_score(GrayFrame(layer), int(x), int(y), a) for x, y in zip(xs, ys)]
                                  for a in arcs], np.int64)
    pa = rng.integers(0, 256, (40, 16, 16), dtype=np.uint8)
    pb = rng.integers(0, 256, (40, 16, 16), dtype=np.uint8)
    out["sad_a"], out["sad_b"] = pa, pb
    out["sad"] = np.array([temporal.sad_block(a, b) for a, b in zip(pa, pb)], np.int64)
    np.savez_compressed(HERE / "divergence.npz", **out)
    print("divergence", out["common"], out["only_full"], out["only_masked"], np.round(out["preserved"], 3))


if __name__ == "__main__":
    if "--only" in sys.argv and sys.argv[sys.argv.index("--only") + 1] == "divergence":
        make_divergence()
        sys.exit(0)
    if "--only" in sys.argv and sys.argv[sys.argv.index("--only") + 1] == "formats":
        make_formats()
        sys.exit(0)
    if "--only" in sys.argv and sys.argv[sys.argv.index("--only") + 1] == "temporal":
        make_temporal()
        sys.exit(0)
    if "--only" in sys.argv and sys.argv[sys.argv.index("--only") + 1] == "ransac":
        make_ransac()
        sys.exit(0)
    if "--only" in sys.argv and sys.argv[sys.argv.index("--only") + 1] == "matching":
        make_matching()
    else:
        main()
        make_matching()
        make_temporal()
        make_formats()
        make_ransac()
        make_divergence()

"""GPU parity of the describe variants (descriptor.py:85-144,271-275).

k_desc_fused computes the orientation as a linear form of the 60 theta = 0
box means with a certified error bound against the reference's sequential
fp64 sum, and falls back to that sequential sum when the bound could move a
rotated sample across a pixel boundary or theta across the -pi / pi cut.
These tests pin: the default path, the forced fallback (VF_ORIENT_SEQ=1), and
the region-SAT describe (VF_DESC_REGION=1), each frame by frame against the
CPU oracle on BASELINE config 1 and a config-5 object stream; and that the
certified theta stays within 1e-9 of the reference's.
"""

import os

import numpy as np
import pytest

from test_gpu_pipeline import compare, oracle_frames, run_engine

pytestmark = pytest.mark.gpu


def _frames(config, n, stream=0):
    from paper_1503_06959_b200 import scenes

    return scenes.generate(scenes.CONFIGS[config], n, streams=[stream])[0].numpy()


@pytest.fixture
def env():
    saved = {}

    def set_(k, v):
        saved.setdefault(k, os.environ.get(k))
        os.environ[k] = v

    yield set_
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


@pytest.mark.parametrize("variant", ["default", "orient_seq", "region"])
@pytest.mark.parametrize("config,stream", [(1, 0), (5, 2)])
def test_describe_variants_vs_oracle(env, variant, config, stream):
    if variant == "orient_seq":
        env("VF_ORIENT_SEQ", "1")
    if variant == "region":
        env("VF_DESC_REGION", "1")
    frames = _frames(config, 6 if config == 5 else 10, stream)
    outs = run_engine(list(frames), mode="intensity")
    compare(outs, oracle_frames(frames, mode="intensity"), f"config{config}/{variant}")


def test_certified_theta_close_to_sequential():
    frames = _frames(1, 8)
    outs = run_engine(list(frames), mode="none")
    ref = oracle_frames(frames, mode="none")
    worst = 0.0
    for o, e in zip(outs, ref):
        d = np.abs(o["theta"] - e["theta"])
        worst = max(worst, float(d.max(initial=0.0)))
    assert worst <= 1e-9, worst

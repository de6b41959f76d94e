"""One profiled step of the detect+describe path for ncu (capture window =
cudaProfilerStart/Stop around step `--warmup`).

    ncu --profile-from-start off --metrics gpu__time_duration.sum,... \
        python tools/prof_step.py --config 5 --mode none --warmup 3
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1503_06959_b200 import scenes  # noqa: E402
from paper_1503_06959_b200.engine import FeatureEngine  # noqa: E402
from paper_1503_06959_b200.types import MaskConfig, PipelineConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--mode", default="intensity")
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--streams", type=int, default=0)
ap.add_argument("--gen", default="cuda")
a = ap.parse_args()
cfg = scenes.CONFIGS[a.config]
S = a.streams or cfg.n_streams
n = a.warmup + a.steps
gen = bench.gen_frames_cpu if a.gen == "cpu" else bench.gen_frames_cuda
frames = gen(cfg, list(range(S)), n, torch.device("cuda", 0))
eng = FeatureEngine(cfg.width, cfg.height, PipelineConfig(mask=MaskConfig(mode=a.mode)), n_streams=S)
for i in range(a.warmup):
    eng.process(frames[i])
torch.cuda.synchronize()
torch.cuda.profiler.start()
for i in range(a.warmup, n):
    eng.process(frames[i])
torch.cuda.synchronize()
torch.cuda.profiler.stop()
r = eng.report(0)
print("frame", r.frame, "n_total", r.n_total, "n_detected", r.n_detected, "coverage", r.coverage)
eng.close()

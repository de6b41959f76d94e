"""Per-call host and device time of ransac_homography_device (diagnostics)."""
import time

import numpy as np
import torch

from paper_1503_06959_b200.matching import ransac_homography_device

rng = np.random.default_rng(0)
P, n = 64, 4096
src = torch.from_numpy(rng.uniform(0, 1900, (P * n, 2))).cuda()
dst = (src + 3.0).contiguous()
off = np.arange(P + 1, dtype=np.int64) * n
for _ in range(3):
    ransac_homography_device(src, dst, off)
torch.cuda.synchronize()
for k in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(10):
        ransac_homography_device(src, dst, off)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host enqueue {1e3 * (t1 - t0) / 10:.3f} ms/call, device {e0.elapsed_time(e1) / 10:.3f} ms/call, "
          f"wall {1e3 * (t2 - t0) / 10:.3f} ms/call")

import sys  # noqa: E402

sys.path.insert(0, ".")
from bench import ClockSampler  # noqa: E402

with ClockSampler(0) as clk:
    time.sleep(1.0)
    for k in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(10):
            ransac_homography_device(src, dst, off)
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        print(f"[sampler on] host enqueue {1e3 * (t1 - t0) / 10:.3f} ms/call, device {e0.elapsed_time(e1) / 10:.3f}")

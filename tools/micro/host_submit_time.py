"""Host-side cost of one step through the C-ABI: vf_process with the same / alternating frame
pointers (graph replay re-points kernel-node arguments when the pointer changes) and the pipelined
submit + collect_delta pair.   python tools/micro/host_submit_time.py [config]"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_1503_06959_b200 import scenes  # noqa: E402
from paper_1503_06959_b200.engine import FeatureEngine  # noqa: E402
from paper_1503_06959_b200.types import MaskConfig, PipelineConfig  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = scenes.CONFIGS[cid]
S = min(cfg.n_streams, 8)
fr = scenes.generate(cfg, 12, streams=range(S), device="cuda").permute(1, 0, 2, 3).contiguous()
eng = FeatureEngine(cfg.width, cfg.height, PipelineConfig(mask=MaskConfig(mode="intensity")), n_streams=S)
for n in range(4):
    eng.process(fr[n])
torch.cuda.synchronize()
for label, idx in (("same pointer", [4] * 200), ("alternating pointers", [4, 5] * 100)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in idx:
        eng.process(fr[i])
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"config {cid} {label}: host enqueue {1e6 * (t1 - t0) / len(idx):.1f} us/step, "
          f"with the GPU {1e6 * (t2 - t0) / len(idx):.1f} us/step")
host = fr.cpu().pin_memory()
out = eng.alloc_delta(S * max(65536, cfg.width * cfg.height // 8))
eng.set_delta(True)
eng.submit(host[0].numpy())
eng.collect_delta(out)
ts, tc = 0.0, 0.0
t0 = time.perf_counter()
eng.submit(host[1].numpy())
for n in range(1, 11):
    a = time.perf_counter()
    if n + 1 < 12:
        eng.submit(host[n + 1].numpy())
    b = time.perf_counter()
    eng.collect_delta(out)
    c = time.perf_counter()
    ts += b - a
    tc += c - b
print(f"config {cid} pipelined: {1e6 * (time.perf_counter() - t0) / 10:.1f} us/step; submit {1e5 * ts:.1f} us, "
      f"collect_delta {1e5 * tc:.1f} us (host time per call)")
eng.close()

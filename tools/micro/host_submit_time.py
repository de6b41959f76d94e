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
cap = S * max(65536, cfg.width * cfg.height // 8)
for delta in (True, False, True):
    out = eng.alloc_delta(cap) if delta else eng.alloc_host(cap)
    collect = eng.collect_delta if delta else eng.collect
    eng.set_delta(delta)
    for n in range(3):
        eng.submit(host[n].numpy())
        collect(out)
    N = 40
    ts, tc, per = 0.0, 0.0, []
    t0 = time.perf_counter()
    eng.submit(host[3 % 12].numpy())
    eng.submit(host[4 % 12].numpy())
    for n in range(N):
        a = time.perf_counter()
        if n + 2 < N:
            eng.submit(host[(n + 5) % 12].numpy())
        b = time.perf_counter()
        collect(out)
        c = time.perf_counter()
        ts += b - a
        tc += c - b
        per.append(1e6 * (c - a))
    per_s = sorted(per)
    print(f"config {cid} pipelined {'delta' if delta else 'full'}: {1e6 * (time.perf_counter() - t0) / N:.1f} us/step; "
          f"submit {1e6 * ts / N:.1f} us, collect {1e6 * tc / N:.1f} us per call; per-step p10 {per_s[N // 10]:.0f} "
          f"p50 {per_s[N // 2]:.0f} p90 {per_s[9 * N // 10]:.0f} us")
eng.close()

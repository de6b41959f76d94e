"""D2H / H2D bandwidth of pinned copies with 1, 2 and 4 concurrent CUDA streams (and both directions at once)."""
import torch

n = 256 << 20
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
dev2 = torch.empty(n, dtype=torch.uint8, device="cuda")
host = torch.empty(n, dtype=torch.uint8).pin_memory()
host2 = torch.empty(n, dtype=torch.uint8).pin_memory()


def run(k, d2h=True, h2d=False, reps=5):
    streams = [torch.cuda.Stream() for _ in range(2 * k)]
    chunk = n // k
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        for i in range(k):
            if d2h:
                with torch.cuda.stream(streams[i]):
                    host[i * chunk:(i + 1) * chunk].copy_(dev[i * chunk:(i + 1) * chunk], non_blocking=True)
            if h2d:
                with torch.cuda.stream(streams[k + i]):
                    dev2[i * chunk:(i + 1) * chunk].copy_(host2[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return n / ms / 1e6


for k in (1, 2, 4):
    print(f"streams {k}: D2H {run(k):.1f} GB/s  H2D {run(k, False, True):.1f} GB/s  both (each) {run(k, True, True):.1f} GB/s")

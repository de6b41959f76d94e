"""Per-pair timing of the Hamming kernels on random rows and on engine descriptors (A/B of the MMA and POPC paths)."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_1503_06959_b200.matching import hamming_matrix_device, radius_match_device  # noqa: E402


def timeit(fn, n=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


tag = os.environ.get("VF_MATCH_POPC", "0")
torch.manual_seed(0)
a = torch.randint(0, 256, (20000, 64), dtype=torch.uint8, device="cuda")
b = torch.randint(0, 256, (20000, 64), dtype=torch.uint8, device="cuda")
print(tag, "random matrix", timeit(lambda: hamming_matrix_device(a, b)), "radius", timeit(lambda: radius_match_device(a, b, 102)))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import bench  # noqa: E402

pairs = bench.match_descriptors(2, torch.device("cuda", 0))
for qa, rb in pairs:
    print(tag, "engine", tuple(qa.shape), tuple(rb.shape), qa.is_contiguous(), qa.data_ptr() % 16,
          "matrix", timeit(lambda: hamming_matrix_device(qa, rb)), "radius", timeit(lambda: radius_match_device(qa, rb, 102)))

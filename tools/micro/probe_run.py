import torch, sys
sys.path.insert(0, '.')
from paper_1503_06959_b200.matching import radius_match_device
torch.manual_seed(0)
a = torch.randint(0, 256, (19745, 64), dtype=torch.uint8, device="cuda")
b = torch.randint(0, 256, (19745, 64), dtype=torch.uint8, device="cuda")
radius_match_device(a, b, 102); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); qi, ri, d = radius_match_device(a, b, 102); e1.record(); torch.cuda.synchronize()
print("ms", e0.elapsed_time(e1), "matches", qi.numel())

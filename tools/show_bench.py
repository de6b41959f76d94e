"""Print value and per-kernel live times of a bench JSON log."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(round(d["value"]), "frames/s", round(d["ms_per_step"] * 1000, 1), "us/step")
for k in d["roofline"]["kernels"]:
    print(f"  {k['kernel']:10s} {k['ms_per_step'] * 1000:7.1f} us")

"""Print the headline numbers and per-kernel live times of bench JSON logs."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "unreadable:", e)
        continue
    if "value" not in d:
        print(path, d)
        continue
    r = d.get("roofline") or {}
    e2e = d.get("e2e") or {}
    cfg = d.get("config", {})
    print(f"{path}: {cfg.get('config', '?')}/{cfg.get('mode', '?')} {d['value']:.0f} frames/s "
          f"{d['ms_per_step'] * 1000:.1f} us/step  frac {r.get('frac', 0):.3f}  e2e {e2e.get('value', 0):.0f}  "
          f"feat/frame {d.get('features_per_frame', 0):.0f} det {d.get('detected_per_frame', 0):.0f} "
          f"cov {d.get('mean_coverage', 0):.3f}")
    for k in r.get("kernels", []):
        print(f"    {k['kernel']:13s} {k['ms_per_step'] * 1000:8.1f} us  frac {k['frac']:.3f}")

"""ncu launch list (tools/prof_all.sh CSV) of one step -> profiles JSON with
the step's DRAM traffic (sum of dram__bytes_read + dram__bytes_write over its
launches) and per-kernel rows.   python tools/traffic_json.py CSV STREAMS OUT"""
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_lines import load  # noqa: E402

csv_path, streams, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
L = load(csv_path)
rows = []
for i in sorted(L):
    d = L[i]
    rows.append({"id": i, "kernel": d["kernel"], "us": d.get("gpu__time_duration.sum"),
                 "dram_read_mb": d.get("dram__bytes_read.sum"), "dram_write_mb": d.get("dram__bytes_write.sum"),
                 "sm_pct": d.get("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                 "warp_inst_m": d.get("smsp__inst_executed.sum"),
                 "l2_hit_pct": d.get("lts__t_sector_hit_rate.pct"),
                 "warps_active_pct": d.get("sm__warps_active.avg.pct_of_peak_sustained_active")})
tot = sum((r["dram_read_mb"] or 0) + (r["dram_write_mb"] or 0) for r in rows) * 1e6
json.dump({"source": csv_path.split("/")[-1], "streams": streams,
           "how": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,... "
                  "--clock-control none, one step (tools/prof_step.py: 3 warm-up steps, eager launches); "
                  "serialized cold-cache replays: compare shares, not absolute times",
           "dram_bytes_per_step": tot, "us_per_step_serialized": sum(r["us"] or 0 for r in rows),
           "kernels": rows}, open(out, "w"), indent=1)
print(out, round(tot / 1e6, 1), "MB")

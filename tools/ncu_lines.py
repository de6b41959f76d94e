"""Pivot an ncu --metrics --csv launch list into one line per launch.

    python tools/ncu_lines.py FILE.csv [--md]
Columns: id, kernel, us, DRAM read MB, DRAM write MB, SM thr %, warp inst (M), L2 hit %, warps active %."""
import csv
import sys

COLS = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "rd MB"), ("dram__bytes_write.sum", "wr MB"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"), ("smsp__inst_executed.sum", "Minst"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps %")]
SCALE = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "%": 1.0,
         "inst": 1e-6, "": 1.0}


def load(path):
    rows = list(csv.reader(open(path)))
    h, launches = None, {}
    for r in rows:
        if r and r[0] == "ID":
            h = r
            continue
        if not h or len(r) != len(h):
            continue
        i = int(r[h.index("ID")])
        d = launches.setdefault(i, {"kernel": r[h.index("Kernel Name")].split("(")[0]})
        name, unit = r[h.index("Metric Name")], r[h.index("Metric Unit")]
        try:
            v = float(r[h.index("Metric Value")].replace(",", ""))
        except ValueError:
            continue
        d[name] = v * SCALE.get(unit, 1.0)
    return launches


if __name__ == "__main__":
    L = load(sys.argv[1])
    md = "--md" in sys.argv
    hdr = ["id", "kernel"] + [c[1] for c in COLS]
    print(("| " + " | ".join(hdr) + " |") if md else "  ".join(hdr))
    if md:
        print("|" + "---|" * len(hdr))
    tot = 0.0
    for i in sorted(L):
        d = L[i]
        vals = [f"{d.get(m, float('nan')):.1f}" for m, _ in COLS]
        tot += d.get("gpu__time_duration.sum", 0.0)
        print(("| " + " | ".join([str(i), d["kernel"]] + vals) + " |") if md else f"{i:3d} {d['kernel']:16s} " + " ".join(f"{v:>8s}" for v in vals))
    print(f"total us {tot:.1f}")

"""Per-CUDA-line summary of an ncu report's source page (cuda,sass view):
instructions executed and warp-stall samples aggregated per source line.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [TOP]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg = {}
    fname = "?"
    hdr = None
    tot_i = tot_s = 0
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if len(r) > 3 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) - 1:
            continue
        if r[0]:   # a CUDA line row carries the line's aggregate
            try:
                ins = int(r[hdr.index("Instructions Executed")])
                smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            except (ValueError, IndexError):
                continue
            key = (fname, int(r[0]))
            a = agg.setdefault(key, [0, 0, r[1].strip()[:90]])
            a[0] += ins
            a[1] += smp
            tot_i += ins
            tot_s += smp
    print(f"total warp-instructions {tot_i:,}  stall samples {tot_s:,}")
    for (f, ln), (ins, smp, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{f}:{ln:5d}  inst {100.0 * ins / max(tot_i, 1):5.1f}%  samp {100.0 * smp / max(tot_s, 1):5.1f}%  {src}")


if __name__ == "__main__":
    main()

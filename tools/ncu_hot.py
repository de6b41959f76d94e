"""Top CUDA source lines of one kernel in an ncu report by warp-stall samples
and executed instructions.   python tools/ncu_hot.py REP KERNEL [TOP]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern, "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
path, hdr, lines = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] not in ("", "Function Name") and len(r) == len(hdr):
        try:
            samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            inst = int(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        lines.append((samp, inst, f"{path}:{r[0]}", r[1].strip()[:110]))
ts = sum(x[0] for x in lines) or 1
ti = sum(x[1] for x in lines) or 1
print(f"total samples {ts}, warp instructions {ti}")
for s_, i_, loc, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * s_ / ts:5.1f}% smp {100 * i_ / ti:5.1f}% inst  {loc:22s} {src}")

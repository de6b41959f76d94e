"""One markdown card per kernel from `ncu --set full` reports: SOL, occupancy,
memory, the dominant stall reasons and the top source lines.

    python tools/ncu_card.py OUT.md [--title=TEXT] REP.ncu-rep[:kernel] ...
"""
import csv
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active",
        "Issue Slots Busy", "Executed Instructions", "Registers Per Thread", "Theoretical Occupancy",
        "Achieved Active Warps Per SM", "Avg. Active Threads Per Warp", "Warp Cycles Per Issued Instruction"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    got = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") in KEYS and d["Metric Name"] not in got:
            got[d["Metric Name"]] = (d["Metric Value"], d.get("Metric Unit", ""))
    return got


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
    res = []
    for k, x in zip(h, v):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                res.append((float(x), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    return sorted(res, reverse=True)[:6]


def hot(rep, kern, top=8):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern, "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
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
        if hdr and len(r) == len(hdr) and r[0].isdigit():
            try:
                smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
                ins = int(r[hdr.index("Instructions Executed")] or 0)
            except ValueError:
                continue
            lines.append((smp, ins, f"{path}:{r[0]}", r[1].strip()[:80]))
    ts = sum(x[0] for x in lines) or 1
    ti = sum(x[1] for x in lines) or 1
    return [(100 * a / ts, 100 * b / ti, c, d) for a, b, c, d in sorted(lines, reverse=True)[:top]]


if __name__ == "__main__":
    title = "config 5, intensity"
    args = []
    for a in sys.argv[2:]:
        if a.startswith("--title="):
            title = a[len("--title="):]
        else:
            args.append(a)
    out = [f"# ncu --set full cards ({title}, one step after 3 warm-up steps; serialized replay)\n"]
    for arg in args:
        rep, _, kern = arg.partition(":")
        kern = kern or rep.rsplit("_", 1)[-1].replace(".ncu-rep", "")
        out.append(f"## {kern}\n")
        out.append("| metric | value |\n|---|---|")
        for k, (v, u) in details(rep).items():
            out.append(f"| {k} | {v} {u} |")
        out.append("\nTop stall reasons (warps per issued instruction): " +
                   ", ".join(f"{n} {x:.2f}" for x, n in stalls(rep)) + "\n")
        out.append("| stall % | inst % | line | source |\n|---|---|---|---|")
        for s, i, loc, src in hot(rep, kern):
            out.append(f"| {s:.1f} | {i:.1f} | {loc} | `{src.replace('|', '/')}` |")
        out.append("")
    open(sys.argv[1], "w").write("\n".join(out) + "\n")
    print(sys.argv[1])

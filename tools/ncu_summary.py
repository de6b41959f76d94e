"""Summarise an ncu report (.ncu-rep) into markdown for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN_kernels.md
    python tools/ncu_summary.py --launches gpurun_out/launches.csv > profiles/rNN_launches.md
"""
import collections
import csv
import subprocess
import sys

METRICS = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
           "Theoretical Occupancy", "Registers Per Thread", "L1/TEX Hit Rate", "L2 Hit Rate",
           "Executed Ipc Active", "Grid Size", "Block Size")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout


def details(rep):
    rows = list(csv.reader(ncu(rep, "--page", "details").splitlines()))
    h = rows[0]
    ki, ii, mi, vi, ui = (h.index(c) for c in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    out = collections.OrderedDict()
    for r in rows[1:]:
        key = (r[ii], r[ki].split("(")[0])
        if r[mi] in METRICS:
            out.setdefault(key, {})[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    return out


def raw(rep):
    rows = list(csv.reader(ncu(rep, "--page", "raw").splitlines()))
    h = rows[0]
    cols = {c: h.index(c) for c in RAW if c in h}
    units = rows[1]
    out = {}
    for r in rows[2:]:
        out[(r[h.index("ID")], r[h.index("Kernel Name")].split("(")[0])] = {
            c: f"{r[i]} {units[i]}" for c, i in cols.items()}
    return out


def stalls(rep, kern):
    rows = list(csv.reader(ncu(rep, "--page", "source", "-k", "regex:" + kern).splitlines()))
    try:
        hi = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
    except StopIteration:
        return ""
    h = rows[hi]
    data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0].startswith("0x")]
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    agg = collections.Counter()
    for r in data:
        for c in reasons:
            try:
                agg[c] += float(r[h.index(c)])
            except ValueError:
                pass
    tot = sum(agg.values()) or 1
    return ", ".join(f"{c[6:]} {v / tot * 100:.0f}%" for c, v in agg.most_common(4))


def main():
    if sys.argv[1] == "--launches":
        rows = list(csv.reader(open(sys.argv[2])))
        hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hi]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        agg = collections.defaultdict(list)
        for r in rows[hi + 1:]:
            agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
        ours = {k: v for k, v in agg.items() if k.startswith("k_")}
        tot = sum(sum(v) for v in ours.values())
        print("| kernel | launches | mean us | share of our kernels |\n|---|---|---|---|")
        for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
            print(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot * 100:.1f}% |")
        return
    rep = sys.argv[1]
    d, r = details(rep), raw(rep)
    print("| id | kernel | duration | DRAM read | DRAM write | DRAM thr | SM thr | IPC | occupancy (ach/theo) | regs | L2 hit | top stalls |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    seen = set()
    for key, m in d.items():
        rr = r.get(key, {})
        st = stalls(rep, key[1]) if key[1] not in seen else ""
        seen.add(key[1])
        print(f"| {key[0]} | {key[1]} | {m.get('Duration', '')} | {rr.get('dram__bytes_read.sum', '')} | "
              f"{rr.get('dram__bytes_write.sum', '')} | {m.get('DRAM Throughput', '')} | "
              f"{m.get('Compute (SM) Throughput', '')} | {m.get('Executed Ipc Active', '')} | "
              f"{m.get('Achieved Occupancy', '')} / {m.get('Theoretical Occupancy', '')} | "
              f"{m.get('Registers Per Thread', '')} | {m.get('L2 Hit Rate', '')} | {st} |")


if __name__ == "__main__":
    main()

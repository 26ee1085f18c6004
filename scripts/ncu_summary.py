"""Summarise an ncu report (--set full) or a launch-list CSV into a small markdown table.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/<name>.md
    python scripts/ncu_summary.py --launches gpurun_out/launches.csv > profiles/<name>.md
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    print(f"ncu --set full summary of `{path}` (one row per profiled launch)\n")
    cols = [m for m in METRICS if m[0] in idx]
    print("| kernel | " + " | ".join(f"{n} ({units[idx[m]]})" for m, n in cols) + " |")
    print("|---|" + "---|" * len(cols))
    for r in data:
        name = r[idx["Kernel Name"]].split("(")[0][-48:]
        print(f"| {name} | " + " | ".join(r[idx[m]] for m, _ in cols) + " |")


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] in ("ns", "nsecond") else (v * 1e3 if r[ui] in ("ms", "msecond") else v)
        agg[r[ki].split("(")[0][-60:]].append(v)
    tot = sum(sum(v) for v in agg.values())
    print(f"ncu launch list `{path}` (gpu__time_duration, serialised / cold cache: compare shares)\n")
    print("| kernel | launches | mean us | total us | share |")
    print("|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.0f} | {sum(v) / tot:.1%} |")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[1])

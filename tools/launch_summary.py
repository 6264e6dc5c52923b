"""Aggregate an ncu --csv launch list (gpu__time_duration + DRAM bytes per launch) per kernel.

Usage: python tools/launch_summary.py launches.csv [header text...]
ncu replays each launch cold and serialised: compare SHARES of the step, not absolutes.
"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = defaultdict(dict)
    for r in rows[1:]:
        per[(r[ii], r[ki])][r[mi]] = float(r[vi].replace(",", ""))
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for (_, name), m in per.items():
        short = name.split("(")[0] if "cheb_" not in name else name.split("(unnamed")[0].split("(adp")[0]
        a = agg[short]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0) / 1e6  # ns -> ms
        a[2] += (m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)) / 1e9
    total = sum(a[1] for a in agg.values())
    for line in sys.argv[2:]:
        print(line)
    print(f"{'kernel':<96} {'launches':>8} {'total ms':>10} {'share':>7} {'ms/launch':>10} {'DRAM GB/launch':>15}")
    for name, (n, ms, gb) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:96]:<96} {n:>8} {ms:>10.3f} {100 * ms / total:>6.1f}% {ms / n:>10.4f} {gb / n:>15.3f}")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

  python tools/launch_summary.py gpurun_out/launches.csv
"""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            break
    hdr, data = rows[i], rows[i + 1:]
    ki, mi, ni = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= mi or r[ni] != "gpu__time_duration.sum":
            continue
        k = r[ki].split("(")[0].replace("void ", "")
        agg[k][0] += 1
        agg[k][1] += float(r[mi].replace(",", ""))
    tot = sum(v[1] for v in agg.values()) or 1.0
    lines = ["| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {c} | {t / 1e3:.1f} | {t / c / 1e3:.1f} | {100 * t / tot:.1f}% |")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))

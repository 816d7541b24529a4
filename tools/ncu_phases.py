#!/usr/bin/env python
"""Aggregate ncu stall samples / executed instructions of k_raster or k_backward by code
region ('// phase X' markers in csrc/kernels.cuh; helpers above the kernel count as 'helpers').

  python tools/ncu_phases.py gpurun_out/prof.ncu-rep k_raster
"""
import collections
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", f"regex:{kern}", "--launch-count", "1"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, res = None, []
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if not r or not r[0] or r[0] == "Line No":
            continue
        try:
            res.append((fname, int(r[0]), float(r[4] or 0), float(r[7] or 0)))
        except (ValueError, IndexError):
            pass
    src = open(os.path.join(ROOT, "paper_2401_06003_b200", "csrc", "kernels.cuh")).read().split("\n")
    start = next(i for i, l in enumerate(src) if f" {kern}(" in l and "__global__" in l) + 1
    marks = [("setup", start)]
    for i, l in enumerate(src[start:], start + 1):
        if l.strip().startswith("// phase"):
            marks.append((l.strip()[3:10].strip(), i))
        if i > start and l.startswith("// ----"):
            marks.append(("after", i))
            break
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    for f, line, s, n in res:
        key = "helpers/" + (f or "?")
        if f == "kernels.cuh":
            key = "helpers(kernels.cuh)"
            for (nm, a), (_, b) in zip(marks, marks[1:]):
                if a <= line < b:
                    key = nm
        agg[key][0] += s
        agg[key][1] += n
    tot_s = sum(v[0] for v in agg.values()) or 1
    tot_n = sum(v[1] for v in agg.values()) or 1
    for k, (s, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{k:28s} stall {100 * s / tot_s:5.1f}%   inst {100 * n / tot_n:5.1f}% ({n / 1e6:.1f}M warp-inst)")


if __name__ == "__main__":
    main()

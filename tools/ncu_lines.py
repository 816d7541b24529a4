#!/usr/bin/env python
"""Aggregate ncu warp-stall samples per CUDA source line.

  python tools/ncu_lines.py gpurun_out/prof.ncu-rep k_raster [top] [launch]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    skip = sys.argv[4] if len(sys.argv) > 4 else "0"
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname = None
    res = []
    hdr = None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or not r[0]:
            continue
        try:
            samples = float(r[4] or 0)
            inst = float(r[7] or 0)
        except (ValueError, IndexError):
            continue
        res.append((samples, inst, f"{fname}:{r[0]}", r[1].strip()[:100]))
    tot = sum(s for s, _, _, _ in res) or 1
    print(f"total stall samples {tot:.0f}")
    for s, inst, loc, src in sorted(res, key=lambda x: -x[0])[:top]:
        print(f"{100 * s / tot:5.1f}%  inst {inst:12.0f}  {loc:18s} {src}")


if __name__ == "__main__":
    main()

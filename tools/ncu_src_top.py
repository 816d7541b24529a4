#!/usr/bin/env python
"""Top source lines (CUDA) of an exported ncu source page (--page source --csv --print-source
cuda,sass; .csv or .csv.gz) by warp-stall samples, with executed instructions and top stalls.

  python tools/ncu_src_top.py profiles/r02/r02_knn_src.csv.gz [N]
"""
import csv
import gzip
import io
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, res = None, []
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not r or not r[0] or hdr is None:
            continue
        try:
            d = dict(zip(hdr, r))
            stalls = {k[6:]: float(d[k] or 0) for k in hdr if k.startswith("stall_") and "(Not" not in k}
            res.append((int(r[0]), r[1][:100], float(d["Warp Stall Sampling (All Samples)"] or 0),
                        float(d["Instructions Executed"] or 0), stalls))
        except (ValueError, KeyError):
            pass
    tot = sum(x[2] for x in res) or 1
    toti = sum(x[3] for x in res) or 1
    for line, src, st, n, stalls in sorted(res, key=lambda x: -x[2])[:top]:
        s3 = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
        print(f"{line:5d} stall {100 * st / tot:5.1f}%  inst {100 * n / toti:5.1f}%  "
              f"{' '.join(f'{k}:{int(v)}' for k, v in s3):40s} {src.strip()}")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""ncu CSV launch lists (one per config, from tools/traffic_views.py) -> per-kernel DRAM bytes
per launch (mean over the captured launches), written as profiles/dram_traffic_r02.json.

  python tools/traffic_json.py out.json C4=gpurun_out/traffic_C4.csv C2=... ...
"""
import collections
import csv
import json
import re
import sys


def parse(path):
    acc = collections.defaultdict(lambda: collections.defaultdict(list))
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    h = rows[hdr]
    iK, iM, iU, iV, iID = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
    per = collections.defaultdict(dict)
    for r in rows[hdr + 1:]:
        name = re.sub(r"^(void )?(trips::)?", "", r[iK]).split("<")[0].split("(")[0]
        per[(r[iID], name)][r[iM]] = float(r[iV].replace(",", "")) * scale.get(r[iU], 1)
    for (_, name), m in per.items():
        acc[name]["dram"].append(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0))
        acc[name]["us"].append(m.get("gpu__time_duration.sum", 0) * 1e6)
    return {k: sum(v["dram"]) / len(v["dram"]) for k, v in acc.items()}, \
        {k: sum(v["us"]) / len(v["us"]) for k, v in acc.items()}


if __name__ == "__main__":
    out = {"_note": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch (mean of the captured launches "
                    "after warm-up; --clock-control none), tools/traffic_views.py + tools/traffic_json.py",
           "_us_per_launch": {}}
    for spec in sys.argv[2:]:
        cfg, path = spec.split("=", 1)
        out[cfg], out["_us_per_launch"][cfg] = parse(path)
    json.dump(out, open(sys.argv[1], "w"), indent=1, sort_keys=True)
    print(json.dumps(out, indent=1, sort_keys=True))

#!/usr/bin/env python
"""Reduction / atomic / scatter ceilings of this B200 (trips_microbench): ops/s and 16-B-op/s for
random-address red.global.add.v4.f32, red.global.add.f32, atomicAdd u32, st.v4 and ld.v4 on an
L2-resident (32 MB) and a DRAM-sized (2 GB) array, rows of 16 and 48 bytes, independent-lane and
warp-coherent address patterns.  Prints one JSON object.

  python tools/microbench.py [--ops 268435456]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06003_b200 import _abi as A  # noqa: E402


def measure(ops=1 << 28, sizes=(("l2", 32 << 20), ("dram", 2 << 30)), rows=(16, 48), patterns=(0, 1),
            names=("red_v4_f32", "red_f32", "atomic_add_u32", "store_v4", "load_v4"), reps=3):
    dev = torch.device("cuda", torch.cuda.current_device())
    out = {}
    big = max(b for _, b in sizes)
    buf = torch.zeros(big // 4, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    for sname, nbytes in sizes:
        for rb in rows:
            for pat in patterns:
                for name in names:
                    op = A.MB_OPS[name]
                    A.trips_microbench(op, pat, buf.data_ptr(), nbytes, rb, ops // 8, st)      # warm-up
                    best = None
                    for _ in range(reps):
                        ms, done = A.trips_microbench(op, pat, buf.data_ptr(), nbytes, rb, ops, st)
                        best = ms if best is None else min(best, ms)
                    out[f"{name}|{sname}|row{rb}|{'random' if pat == 0 else 'coherent'}"] = {
                        "G_ops_per_s": done / (best * 1e-3) / 1e9, "ms": best, "ops": done}
    del buf
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", type=int, default=1 << 28)
    args = ap.parse_args()
    res = measure(args.ops)
    for k, v in res.items():
        print(f"{k:48s} {v['G_ops_per_s']:8.1f} G/s", file=sys.stderr)
    print(json.dumps(res))

"""Builds libtrips.so (the C-ABI library) in-tree with nvcc for sm_100a.

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.

  python paper_2401_06003_b200/build.py                       # in-tree libtrips.so
  python paper_2401_06003_b200/build.py --out X.so -DFLAG     # experiment variant
"""
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtrips.so")
SOURCES = [os.path.join(CSRC, "trips_api.cu")]
NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "--expt-relaxed-constexpr",
              "-fmad=true", "-ftz=false", "-prec-div=true", "-prec-sqrt=true"]


def deps():
    return (glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
            + [os.path.join(ROOT, "include", "trips.h"), os.path.abspath(__file__)])


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    return "nvcc"


def build(force=False, verbose=False, out=None, extra=()):
    out = out or LIB
    if not force and not extra and os.path.exists(out) and os.path.getmtime(out) >= max(
            os.path.getmtime(d) for d in deps()):
        return out
    tmp = out + f".tmp{os.getpid()}"
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), *SOURCES, "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libtrips.so")
    if verbose:
        sys.stderr.write(res.stderr)
    if out == LIB:
        with open(os.path.join(CSRC, "ptxas_info.txt"), "w") as f:
            # registers / spills / shared memory per kernel; compile times dropped (not reproducible)
            f.write("".join(l for l in res.stderr.splitlines(True) if "Compile time" not in l))
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    out = None
    if "--out" in args:
        k = args.index("--out")
        out = args[k + 1]
        del args[k:k + 2]
    extra = [a for a in args if a.startswith("-D")]
    print(build(force=True, verbose="-v" in args, out=out, extra=extra))

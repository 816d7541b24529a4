"""Builds the C oracle twice: real=float (parity reference) and real=double (FD pins).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Flags pin IEEE behaviour:
no FMA contraction, no fast-math, SSE arithmetic (x86-64 default).
"""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "trips_oracle.c")
LIBS = {"float": os.path.join(HERE, "liboracle_f32.so"), "double": os.path.join(HERE, "liboracle_f64.so")}
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fno-finite-math-only",
          "-fPIC", "-shared", "-Wall", "-Wno-unused-function"]


def build(force: bool = False) -> dict:
    for real, out in LIBS.items():
        if (not force and os.path.exists(out)
                and os.path.getmtime(out) >= os.path.getmtime(SRC)):
            continue
        tmp = out + f".tmp{os.getpid()}"
        cmd = ["gcc", *CFLAGS, f"-DORACLE_REAL={real}", SRC, "-o", tmp, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, out)
    return dict(LIBS)


if __name__ == "__main__":
    print(build(force=True))

"""The C ABI used from plain C (tests/c/abi_parity.c): include/trips.h compiles as C11 and the
program links against libtrips.so (CPU); on a GPU it runs project -> forward -> backward on a
seeded scene with cudaMalloc'd buffers and checks counts and kept lists bit-exact, features and
gradients within the SURVEY.md 8(c) tolerances against the C oracle (gpu)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(tmp_path):
    from oracle import build as oracle_build
    from paper_2401_06003_b200 import _abi
    _abi.lib()                                                   # builds libtrips.so if missing
    oracle_build.build()
    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    lib_dir = os.path.join(ROOT, "paper_2401_06003_b200")
    ora_dir = os.path.join(ROOT, "oracle")
    exe = str(tmp_path / "abi_parity")
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), os.path.join(ROOT, "tests", "c", "abi_parity.c"), "-o", exe,
           "-L", lib_dir, "-ltrips", "-L", ora_dir, "-loracle_f32", "-L", os.path.join(CUDA, "lib64"), "-lcudart",
           "-lm", f"-Wl,-rpath,{lib_dir}:{ora_dir}:{os.path.join(CUDA, 'lib64')}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_program_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_program_parity_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bad counts 0, kept 0, features 0, grads 0" in r.stdout, r.stdout

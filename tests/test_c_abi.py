"""The C ABI from plain C (tests/c/abi_smoke.c): the header compiles as C11
with -Wall -Wextra -Werror (CPU suite); on the GPU the program links against
libgespmm.so + cudart and runs the host entry, the device COO builder, an
overlap_prev plan and the workspace release, bit-exact against a naive loop."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c", "abi_smoke.c")
CUDA = "/usr/local/cuda"
FLAGS = ["-std=c11", "-Wall", "-Wextra", "-Werror", "-ffp-contract=off", "-O2",
         "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include")]


def test_header_is_clean_c11(tmp_path):
    out = subprocess.run(["gcc"] + FLAGS + ["-c", SRC, "-o", str(tmp_path / "abi.o")],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr


@pytest.mark.gpu
def test_c_program_runs_on_the_gpu(tmp_path):
    lib_dir = os.path.join(ROOT, "paper_2007_03179_b200")
    exe = str(tmp_path / "abi_smoke")
    out = subprocess.run(["gcc"] + FLAGS + [SRC, "-o", exe, "-L", lib_dir, "-lgespmm",
                          "-L", os.path.join(CUDA, "lib64"), "-lcudart",
                          f"-Wl,-rpath,{lib_dir}", f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}"],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    run = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "abi_smoke: ok" in run.stdout

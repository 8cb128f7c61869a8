"""The C++ drop-in (include/gespmm/native_spmm.hpp): build the reference-style
test program against libgespmm.so here (CPU: compile + link check), run it on
the GPU (gpu marker)."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
OUT = os.path.join(ROOT, "build", "test_dropin")


def _build():
    from paper_2007_03179_b200 import _lib
    _lib.lib()  # ensures libgespmm.so exists
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           SRC, "-L", os.path.dirname(_lib.LIB_PATH), "-lgespmm",
           f"-Wl,-rpath,{os.path.dirname(_lib.LIB_PATH)}", "-o", OUT]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return OUT


def test_dropin_compiles_and_links():
    exe = _build()
    assert os.path.exists(exe)
    nm = subprocess.run(["nm", "-u", exe], capture_output=True, text=True).stdout
    assert "gespmm_spmm_host" in nm


@pytest.mark.gpu
def test_dropin_reference_cases_on_gpu(cuda):
    exe = _build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout

"""The C++ drop-in (include/gespmm/native_spmm.hpp): build the reference-style
test programs against libgespmm.so here (CPU: compile + link check), run them
on the GPU (gpu marker).

* tests/cpp/test_dropin.cpp — the reference's test cases as a drop-in user's
  program (errors, arg indices, fault hook, bench);
* tests/cpp/test_reference_api.cpp — the reference README's library use and
  the cases of test_kernels.cpp / test_native.cpp / test_csr / test_io, with
  the reference's names (from_coo, validate, KernelConfig, load_matrix, ...)."""
import os
import subprocess

import pytest

from conftest import ROOT

PROGRAMS = ["test_dropin", "test_reference_api"]


def _build(name):
    from paper_2007_03179_b200 import _lib
    _lib.lib()  # ensures libgespmm.so exists
    src = os.path.join(ROOT, "tests", "cpp", name + ".cpp")
    out = os.path.join(ROOT, "build", name)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           src, "-L", os.path.dirname(_lib.LIB_PATH), "-lgespmm",
           f"-Wl,-rpath,{os.path.dirname(_lib.LIB_PATH)}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


@pytest.mark.parametrize("name", PROGRAMS)
def test_dropin_compiles_and_links(name):
    exe = _build(name)
    assert os.path.exists(exe)
    nm = subprocess.run(["nm", "-u", exe], capture_output=True, text=True).stdout
    assert "gespmm_spmm_host" in nm


def test_host_only_cases_run_without_gpu():
    """The data-model cases (from_coo, validate, formats) need no device."""
    exe = _build("test_reference_api")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    for case in ("from_coo sorts", "validate reports every violation",
                 "KernelConfig and check_config", "CSR1 cache and Matrix Market"):
        line = [ln for ln in r.stdout.splitlines() if case in ln]
        assert line and line[0].startswith("ok"), (case, r.stdout, r.stderr)


@pytest.mark.gpu
@pytest.mark.parametrize("name", PROGRAMS)
def test_dropin_reference_cases_on_gpu(cuda, name):
    exe = _build(name)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout

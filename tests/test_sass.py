"""CPU: pin the exact-mode SASS of every shipped SpMM kernel.

Bit-exactness with the reference (product and combine rounded separately,
-ffp-contract=off, proj/CMakeLists.txt:10-12) holds only while the compiler
never contracts the fold's FMUL + FADD into an FFMA.  The library is built
with --fmad=false; this test reads the SASS of libgespmm.so with cuobjdump
and fails if a compiler change ever reintroduces a fused multiply-add in an
exact (FAST=false) kernel:

* sum / max / min: no FFMA and no FFMA2 at all;
* mean: no FFMA2, and no more FFMA than the IEEE division sequences need
  (<= 5 per MUFU.RCP, + 2) — the fold itself is the sum's.

Fast-mode (FAST=true) sum kernels must contain FFMA or FFMA2 (the contraction
the option asks for), which also proves the parser sees the kernels."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2007_03179_b200", "libgespmm.so")
CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"

pytestmark = pytest.mark.skipif(not (os.path.exists(LIB) and os.path.exists(CUOBJDUMP)),
                                reason="libgespmm.so or cuobjdump missing")

KERNEL = re.compile(r"(k_naive|k_crc|k_warp|k_cta|k_hub)<(\d+), (true|false)")
OPS = {0: "sum", 1: "mean", 2: "max", 3: "min"}


@pytest.fixture(scope="module")
def kernels():
    sass = subprocess.run([CUOBJDUMP, "-sass", LIB], capture_output=True, text=True,
                          check=True).stdout
    parts = re.split(r"\n\s*Function : ", sass)[1:]
    names = [p.split("\n", 1)[0].strip() for p in parts]
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True,
                         check=True).stdout.splitlines()
    out = []
    for d, body in zip(dem, parts):
        m = KERNEL.search(d)
        if not m:
            continue
        out.append(dict(name=d, kind=m.group(1), op=OPS[int(m.group(2))],
                        fast=m.group(3) == "true",
                        ffma=len(re.findall(r"\bFFMA\b", body)),
                        ffma2=len(re.findall(r"\bFFMA2\b", body)),
                        rcp=len(re.findall(r"\bMUFU\.RCP\b", body))))
    return out


def test_every_kernel_family_is_present(kernels):
    kinds = {(k["kind"], k["op"], k["fast"]) for k in kernels}
    for kind in ("k_naive", "k_crc", "k_warp", "k_cta", "k_hub"):
        for op in ("sum", "mean", "max", "min"):
            assert (kind, op, False) in kinds, (kind, op)
    assert len(kernels) > 200


def test_exact_sum_max_min_have_no_fused_multiply_add(kernels):
    bad = [k["name"] for k in kernels
           if not k["fast"] and k["op"] != "mean" and (k["ffma"] or k["ffma2"])]
    assert not bad, f"FFMA in exact kernels: {bad[:5]}"


def test_exact_mean_fuses_only_inside_the_division(kernels):
    bad = [(k["name"], k["ffma"], k["rcp"]) for k in kernels
           if not k["fast"] and k["op"] == "mean"
           and (k["ffma2"] or k["ffma"] > 5 * k["rcp"] + 2)]
    assert not bad, f"mean fold contracted: {bad[:5]}"


def test_fast_sum_kernels_do_contract(kernels):
    fast_sum = [k for k in kernels if k["fast"] and k["op"] == "sum"]
    assert fast_sum and all(k["ffma"] + k["ffma2"] > 0 for k in fast_sum)

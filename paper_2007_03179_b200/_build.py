"""In-tree build of libgespmm.so for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2007_03179_b200._build        # or __graft_entry__.build()

Objects go to build/ (git-ignored); the shared library lands next to this file
so it travels to the GPU box with the repo snapshot.  cudart is linked
statically: the library needs only libcuda from the driver.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "gespmm")
LIB = os.path.join(PKG, "libgespmm.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xcompiler", "-ffp-contract=off", "--fmad=false",
                     "-Xptxas", "-warn-spills", "-I", INCLUDE, "-I", CSRC]
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra",
             "-I", INCLUDE, "-I", CSRC, "-I", "/usr/local/cuda/include"]

CU_SOURCES = ["api.cu", "validate.cu", "kernels_faithful.cu", "kernels_tuned.cu", "diag.cu",
              "transpose.cu", "peer.cu", "h2dpack.cu", "coo.cu"]
# measured slower on B200: only in the GESPMM_EXPERIMENTAL build
EXPERIMENTAL_CU = ["hotcols.cu", "cluster.cu", "hotrows.cu"]
LIB_EXP = os.path.join(PKG, "libgespmm_exp.so")
BUILD_EXP = os.path.join(ROOT, "build", "gespmm_exp")
CXX_SOURCES = ["gen.cpp", "io.cpp", "h2dpack_host.cpp", "host_api.cpp"]
HEADERS = ["common.cuh", "launch.h"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stderr


def build(verbose: bool = False, force: bool = False, defines=(), build_dir=None,
          lib=None, experimental: bool = False) -> str:
    """defines/build_dir/lib: an experimental variant (-D flags) built into its
    own object dir and library path (tools/variant_build.py).
    experimental: also compile the measured-slower options (cluster DSMEM hot
    rows, hot-column L2 map, column slices, L2 persistence) into
    libgespmm_exp.so (selected at run time with GESPMM_EXPERIMENTAL=1)."""
    if experimental:
        defines = tuple(defines) + ("GESPMM_EXPERIMENTAL",)
        build_dir = build_dir or BUILD_EXP
        lib = lib or LIB_EXP
    BUILD = build_dir or globals()["BUILD"]
    LIB = lib or globals()["LIB"]
    cu_sources = CU_SOURCES + (EXPERIMENTAL_CU if "GESPMM_EXPERIMENTAL" in defines else [])
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "gespmm", "gespmm.h")]
    jobs, objs = [], []
    for src in cu_sources + CXX_SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if force or _stale(obj, [path] + hdrs):
            if src.endswith(".cu"):
                cmd = [NVCC] + NVCC_FLAGS + [f"-D{d}" for d in defines] + ["-c", path, "-o", obj]
                if src == "kernels_tuned.cu" and verbose:
                    cmd += ["-Xptxas", "-v"]
            else:
                cmd = ["g++"] + CXX_FLAGS + [f"-D{d}" for d in defines] + ["-c", path, "-o", obj]
                if src == "h2dpack_host.cpp":
                    cmd.insert(1, "-fopenmp")
            jobs.append(cmd)
    log = []
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            for out in ex.map(_run, jobs):
                if out:
                    log.append(out)
    if force or jobs or _stale(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs +
             ["-lgomp", "-lpthread"])
    text = "\n".join(log)
    if verbose and text:
        print(text, file=sys.stderr)
    return text


if __name__ == "__main__":
    exp = "--experimental" in sys.argv or os.environ.get("GESPMM_EXPERIMENTAL") == "1"
    build(verbose="-v" in sys.argv, force="-f" in sys.argv, experimental=exp)
    print(LIB_EXP if exp else LIB)

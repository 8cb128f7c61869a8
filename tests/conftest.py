import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (large shapes)")
    config.addinivalue_line("markers", "experimental: exercises the GESPMM_EXPERIMENTAL build's "
                                       "options (skipped on the default library)")


def experimental_built() -> bool:
    import paper_2007_03179_b200._lib as L
    return L.experimental_built()


def requires_experimental(fn):
    """Tests of options compiled only into libgespmm_exp.so; the default
    suite runs them through test_gpu_parity::test_experimental_build_suite."""
    fn = pytest.mark.experimental(fn)
    return pytest.mark.skipif("not __import__('conftest').experimental_built()",
                              reason="default build: experimental options not compiled")(fn)


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_npz():
    return np.load(os.path.join(GOLDEN_DIR, "small_cases.npz"))


@pytest.fixture(scope="session")
def cuda():
    import torch
    assert torch.cuda.is_available(), "GPU test run without a CUDA device"
    return torch.device("cuda:0")


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def first_divergence(got, want):
    """spmm_cli.cpp:286-294 style: first (i, j) whose bits differ, or None."""
    g, w = bits(got), bits(want)
    if g.shape != w.shape:
        return ("shape", g.shape, w.shape)
    diff = np.argwhere(g != w)
    if diff.size == 0:
        return None
    i, j = diff[0]
    return (int(i), int(j), float(np.asarray(got)[i, j]), float(np.asarray(want)[i, j]))

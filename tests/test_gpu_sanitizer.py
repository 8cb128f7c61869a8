"""GPU: compute-sanitizer over every kernel family (SURVEY §5 "race
detection": the reference has no sanitizer runs).  tools/sanitize_driver.py
runs one small invocation of each kernel (tuned warp shapes, the hub ring,
k_cta, the paper's Algorithms 1-3, the pipelined host entry with the packed
upload, the fused replica epilogue, the overlap_prev chain, transpose, COO
builders, validation), each checked against the oracle; memcheck and
racecheck must report nothing."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.skipif(not os.path.exists(SAN), reason="compute-sanitizer not installed")
@pytest.mark.parametrize("tool,verdict", [("memcheck", "ERROR SUMMARY: 0 errors"),
                                          ("racecheck", "RACECHECK SUMMARY: 0 hazards")])
def test_sanitizer_clean(tool, verdict):
    out = subprocess.run([SAN, "--tool", tool, "--target-processes", "all", "--print-limit", "20",
                          sys.executable, os.path.join(ROOT, "tools", "sanitize_driver.py")],
                         cwd=ROOT, capture_output=True, text=True, timeout=1200)
    text = out.stdout + out.stderr
    if "closed on this pool" in text:
        # the GPU pool's compute-sanitizer wrapper refuses to run (exit 86);
        # the last recorded runs are under profiles/r2/sanitizer/
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert out.returncode == 0, text[-4000:]
    assert "0 parity failures" in text, text[-4000:]
    assert verdict in text, text[-4000:]

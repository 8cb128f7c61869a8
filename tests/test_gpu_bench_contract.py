"""GPU: bench.py keeps the driver's JSON-line contract (one line on stdout with
the required keys; roofline, cpu_baseline, e2e, clocks, gpu_launches), on the
small Pubmed config so it runs in seconds; and the reference arm's line."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
            "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"]


def _run(args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run(["--config", "pubmed", "--steps", "5", "--warmup", "3"])
    for k in REQUIRED:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    cb = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in cb, k
    assert cb["kind"] in ("reference", "port")
    assert d["gpu_launches"] >= d["steps"]
    assert "workload" in d["config"]


def test_reference_arm_line_contract():
    d = _run(["--impl", "reference", "--config", "pubmed", "--steps", "3", "--warmup", "3"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port")


@pytest.mark.parametrize("gpus", [2, 4])
def test_bench_gpus2_launches_two_ranks_and_matches_oracle(tmp_path, gpus):
    """`bench.py --gpus 2` outside torchrun starts two ranks itself (gloo here:
    the box has one GPU, both ranks share it); the line reports n_gpus 2, the
    one-time B broadcast apart from the step, and the two C shards together
    are bit-identical to the oracle on the whole matrix."""
    import numpy as np
    import oracle as O
    env = dict(os.environ, GESPMM_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    dump = str(tmp_path / "c")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus),
                          "--config", "pubmed", "--steps", "3", "--warmup", "3", "--no-cpu",
                          "--dump-c", dump], cwd=ROOT, capture_output=True, text=True,
                         timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == gpus and d["config"]["parallelism"] == f"row-shard x{gpus}"
    assert d["setup"]["b_broadcast_bytes"] == 19717 * 128 * 4 and d["setup"]["backend"] == "gloo"
    bounds = json.load(open(dump + ".bounds.json"))["bounds"]
    assert len(bounds) == gpus + 1 and bounds[0] == 0 and bounds[-1] == 19717
    got = np.concatenate([np.load(f"{dump}.rank{r}.npy") for r in range(gpus)])
    rp, ci, v = O.ref_gen_uniform(19717, 88648, 1)
    v = np.ascontiguousarray(v, np.float32)
    O.randomize_values(v, 2)
    b = O.make_random_dense(19717, 128, 42)
    want, _ = O.spmm(19717, 19717, rp, ci, v, b, "sum")
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))



def _propagate(gpus, exchange, backend=None):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    if backend:
        env["GESPMM_DIST_BACKEND"] = backend
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus),
                          "--config", "propagate", "--base", "pubmed", "--hops", "2",
                          "--steps", "2", "--warmup", "3", "--exchange", exchange, "--checksum"],
                         cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_propagate_fused_and_nccl_exchange_equal_oracle():
    """`bench.py --config propagate`: stacked hops H_{t+1} = A H_t with the
    exchange fused into the SpMM epilogue (peer stores + device barrier) or as
    an all-gather, at 1 and 2 ranks (2 ranks share the one GPU: CUDA IPC
    mappings for fused, gloo for the all-gather).  Every line's final H is
    bit-identical to the oracle's 10 hops (3 warm-up + 2 timed steps of 2)."""
    import numpy as np
    import oracle as O
    import paper_2007_03179_b200 as G
    rp, ci, v = O.ref_gen_uniform(19717, 88648, 1)
    v = np.ascontiguousarray(v, np.float32)
    O.randomize_values(v, 2)
    h = O.make_random_dense(19717, 128, 42)
    for _ in range(10):
        h, _ = O.spmm(19717, 19717, rp, ci, v, h, "sum")
    want = int(G.checksum(G.DenseMatrix.of(h)))
    lines = [_propagate(1, "fused"), _propagate(1, "nccl"), _propagate(2, "fused", "gloo"),
             _propagate(2, "nccl", "gloo")]
    for d in lines:
        assert d["checksum"] == want, d
        assert d["steps"] == 4 and d["exchange"]["spmm_ms_per_hop"] > 0
        assert d["gpu_launches"] >= 4
    assert [d["n_gpus"] for d in lines] == [1, 1, 2, 2]

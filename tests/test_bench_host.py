"""CPU: bench.py pieces that run without a GPU — the reference arm is built
and timed with no product code loaded, both arms emit the same `config`."""
import json
import os
import subprocess
import sys

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_arm_loads_no_product_code():
    code = ("import sys, json; sys.argv=['bench.py','--impl','reference','--config','pubmed',"
            "'--steps','3','--warmup','3']; import bench; rc = bench.main(); "
            "maps = open('/proc/self/maps').read(); "
            "print(json.dumps({'rc': rc, 'pkg': any(m.startswith('paper_2007_03179_b200') "
            "for m in sys.modules), 'so': 'libgespmm' in maps, 'ref': 'libspmmref' in maps}))")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    line, probe = lines[0], lines[-1]
    assert probe == {"rc": 0, "pkg": False, "so": False, "ref": True}
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["cpu_baseline"]["cpu_model"]
    import bench
    assert line["config"] == bench.config_of(bench.CONFIGS["pubmed"], 1)


def test_config_of_is_shared_and_stable():
    import bench
    for name, cfg in bench.CONFIGS.items():
        c = bench.config_of(cfg, 4)
        assert c["workload"] == cfg["desc"] and c["parallelism"] == "row-shard x4"
        assert c["rows"] == cfg["rows"] and c["nnz"] == cfg["nnz"] and c["n"] == cfg["n"]


def test_bench_rejects_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--config", "pubmed"], cwd=ROOT, capture_output=True, text=True,
                         timeout=300, env=env)
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr

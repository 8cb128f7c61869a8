"""The reference CLI's record schema (spmm_cli.cpp:108-219, 566-611): CSV
header column for column, base-record keys, RFC-4180 quoting, checksum text.
The GPU test runs one bench through the device and checks the records
against the oracle."""
import json

import numpy as np
import pytest

import oracle as O
import paper_2007_03179_b200 as G
from paper_2007_03179_b200 import records as R

# spmm_cli.cpp:168-172, verbatim
REFERENCE_CSV_HEADER = (
    "matrix,backend,variant,cf,op,m,k,n,nnz,warp_size,warps_per_block,b_seed,"
    "gld_transactions,gst_transactions,requested_load_bytes,transferred_load_bytes,"
    "gld_efficiency,shared_loads,shared_stores,rowptr_load_tx,colind_load_tx,val_load_tx,"
    "b_load_tx,c_store_tx,workers,repeats,elapsed_s,gflops,checksum,verification,error")
BASE_KEYS = ["tool", "version", "timestamp", "input", "m", "k", "n", "nnz", "backend", "variant",
             "cf", "op", "warp_size", "warps_per_block", "b_seed"]  # spmm_cli.cpp:139-165


def test_csv_header_is_the_references():
    assert R.CSV_HEADER == REFERENCE_CSV_HEADER
    assert len(R.CSV_HEADER.split(",")) == 31


def test_base_record_keys_and_csv_row_shape():
    s = R.RunSettings(input_descriptor="gen:100,500,1", generator={"rows": 100, "nnz": 500,
                      "seed": 1, "self_loops": False}, m=100, k=100, n=32, nnz=500,
                      variant="crc-cwm", cf=2, op="max")
    rec = R.base_record(s)
    assert list(rec) == BASE_KEYS
    assert rec["tool"] == "spmm-lab" and rec["input"]["generator"]["nnz"] == 500
    line = R.csv_line(s)
    # the descriptor's comma forces quoting; 31 columns after parsing
    import csv
    import io
    row = next(csv.reader(io.StringIO(line)))
    assert len(row) == 31 and row[0] == "gen:100,500,1" and row[2] == "crc-cwm"
    assert row[12:24] == [""] * 12  # no simulator counts
    assert R.csv_field('a"b') == '"a""b"'
    assert R.hex_checksum(0x1234) == "0000000000001234"
    json.loads(R.dumps(rec))


@pytest.mark.gpu
def test_bench_records_on_device_match_oracle():
    a = G.gen_uniform_random(G.GraphGenSpec(2000, 20000, 5))
    G.randomize_values(a, 6)
    variants = [G.KernelVariant.naive(), G.KernelVariant.crc_cwm(2), G.KernelVariant.tuned()]

    def reference(m, b, op):
        return O.spmm(m.n_rows, m.n_cols, m.row_ptr, m.col_ind, m.vals, b.data, op)[0]

    out = list(R.bench_records(a, "gen:2000,20000,5", [32, 128], variants, "sum", repeats=3,
                               reference=reference))
    assert len(out) == 6
    for rec, line in out:
        assert rec["backend"] == "b200" and rec["verification"] == "bitwise"
        b = G.make_random_dense(a.n_cols, rec["n"], 42)
        want = O.checksum(reference(a, b, "sum"))
        assert rec["b200"]["checksum"] == R.hex_checksum(want)
        assert rec["b200"]["flops"] == 2 * a.nnz() * rec["n"] and rec["b200"]["gflops"] > 0
        import csv
        import io
        assert next(csv.reader(io.StringIO(line)))[28] == R.hex_checksum(want)
    assert "speedup_vs_first" in out[1][0]["b200"]

"""CPU: CSR1 cache round trips over random matrices (hypothesis): what
save_csr_cache writes, read_csr_cache returns bit for bit, and the byte
layout is the reference's (io.hpp:50-63; test_io.cpp:14-34)."""
import struct

import numpy as np
from hypothesis import given, seed, settings
from hypothesis import strategies as st

import paper_2007_03179_b200 as G


@seed(20261021)
@settings(max_examples=40, deadline=None)
@given(m=st.integers(0, 200), k=st.integers(1, 300), nnz=st.integers(0, 3000),
       data=st.integers(0, 1 << 30))
def test_csr1_round_trip_random(tmp_path_factory, m, k, nnz, data):
    rng = np.random.default_rng(data)
    rows = rng.integers(0, max(m, 1), nnz) if m else np.zeros(0, np.int64)
    cols = rng.integers(0, k, len(rows))
    keys = np.unique(rows * k + cols) if m else np.zeros(0, np.int64)
    r, c = keys // k, keys % k
    rp = np.zeros(m + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    a = G.CsrMatrix(m, k, np.cumsum(rp).astype(np.uint32), c.astype(np.uint32),
                    rng.standard_normal(len(keys)).astype(np.float32))
    path = tmp_path_factory.mktemp("csr1") / "m.csr1"
    G.save_csr_cache(str(path), a)
    raw = path.read_bytes()
    assert raw[:4] == b"CSR1"
    assert struct.unpack("<QQQ", raw[4:28]) == (m, k, len(keys))
    assert len(raw) == 28 + 4 * (m + 1) + 8 * len(keys)
    back = G.read_csr_cache(str(path))
    assert (back.n_rows, back.n_cols) == (m, k)
    assert np.array_equal(back.row_ptr, a.row_ptr)
    assert np.array_equal(back.col_ind, a.col_ind)
    assert np.array_equal(back.vals.view(np.uint32), a.vals.view(np.uint32))

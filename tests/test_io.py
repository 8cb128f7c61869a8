"""CSR1 binary cache (reference io.hpp:15-16, 50-115; tests mirror
proj/tests/test_io.cpp): pinned byte layout, bit-exact round trip, the
reference's error texts, and byte-for-byte agreement with the reference's own
save_csr_cache / load_matrix (oracle/_ref).  The streaming device loader is
checked on the GPU."""
import os

import numpy as np
import pytest

import oracle as O
import paper_2007_03179_b200 as G

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _m(rows, cols, rp, ci, v):
    return G.CsrMatrix(rows, cols, np.array(rp, np.uint32), np.array(ci, np.uint32),
                       np.array(v, np.float32))


def test_csr_cache_byte_layout_is_pinned(tmp_path):
    # test_io.cpp:14-35
    p = tmp_path / "one.csr"
    G.save_csr_cache(p, _m(1, 2, [0, 1], [1], [1.5]))
    want = bytes([ord("C"), ord("S"), ord("R"), ord("1"),
                  1, 0, 0, 0, 0, 0, 0, 0,
                  2, 0, 0, 0, 0, 0, 0, 0,
                  1, 0, 0, 0, 0, 0, 0, 0,
                  0, 0, 0, 0, 1, 0, 0, 0,
                  1, 0, 0, 0,
                  0x00, 0x00, 0xC0, 0x3F])
    assert p.read_bytes() == want


def test_csr_cache_round_trips_bit_exactly(tmp_path):
    # test_io.cpp:37-52
    m = G.gen_uniform_random(G.GraphGenSpec(64, 512, 5))
    G.randomize_values(m, 6)
    p = tmp_path / "r.csr"
    G.save_csr_cache(p, m)
    r = G.read_csr_cache(p)
    assert (r.n_rows, r.n_cols) == (m.n_rows, m.n_cols)
    assert np.array_equal(r.row_ptr, m.row_ptr)
    assert np.array_equal(r.col_ind, m.col_ind)
    assert np.array_equal(r.vals.view(np.uint32), m.vals.view(np.uint32))


def test_csr_cache_empty_matrix(tmp_path):
    p = tmp_path / "e.csr"
    G.save_csr_cache(p, G.CsrMatrix.empty(3, 4))
    r = G.read_csr_cache(p)
    assert (r.n_rows, r.n_cols, r.nnz()) == (3, 4, 0)
    assert np.array_equal(r.row_ptr, np.zeros(4, np.uint32))
    assert os.path.getsize(p) == 28 + 16


def _truncations(tmp_path):
    m = _m(1, 1, [0, 1], [0], [2.0])
    p = tmp_path / "t.csr"
    G.save_csr_cache(p, m)
    full = p.read_bytes()
    cases = {
        "magic": b"XSR1aaaaaaaaaaaaaaaaaaaaaaaa",
        "short": b"CS",
        "header": full[:20],
        "row_ptr": full[:30],
        "col_ind": full[:38],
        "vals": full[:-2],  # test_io.cpp:54-70
        "range": b"CSR1" + (2**32).to_bytes(8, "little") + bytes(16),
    }
    out = {}
    for name, data in cases.items():
        q = tmp_path / f"{name}.csr"
        q.write_bytes(data)
        out[name] = q
    return out


def test_csr_cache_rejects_bad_magic_and_truncation(tmp_path):
    files = _truncations(tmp_path)
    want = {
        "magic": "csr cache: bad magic (expected CSR1)",
        "short": "csr cache: bad magic (expected CSR1)",
        "header": "csr cache: truncated header",
        "row_ptr": "csr cache: truncated row_ptr",
        "col_ind": "csr cache: truncated col_ind",
        "vals": "csr cache: truncated vals",
        "range": "csr cache: dimensions exceed 32-bit range",
    }
    for name, path in files.items():
        with pytest.raises(G.Error) as e:
            G.read_csr_cache(path)
        assert str(e.value) == want[name], name


def test_missing_file_and_extension_dispatch(tmp_path):
    with pytest.raises(G.Error, match="cannot open"):
        G.read_csr_cache(tmp_path / "nope.csr")
    # the reference opens the file before dispatching on the extension (io.hpp:100-113)
    with pytest.raises(G.Error, match="cannot open"):
        G.load_matrix(tmp_path / "x.bin")
    (tmp_path / "x.bin").write_bytes(b"x")
    with pytest.raises(G.Error, match=r"unknown matrix extension '\.bin' \(expected \.mtx or \.csr\)"):
        G.load_matrix(tmp_path / "x.bin")


@needs_ref
def test_writer_matches_reference_bytes(tmp_path):
    m = G.gen_uniform_random(G.GraphGenSpec(300, 4000, 11))
    G.randomize_values(m, 12)
    ours, theirs = tmp_path / "ours.csr", tmp_path / "ref.csr"
    G.save_csr_cache(ours, m)
    O.ref_save_csr_cache(str(theirs), m.n_rows, m.n_cols, m.row_ptr, m.col_ind, m.vals)
    assert ours.read_bytes() == theirs.read_bytes()
    rm, rk, rp, ci, v = O.ref_load_matrix(str(ours))
    assert (rm, rk) == (m.n_rows, m.n_cols)
    assert np.array_equal(rp, m.row_ptr) and np.array_equal(ci, m.col_ind)
    assert np.array_equal(v.view(np.uint32), m.vals.view(np.uint32))


@needs_ref
def test_error_texts_match_reference(tmp_path):
    for name, path in _truncations(tmp_path).items():
        with pytest.raises(O.RefError) as want:
            O.ref_load_matrix(str(path))
        with pytest.raises(G.Error) as got:
            G.read_csr_cache(path)
        assert str(got.value) == str(want.value), name


# ---------------------------------------------------------------------------
# GPU: streaming loader into HBM + device canonical check
# ---------------------------------------------------------------------------

@pytest.mark.gpu
def test_device_loader_round_trip(tmp_path, cuda):
    a = G.gen_powerlaw(20000, 600000, 3000, 1.0, 3)
    G.randomize_values(a, 4)
    p = tmp_path / "pl.csr"
    G.save_csr_cache(p, a)
    d = G.DeviceCsr.load(p, cuda)
    h = d.to_host()
    assert (h.n_rows, h.n_cols) == (a.n_rows, a.n_cols)
    assert np.array_equal(h.row_ptr, a.row_ptr) and np.array_equal(h.col_ind, a.col_ind)
    assert np.array_equal(h.vals.view(np.uint32), a.vals.view(np.uint32))
    m = G.load_matrix(p)
    assert np.array_equal(m.col_ind, a.col_ind)


@pytest.mark.gpu
def test_device_loader_multi_chunk(tmp_path, cuda):
    # > 2 staging chunks (32 MB each) with array boundaries inside chunks
    a = G.gen_powerlaw(150000, 9_000_000, 20000, 1.0, 5)
    G.randomize_values(a, 6)
    p = tmp_path / "big.csr"
    G.save_csr_cache(p, a)
    d = G.DeviceCsr.load(p, cuda)
    assert np.array_equal(d.col_ind.cpu().numpy().view(np.uint32), a.col_ind)
    assert np.array_equal(d.vals.cpu().numpy().view(np.uint32), a.vals.view(np.uint32))
    assert np.array_equal(d.row_ptr.cpu().numpy().view(np.uint32), a.row_ptr)


@pytest.mark.gpu
def test_device_loader_rejects_non_canonical_like_reference(tmp_path, cuda):
    bad = _m(2, 3, [0, 2, 3], [1, 0, 2], [1.0, 1.0, 1.0])  # row 0 not increasing
    p = tmp_path / "bad.csr"
    G.save_csr_cache(p, bad)
    with pytest.raises(G.Error) as got:
        G.DeviceCsr.load(p, cuda)
    assert "load_matrix: matrix is not canonical CSR" in str(got.value)
    with pytest.raises(G.Error) as got_host:
        G.load_matrix(p)
    assert str(got_host.value) == str(got.value)
    if O.ref_available():
        with pytest.raises(O.RefError) as want:
            O.ref_load_matrix(str(p))
        assert str(got.value) == str(want.value)
    d = G.DeviceCsr.load(p, cuda, validate=False)
    assert d.nnz() == 3

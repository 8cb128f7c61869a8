"""CPU: the library's host data-model entry points against the reference
itself (oracle/_ref: the unmodified csr.hpp / matrix_market.hpp / io.hpp):
gespmm_validate_host (every violation), gespmm_from_coo (both dedup
policies) and gespmm_mtx_parse behind load_matrix('.mtx')."""
import numpy as np
import pytest
from hypothesis import given, seed, settings
from hypothesis import strategies as st

import oracle as O
import paper_2007_03179_b200 as G

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@needs_ref
@seed(20261101)
@settings(max_examples=300, deadline=None)
@given(m=st.integers(0, 12), k=st.integers(0, 12), data=st.data())
def test_validate_matches_reference_on_random_broken_csr(m, k, data):
    """Random row_ptr / col_ind (often non-canonical, lengths off by one):
    same violation count and same first message as the reference's validate."""
    rp_len = data.draw(st.sampled_from([m + 1, m + 1, m + 1, m, m + 2]))
    rp = np.sort(np.array(data.draw(st.lists(st.integers(0, 30), min_size=rp_len,
                                             max_size=rp_len)), np.uint32))
    if rp_len and data.draw(st.booleans()):
        rp[0] = 0
    if rp_len > 2 and data.draw(st.booleans()):  # break monotonicity
        rp[1], rp[2] = rp[2], rp[1]
    nnz = int(rp[-1]) if rp_len else 0
    nnz = max(0, nnz + data.draw(st.sampled_from([0, 0, 0, -1, 1])))
    ci = np.array(data.draw(st.lists(st.integers(0, max(k + 1, 1)), min_size=nnz,
                                     max_size=nnz)), np.uint32)
    v_len = nnz + data.draw(st.sampled_from([0, 0, 0, 1]))
    vals = np.ones(v_len, np.float32)
    want_n, want_msg = O.ref_validate(m, k, rp, ci, vals)
    rep = G.validate(G.CsrMatrix(m, k, rp, ci, vals))
    assert len(rep.violations) == want_n
    if want_n:
        assert rep.violations[0] == want_msg


@needs_ref
@seed(20261102)
@settings(max_examples=200, deadline=None)
@given(rows=st.integers(0, 9), cols=st.integers(1, 9),
       ent=st.lists(st.tuples(st.integers(0, 8), st.integers(0, 8),
                              st.floats(-4, 4, width=32)), max_size=40))
def test_from_coo_sum_matches_reference(rows, cols, ent):
    ent = [(r, c, v) for r, c, v in ent if r < rows and c < cols]
    r = np.array([e[0] for e in ent], np.uint32)
    c = np.array([e[1] for e in ent], np.uint32)
    v = np.array([e[2] for e in ent], np.float32)
    wrp, wci, wv = O.ref_from_coo(rows, cols, r, c, v)
    got = G.from_coo(rows, cols, (r, c, v), "sum")
    assert np.array_equal(got.row_ptr, wrp) and np.array_equal(got.col_ind, wci)
    assert np.array_equal(got.vals.view(np.uint32), wv.view(np.uint32))


def test_from_coo_last_policy_and_bounds_text():
    m = G.from_coo(2, 3, [(1, 2, 1.0), (0, 1, 2.0), (1, 2, 7.0), (1, 0, 3.0)], "last")
    assert m.row_ptr.tolist() == [0, 1, 3] and m.col_ind.tolist() == [1, 0, 2]
    assert m.vals.tolist() == [2.0, 3.0, 7.0]
    with pytest.raises(G.Error, match=r"coo entry \(2, 0, 1.5\) outside declared 2x3 bounds"):
        G.from_coo(2, 3, [(2, 0, 1.5)])


MTX_CASES = [
    "%%MatrixMarket matrix coordinate real general\n% c\n3 4 3\n1 1 2.5\n3 4 -1\n1 1 0.5\n",
    "%%MatrixMarket matrix coordinate pattern symmetric\n4 4 3\n2 1\n4 4\n3 2\n",
    "%%MatrixMarket matrix coordinate integer general\r\n2 2 2\r\n1 2 3\r\n2 1 4\r\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "%%MatrixMarket matrix array real general\n2 2\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 x\n",
    "%%MatrixMarket matrix coordinate real general\n2 2\n",
    "not a header\n",
    "",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
]


@needs_ref
@pytest.mark.parametrize("i", range(len(MTX_CASES)))
def test_load_matrix_mtx_matches_reference(tmp_path, i):
    p = tmp_path / "m.mtx"
    p.write_bytes(MTX_CASES[i].encode())
    try:
        want = O.ref_load_matrix(str(p))
        err = None
    except O.RefError as e:
        want, err = None, str(e)
    if err is not None:
        with pytest.raises(G.Error) as got:
            G.load_matrix(p)
        assert str(got.value) == err
        return
    got = G.load_matrix(p)
    m, k, rp, ci, v = want
    assert (got.n_rows, got.n_cols) == (m, k)
    assert np.array_equal(got.row_ptr, rp) and np.array_equal(got.col_ind, ci)
    assert np.array_equal(got.vals.view(np.uint32), v.view(np.uint32))

"""CPU: pin the oracle restatement (oracle/spmm_oracle.c) before trusting it.

1. against the committed golden fixtures made from the UNMODIFIED reference
   (tests/golden/make_golden.py): hand cases, the seed-404 / seed-20260810
   corpora, the Cora/Pubmed config checksums, the validation messages;
2. against the reference itself, where oracle/_ref was built here;
3. the new ops (mean, min, arg) against identities that tie them to the
   reference's own sum and max.
"""
import numpy as np
import pytest

import oracle as O
import paper_2007_03179_b200 as G
from conftest import bits, first_divergence


def _inputs(spec):
    a = G.gen_uniform_random(G.GraphGenSpec(spec["rows"], spec["nnz"], spec["gen_seed"],
                                            spec["loops"]))
    G.randomize_values(a, spec["val_seed"])
    b = G.make_random_dense(spec["rows"], spec["n"], spec["b_seed"])
    return a, b


def test_hand_cases_bitwise(golden, golden_npz):
    for case in golden["hand_cases"]:
        i = case["npz_index"]
        rp, ci, v = (golden_npz[f"hand{i}_{k}"] for k in ("row_ptr", "col_ind", "vals"))
        b, want = golden_npz[f"hand{i}_b"], golden_npz[f"hand{i}_want"]
        got, _ = O.spmm(case["m"], case["k"], rp, ci, v, b, case["op"], threads=1)
        assert first_divergence(got, want) is None, case["name"]
        assert O.checksum(got) == case["checksum"], case["name"]


def test_hand_case_values_match_reference_tests(golden, golden_npz):
    """The literal expectations of test_kernels.cpp / test_oracle.cpp."""
    names = {c["name"]: c["npz_index"] for c in golden["hand_cases"]}
    want = golden_npz[f"hand{names['single_row_2_3']}_want"]
    assert want[0, 0] == 2.0 and want[0, 1] == 3.0
    want = golden_npz[f"hand{names['two_rows_times_ones']}_want"]
    assert np.all(want == 3.0)
    want = golden_npz[f"hand{names['max_pool_neighbors']}_want"]
    assert want[0, 0] == 5.0 and want[1, 0] == np.finfo(np.float32).min
    want = golden_npz[f"hand{names['upper_triangular_times_identity']}_want"]
    assert want.tolist() == [[1.0, 2.0], [0.0, 3.0]]
    want = golden_npz[f"hand{names['empty_rows_sum_seed']}_want"]
    assert np.all(bits(want) == 0)
    want = golden_npz[f"hand{names['cwm_lane_owns_strided_columns']}_want"]
    assert want[0, 0] == 2.0 and want[0, 32] == 66.0


def test_small_cases_bitwise(golden, golden_npz):
    for case in golden["small_cases"]:
        i = case["npz_index"]
        rp, ci, v, b, want = (golden_npz[f"small{i}_{k}"]
                              for k in ("row_ptr", "col_ind", "vals", "b", "want"))
        got, _ = O.spmm(case["rows"], case["rows"], rp, ci, v, b, case["op"], threads=2)
        assert first_divergence(got, want) is None


def test_random_corpus_checksums(golden):
    """225 reference-shaped cases (test_kernels.cpp:118-137, acceptance.cpp:73-116)."""
    for spec in golden["random_corpus"]:
        a, b = _inputs(spec)
        got, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b.data, spec["op"])
        assert O.checksum(got) == spec["checksum"], spec


@pytest.mark.parametrize("idx", range(8))
def test_config_checksums(golden, idx):
    """BASELINE configs 0-1 on the reference generator: the survey's probe checksums."""
    spec = golden["configs"][idx]
    a = G.gen_uniform_random(G.GraphGenSpec(spec["rows"], spec["nnz"], spec["gen_seed"]))
    G.randomize_values(a, spec["val_seed"])
    b = G.make_random_dense(spec["rows"], spec["n"], spec["b_seed"])
    got, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b.data, spec["op"])
    assert O.checksum(got) == spec["checksum"]


def test_validation_messages(golden):
    for case in golden["validation"]:
        n, first = O.validate(case["m"], case["k"], np.array(case["row_ptr"], np.uint32),
                              np.array(case["col_ind"], np.uint32),
                              np.array(case["vals"], np.float32))
        if case["name"] == "dimension_mismatch" or case["name"] == "zero_n":
            assert n == 0
            continue
        assert n == case["violations"], case["name"]
        assert first == case["first_violation"], case["name"]


def test_skip_tail_fault_changes_result():
    rng = np.random.default_rng(88)
    a = G.gen_uniform_random(G.GraphGenSpec(40, 300, 3))
    G.randomize_values(a, 4)
    b = G.make_random_dense(40, 16, 2)
    good, _ = O.spmm(40, 40, a.row_ptr, a.col_ind, a.vals, b.data, "sum")
    bad, _ = O.spmm(40, 40, a.row_ptr, a.col_ind, a.vals, b.data, "sum", skip_tail=True)
    assert first_divergence(bad, good) is not None
    del rng


def _rand(seed, rows=150, nnz=2500, n=37):
    a = G.gen_uniform_random(G.GraphGenSpec(rows, nnz, seed))
    G.randomize_values(a, seed + 1)
    b = G.make_random_dense(rows, n, seed + 2)
    return a, b


def test_min_is_negated_max_of_negated_values():
    """min(v*b) == -max((-v)*b) bitwise, arg included: pins min through the reference's max."""
    for seed in range(5):
        a, b = _rand(seed)
        mn, amn = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b.data, "min",
                         want_arg=True)
        mx, amx = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, -a.vals, b.data, "max",
                         want_arg=True)
        assert first_divergence(mn, -mx) is None
        assert np.array_equal(amn, amx)


def test_mean_is_sum_over_degree():
    for seed in range(3):
        a, b = _rand(seed + 10)
        s, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b.data, "sum")
        m, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b.data, "mean")
        deg = np.diff(a.row_ptr.astype(np.int64)).astype(np.float32)[:, None]
        want = np.where(deg > 0, s / np.where(deg > 0, deg, 1), s).astype(np.float32)
        assert first_divergence(m, want) is None


def test_arg_is_earliest_position_of_the_max():
    for seed in range(3):
        a, b = _rand(seed + 20, rows=60, nnz=700, n=9)
        # make ties likely: quantise B
        bq = np.round(b.data * 4) / 4
        mx, arg = O.spmm(60, 60, a.row_ptr, a.col_ind, a.vals, bq, "max", want_arg=True)
        _, argc = O.spmm(60, 60, a.row_ptr, a.col_ind, a.vals, bq, "max", want_arg=True,
                         arg_kind=O.ARG_COLUMN)
        for i in range(60):
            s, e = a.row_ptr[i], a.row_ptr[i + 1]
            for j in range(9):
                prods = (a.vals[s:e] * bq[a.col_ind[s:e], j]).astype(np.float32)
                if e == s:
                    assert arg[i, j] == -1 and mx[i, j] == np.finfo(np.float32).min
                    continue
                p = s + int(np.argmax(prods))  # numpy: first occurrence of the max
                assert arg[i, j] == p and mx[i, j] == prods.max()
                assert argc[i, j] == a.col_ind[p]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")
def test_restatement_equals_reference_sum_max():
    for seed in range(6):
        a, b = _rand(seed + 30, rows=300, nnz=5000, n=[1, 5, 33, 64, 128, 130][seed])
        for op in ("sum", "max"):
            for variant, cf in (("naive", 1), ("crc", 1), ("crc-cwm", 4)):
                want = O.ref_native_spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals,
                                         b.data, op, variant, cf, 3)
                got, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b.data, op)
                assert first_divergence(got, want) is None


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")
def test_restatement_equals_reference_skip_tail():
    a, b = _rand(77, rows=80, nnz=3000, n=20)
    want = O.ref_native_spmm(80, 80, a.row_ptr, a.col_ind, a.vals, b.data, "sum", "crc", 1, 2,
                             skip_tail=True)
    got, _ = O.spmm(80, 80, a.row_ptr, a.col_ind, a.vals, b.data, "sum", skip_tail=True)
    assert first_divergence(got, want) is None


def test_powerlaw_sample_against_dense_oracle():
    """The restatement on a power-law sample equals a numpy float32 ordered fold."""
    a = G.gen_powerlaw(400, 12000, 390, 1.0, 5)
    G.randomize_values(a, 6)
    b = G.make_random_dense(400, 8, 7)
    got, _ = O.spmm(400, 400, a.row_ptr, a.col_ind, a.vals, b.data, "sum")
    want = np.zeros((400, 8), np.float32)
    for i in range(400):
        acc = np.zeros(8, np.float32)
        for p in range(a.row_ptr[i], a.row_ptr[i + 1]):
            acc = (acc + (a.vals[p] * b.data[a.col_ind[p]]).astype(np.float32)).astype(np.float32)
        want[i] = acc
    assert first_divergence(got, want) is None


@pytest.mark.parametrize("shape", [(2000, 60000, 1500, 7), (50000, 2_000_000, 5000, 1),
                                   (2449, 123_718, 1748, 1), (3, 4, 2, 5)])
def test_powerlaw_restatement_matches_product(shape):
    """The oracle's C restatement of the power-law generator (the reference arm's
    input builder) is bit-identical to the product's gespmm_gen_powerlaw."""
    rows, nnz, maxdeg, seed = shape
    rp, ci, v = O.gen_powerlaw(rows, nnz, maxdeg, 1.0, seed)
    a = G.gen_powerlaw(rows, nnz, maxdeg, 1.0, seed)
    assert np.array_equal(rp, a.row_ptr) and np.array_equal(ci, a.col_ind)
    assert np.array_equal(v, a.vals)
    assert int(rp[-1]) == nnz


def test_value_and_dense_restatements_match_reference():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    for n, seed in ((0, 1), (1, 2), (1000, 2), (99991, 123456789)):
        v = np.zeros(n, np.float32)
        O.randomize_values(v, seed)
        assert np.array_equal(v.view(np.uint32), O.ref_randomize_values(np.zeros(n), seed)
                              .view(np.uint32))
    for r, c, seed in ((1, 1, 42), (300, 17, 42), (64, 128, 7)):
        assert np.array_equal(O.make_random_dense(r, c, seed).view(np.uint32),
                              O.ref_make_random_dense(r, c, seed).view(np.uint32))

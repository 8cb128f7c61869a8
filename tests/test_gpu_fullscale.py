"""GPU, full BASELINE sizes: the whole output compared bit for bit with the
reference's own CPU native_spmm (oracle/_ref: the unmodified headers,
native.hpp:101-143, every host thread) — not a row sample — plus the ops the
reference lacks (argmax, mean) against the oracle restatement, and the GCN
widths of A and A^T.

Each case reports the checksum (dense.hpp:62-72) of both sides and the first
divergent element (spmm_cli.cpp:286-294 style) on failure."""
import numpy as np
import pytest

import oracle as O
import paper_2007_03179_b200 as G
from conftest import first_divergence

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

REDDIT = (232_965, 114_800_000, 21_657)
PRODUCTS = (2_449_029, 123_718_280, 17_481)


def _gpu(a, b, op, want_arg=False, exec=None):
    import torch
    d = G.DeviceCsr.from_host(a, "cuda:0")
    bt = torch.from_numpy(b).to("cuda:0")
    c, arg = G.spmm(d, bt, op, want_arg=want_arg, exec=exec or G.ExecOptions())
    torch.cuda.synchronize()
    out = c.cpu().numpy(), (arg.cpu().numpy() if arg is not None else None)
    del d, bt, c, arg
    torch.cuda.empty_cache()
    return out


def _matrix(shape, seed=1, vseed=2):
    m, nnz, maxdeg = shape
    a = G.gen_powerlaw(m, nnz, maxdeg, 1.0, seed)
    G.randomize_values(a, vseed)
    return a


def _assert_bits(got, want, what):
    div = first_divergence(got, want)
    assert div is None, f"{what}: first divergence {div}; checksum got " \
                        f"{O.checksum(got):#x} want {O.checksum(want):#x}"


@needs_ref
def test_reddit_n128_sum_whole_matrix_equals_reference(cuda):
    a = _matrix(REDDIT)
    b = G.make_random_dense(a.n_cols, 128, 42).data
    got, _ = _gpu(a, b, "sum")
    want = O.ref_native_spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b, "sum",
                             "crc-cwm", 2, 0)
    _assert_bits(got, want, "Reddit N=128 sum")
    assert O.ref_checksum(got) == O.ref_checksum(want)


@needs_ref
def test_products_n256_max_whole_matrix_and_argmax(cuda):
    a = _matrix(PRODUCTS)
    b = G.make_random_dense(a.n_cols, 256, 42).data
    got, arg = _gpu(a, b, "max", want_arg=True)
    want = O.ref_native_spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b, "max",
                             "crc-cwm", 2, 0)
    _assert_bits(got, want, "products N=256 max")
    del want
    # argmax has no reference implementation: the threaded restatement, all rows
    want_c, want_arg = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b, "max",
                              want_arg=True)
    _assert_bits(got, want_c, "products N=256 max (restatement)")
    bad = np.argwhere(arg != want_arg)
    assert bad.size == 0, f"argmax: {len(bad)} mismatches, first {bad[0].tolist()}"
    # every non-empty row's argmax points into that row
    rp = a.row_ptr.astype(np.int64)
    rows = np.repeat(np.arange(a.n_rows), np.diff(rp))
    nonempty = np.diff(rp) > 0
    sel = arg[nonempty]
    assert (sel >= 0).all()
    assert np.array_equal(rows[sel[:, 0]], np.nonzero(nonempty)[0])


@pytest.mark.parametrize("n", [32, 64, 128])
@pytest.mark.parametrize("op", ["mean", "min"])
def test_pubmed_mean_min_whole_matrix(cuda, n, op):
    """Pubmed shape through the reference's own uniform generator (when built),
    mean and min (no reference implementation) against the restatement, whose
    sum/max are pinned to the reference in test_oracle.py."""
    if O.ref_available():
        rp, ci, v = O.ref_gen_uniform(19_717, 88_648, 1)
        a = G.CsrMatrix(19_717, 19_717, rp, ci, np.ascontiguousarray(v, np.float32))
    else:
        a = G.gen_uniform_random(G.GraphGenSpec(19_717, 88_648, 1))
    G.randomize_values(a, 2)
    b = G.make_random_dense(a.n_cols, n, 42).data
    got, arg = _gpu(a, b, op, want_arg=op == "min")
    want, warg = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b, op,
                        want_arg=op == "min")
    _assert_bits(got, want, f"Pubmed N={n} {op}")
    if warg is not None:
        assert np.array_equal(arg, warg)


@needs_ref
@pytest.mark.parametrize("n", [256, 44])
def test_gcn_widths_a_and_at_equal_reference(cuda, n):
    """The GCN's aggregations on the Reddit shape: A = D^-1/2 (A+I) D^-1/2 and
    its transpose (built on the device), at the hidden width 256 and the padded
    class width 44, each against the reference's native_spmm."""
    from paper_2007_03179_b200 import gcn
    a = gcn.normalize_adjacency(_matrix(REDDIT))
    at = G.DeviceCsr.from_host(a, "cuda:0").transpose().to_host()
    x = G.make_random_dense(a.n_cols, n, 3).data
    variant, cf = ("crc", 1) if n <= 32 else ("crc-cwm", 2)
    for name, m in (("A", a), ("A^T", at)):
        got, _ = _gpu(m, x, "sum")
        want = O.ref_native_spmm(m.n_rows, m.n_cols, m.row_ptr, m.col_ind, m.vals, x, "sum",
                                 variant, cf, 0)
        _assert_bits(got, want, f"GCN {name} N={n}")


@needs_ref
@pytest.mark.parametrize("op", ["sum", "max"])
def test_cora_equals_reference_dense_oracle(cuda, op):
    """BASELINE config 0 (Cora shape, N=16) against the reference's
    independent brute-force oracle dense_reference (oracle.hpp:42-57: the
    densified A folded in ascending k), every kernel variant."""
    rp, ci, v = O.ref_gen_uniform(2708, 10556, 1)
    a = G.CsrMatrix(2708, 2708, rp, ci, np.ascontiguousarray(v, np.float32))
    G.randomize_values(a, 2)
    b = G.make_random_dense(2708, 16, 42).data
    want = O.ref_dense_reference(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b, op)
    for variant in (G.KernelVariant.tuned(), G.KernelVariant.naive(), G.KernelVariant.crc(),
                    G.KernelVariant.crc_cwm(2), G.KernelVariant.crc_cwm(8)):
        c = G.native_spmm(a, G.DenseMatrix.of(b), variant, G.reduce_op_by_name(op))
        _assert_bits(c.data, want, f"Cora N=16 {op} {variant}")


def _shard(a, g, world):
    from paper_2007_03179_b200 import dist as D
    bounds = D.partition_rows(a.row_ptr, world)
    return D.shard_csr(a, bounds[g], bounds[g + 1])


@pytest.mark.parametrize("g", [0, 7])
def test_products_8way_shard_split_hub_rows_bit_exact(cuda, g):
    """An 8-way products shard takes the split-hub-row path (segments through
    k_warp + ordered combine): max and argmax over the whole shard equal the
    restatement bit for bit."""
    a = _shard(_matrix(PRODUCTS), g, 8)
    b = G.make_random_dense(a.n_cols, 256, 42).data
    d = G.DeviceCsr.from_host(a, "cuda:0")
    plan = G.Plan(d, 256, "max")
    assert "split" in plan.description, plan.description
    plan.close()
    got, arg = _gpu(a, b, "max", want_arg=True)
    want, want_arg = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b, "max",
                            want_arg=True)
    _assert_bits(got, want, f"products shard {g}/8 max")
    assert np.array_equal(arg, want_arg)


@pytest.mark.parametrize("g", [0, 3])
def test_reddit_8way_shard_exact_ring_bit_exact(cuda, g):
    """An 8-way Reddit shard, exact sum: its hub rows go through the ring
    kernel run ahead of the warp kernel; the whole shard equals the
    reference's fold bit for bit."""
    a = _shard(_matrix(REDDIT), g, 8)
    b = G.make_random_dense(a.n_cols, 128, 42).data
    d = G.DeviceCsr.from_host(a, "cuda:0")
    plan = G.Plan(d, 128, "sum")
    assert "hub_rows=0 " not in plan.description and "split" not in plan.description
    plan.close()
    got, _ = _gpu(a, b, "sum")
    want, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b, "sum")
    _assert_bits(got, want, f"Reddit shard {g}/8 sum")


def test_reddit_8way_shard_fast_sum_split_within_tolerance(cuda):
    """Fast mode on an 8-way Reddit shard: hub rows split into segments (the
    partial sums reassociate the fold), everything FFMA; within the north_star
    tolerance, |got - want| <= 1e-5 * max(|want|, sum |v * b|), on the whole
    shard."""
    a = _shard(_matrix(REDDIT), 0, 8)
    b = G.make_random_dense(a.n_cols, 128, 42).data
    d = G.DeviceCsr.from_host(a, "cuda:0")
    plan = G.Plan(d, 128, "sum", exec=G.ExecOptions(exact=False))
    assert "split" in plan.description, plan.description
    plan.close()
    got, _ = _gpu(a, b, "sum", exec=G.ExecOptions(exact=False))
    want, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b, "sum")
    mag, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, np.abs(a.vals), np.abs(b), "sum")
    err = np.abs(got.astype(np.float64) - want)
    assert np.all(err <= 1e-5 * np.maximum(np.abs(want), mag) + 1e-30), float(np.max(err / (mag + 1e-30)))

"""GPU: device COO <-> CSR (gespmm_from_coo_device / gespmm_to_coo_device)
against the reference's own from_coo (oracle/_ref, csr.hpp:58-93): row_ptr,
col_ind and the folded values bit-identical for both dedup policies, on
duplicate-heavy random triples, empty rows/inputs, the bounds error text, and
the Reddit-scale shuffled edge list of the benchmark graph."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2007_03179_b200 as G

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _dev(r, c, v):
    return (torch.from_numpy(np.ascontiguousarray(r, np.uint32).view(np.int32)).to(DEV),
            torch.from_numpy(np.ascontiguousarray(c, np.uint32).view(np.int32)).to(DEV),
            torch.from_numpy(np.ascontiguousarray(v, np.float32)).to(DEV))


def _check(d, rp, ci, v):
    assert np.array_equal(d.row_ptr.cpu().numpy().view(np.uint32), rp)
    assert np.array_equal(d.col_ind.cpu().numpy().view(np.uint32), ci)
    assert np.array_equal(d.vals.cpu().numpy().view(np.uint32), v.view(np.uint32))


@needs_ref
@pytest.mark.parametrize("policy", ["sum", "last"])
@pytest.mark.parametrize("rows,cols,count,seed", [
    (50, 40, 3000, 1),        # ~1.5 duplicates per position: long runs
    (1000, 1000, 20000, 2),   # sparse, few duplicates, empty rows
    (1, 5, 200, 3),           # one row, every run long
    (300, 1, 500, 4),         # one column
    (7, 9, 0, 5),             # empty input
    (70000, 90000, 200000, 6),  # keys above 32 bits
])
def test_from_coo_device_equals_reference(rows, cols, count, seed, policy):
    rng = np.random.default_rng(seed)
    r = rng.integers(0, rows, count).astype(np.uint32)
    c = rng.integers(0, cols, count).astype(np.uint32)
    v = (rng.standard_normal(count) * 3).astype(np.float32)
    wrp, wci, wv = O.ref_from_coo(rows, cols, r, c, v, policy)
    d = G.DeviceCsr.from_coo(rows, cols, *_dev(r, c, v), policy=policy)
    _check(d, wrp, wci, wv)
    # to_coo round trip: the canonical triples in row-major order
    rr, cc, vv = d.to_coo()
    want_r = np.repeat(np.arange(rows, dtype=np.uint32), np.diff(wrp.astype(np.int64)))
    assert np.array_equal(rr.cpu().numpy().view(np.uint32), want_r)
    assert np.array_equal(cc.cpu().numpy().view(np.uint32), wci)
    assert np.array_equal(vv.cpu().numpy().view(np.uint32), wv.view(np.uint32))


@needs_ref
def test_from_coo_device_bounds_error_text():
    r = np.array([0, 1, 5, 9, 2], np.uint32)
    c = np.array([0, 7, 1, 0, 3], np.uint32)
    v = np.array([1.0, 2.5, -0.125, 3.0, 1e-7], np.float32)
    with pytest.raises(O.RefError) as want:
        O.ref_from_coo(4, 6, r, c, v)
    with pytest.raises(G.Error) as got:
        G.DeviceCsr.from_coo(4, 6, *_dev(r, c, v))
    assert str(got.value) == str(want.value)  # first offender in input order: (1, 7, 2.5)


def test_from_coo_device_rebuilds_the_benchmark_graph():
    """The Reddit-shaped benchmark CSR, expanded to triples and shuffled, comes
    back bit-identical (unique positions: the fold is a copy)."""
    a = G.gen_powerlaw(232965, 114800000, 21657, 1.0, 1)
    G.randomize_values(a, 2)
    d = G.DeviceCsr.from_host(a, DEV)
    r, c, v = d.to_coo()
    perm = torch.randperm(r.numel(), device=DEV, generator=torch.Generator(DEV).manual_seed(0))
    back = G.DeviceCsr.from_coo(a.n_rows, a.n_cols, r[perm].contiguous(), c[perm].contiguous(),
                                v[perm].contiguous())
    _check(back, np.asarray(a.row_ptr, np.uint32), np.asarray(a.col_ind, np.uint32),
           np.asarray(a.vals, np.float32))


@needs_ref
def test_release_workspace_between_calls():
    """gespmm_release_workspace frees the COO scratch and the host entry's
    staging; the next calls reallocate and stay bit-exact."""
    rng = np.random.default_rng(9)
    r = rng.integers(0, 500, 40000).astype(np.uint32)
    c = rng.integers(0, 700, 40000).astype(np.uint32)
    v = rng.standard_normal(40000).astype(np.float32)
    wrp, wci, wv = O.ref_from_coo(500, 700, r, c, v)
    a = G.gen_powerlaw(3000, 200000, 2900, 1.0, 12)
    G.randomize_values(a, 13)
    b = G.make_random_dense(3000, 64, 14)
    want, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b.data, "sum")
    for _ in range(2):
        _check(G.DeviceCsr.from_coo(500, 700, *_dev(r, c, v)), wrp, wci, wv)
        got = G.native_spmm(a, b, G.KernelVariant.tuned(), G.ops.sum(),
                            exec=G.ExecOptions(h2d_pack=1))
        assert np.array_equal(got.data.view(np.uint32), want.view(np.uint32))
        G.release_workspace()

"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle.

Bar: bit-exact for every op in exact mode (sum/mean included — each output
element is folded by one thread in CSR order with separate mul/add), arg
indices identical; fast mode (FFMA) sum within 1e-5 of sum|v*b|.
"""
import numpy as np
import pytest

import oracle as O
import paper_2007_03179_b200 as G
from conftest import bits, first_divergence, requires_experimental

pytestmark = pytest.mark.gpu

ALL_VARIANTS = [G.KernelVariant.naive(), G.KernelVariant.crc(), G.KernelVariant.crc_cwm(2),
                G.KernelVariant.crc_cwm(4), G.KernelVariant.crc_cwm(8), G.KernelVariant.tuned()]
OPS = ["sum", "mean", "max", "min"]


def _oracle(a, b, op, want_arg=False, arg_kind=O.ARG_EDGE, skip_tail=False):
    bd = b.data if isinstance(b, G.DenseMatrix) else b
    return O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, bd, op, want_arg=want_arg,
                  arg_kind=arg_kind, skip_tail=skip_tail)


def _inputs(spec):
    a = G.gen_uniform_random(G.GraphGenSpec(spec["rows"], spec["nnz"], spec["gen_seed"],
                                            spec["loops"]))
    G.randomize_values(a, spec["val_seed"])
    b = G.make_random_dense(spec["rows"], spec["n"], spec["b_seed"])
    return a, b


def _powerlaw(rows, nnz, maxdeg, seed, n):
    a = G.gen_powerlaw(rows, nnz, maxdeg, 1.0, seed)
    G.randomize_values(a, seed + 1)
    b = G.make_random_dense(rows, n, seed + 2)
    return a, b


def test_hand_cases_every_variant(golden, golden_npz, cuda):
    for case in golden["hand_cases"]:
        i = case["npz_index"]
        a = G.CsrMatrix(case["m"], case["k"], golden_npz[f"hand{i}_row_ptr"],
                        golden_npz[f"hand{i}_col_ind"], golden_npz[f"hand{i}_vals"])
        b = G.DenseMatrix.of(golden_npz[f"hand{i}_b"])
        want = golden_npz[f"hand{i}_want"]
        for v in ALL_VARIANTS:
            c = G.native_spmm(a, b, v, G.reduce_op_by_name(case["op"]))
            assert first_divergence(c.data, want) is None, (case["name"], v)
            assert G.checksum(c) == case["checksum"]


def test_random_corpus_every_variant(golden, cuda):
    """225 reference-shaped cases x 6 variants, checksum-equal to the reference."""
    for spec in golden["random_corpus"]:
        a, b = _inputs(spec)
        op = G.reduce_op_by_name(spec["op"])
        for v in ALL_VARIANTS:
            c = G.native_spmm(a, b, v, op)
            assert G.checksum(c) == spec["checksum"], (spec, v)


def test_config_checksums(golden, cuda):
    for spec in golden["configs"]:
        a = G.gen_uniform_random(G.GraphGenSpec(spec["rows"], spec["nnz"], spec["gen_seed"]))
        G.randomize_values(a, spec["val_seed"])
        b = G.make_random_dense(spec["rows"], spec["n"], spec["b_seed"])
        op = G.reduce_op_by_name(spec["op"])
        for v in (G.select_variant(spec["n"]), G.KernelVariant.tuned()):
            assert G.checksum(G.native_spmm(a, b, v, op)) == spec["checksum"]


@pytest.mark.parametrize("op", OPS)
def test_new_ops_and_args_every_variant(op, cuda):
    for seed, (rows, nnz, n) in enumerate([(300, 6000, 33), (500, 9000, 128), (97, 900, 5),
                                           (256, 20000, 256), (64, 4000, 500)]):
        a = G.gen_uniform_random(G.GraphGenSpec(rows, nnz, seed + 100))
        G.randomize_values(a, seed + 200)
        b = G.make_random_dense(rows, n, seed + 300)
        want_arg = op in ("max", "min")
        for kind in ((O.ARG_EDGE, O.ARG_COLUMN) if want_arg else (O.ARG_EDGE,)):
            want, warg = _oracle(a, b, op, want_arg, kind)
            ak = "column" if kind == O.ARG_COLUMN else "edge"
            ex = G.ExecOptions(arg_kind=ak)
            runs = [(v, ex) for v in ALL_VARIANTS]
            # every row through the hub kernels too (ring-fed k_hub / LDG k_cta)
            runs.append((G.KernelVariant.tuned(), G.ExecOptions(arg_kind=ak, hub_threshold=1)))
            for v, e in runs:
                c, arg = G.native_spmm_arg(a, b, v, G.reduce_op_by_name(op), exec=e,
                                           want_arg=want_arg)
                assert first_divergence(c.data, want) is None, (op, v, rows, n, e.hub_threshold)
                if want_arg:
                    assert np.array_equal(arg, warg), (op, v, kind, e.hub_threshold)


N_SWEEP = [1, 2, 3, 4, 5, 8, 12, 16, 24, 31, 32, 33, 48, 64, 66, 96, 100, 127, 128, 129, 192,
           256, 260, 500, 512, 513, 1000]


@pytest.mark.parametrize("n", N_SWEEP)
def test_tuned_shapes_over_n(n, cuda):
    """Every (VEC, LPR, CF) shape the tuner can pick, on a power-law matrix."""
    a, b = _powerlaw(700, 30000, 650, n, n)
    for op in ("sum", "max"):
        want, warg = _oracle(a, b, op, op == "max")
        c, arg = G.native_spmm_arg(a, b, G.KernelVariant.tuned(), G.reduce_op_by_name(op),
                                   want_arg=op == "max")
        assert first_divergence(c.data, want) is None, (n, op)
        if op == "max":
            assert np.array_equal(arg, warg)


@pytest.mark.parametrize("n", [30, 32, 64, 96, 128, 130, 200, 256, 512, 520, 1000])
@pytest.mark.parametrize("op", OPS)
def test_hub_rows_row_per_cta(n, op, cuda):
    """Force the row-per-CTA hub kernels (threshold 40): the TMA-ring k_hub when
    N % 4 == 0 (rows spanning many ring rounds, ragged column tiles at 200/520/
    1000), the LDG k_cta otherwise (30, 130); bit-exact (columns split, never
    nonzeros)."""
    a, b = _powerlaw(3000, 150000, 2999, 7, n)
    ex = G.ExecOptions(hub_threshold=40)
    want_arg = op in ("max", "min")
    want, warg = _oracle(a, b, op, want_arg)
    c, arg = G.native_spmm_arg(a, b, G.KernelVariant.tuned(), G.reduce_op_by_name(op), exec=ex,
                               want_arg=want_arg)
    assert first_divergence(c.data, want) is None
    if want_arg:
        assert np.array_equal(arg, warg)


def test_row_length_boundaries(cuda):
    """Rows of length 0, 1, 7-9, 15-17, 31-33, 255-257, 513 and one of 20000
    (chunk edges of every staged-tile geometry: 8 entries per row at 4 and 8
    lanes, 16 and 32 above); N=12/16 run the 4-lane rows."""
    lens = [0, 1, 31, 32, 33, 255, 256, 257, 513, 20000, 0, 7, 8, 9, 15, 16, 17]
    k = 25000
    rng = np.random.default_rng(5)
    rp = np.zeros(len(lens) + 1, np.uint32)
    cols = []
    for i, L in enumerate(lens):
        cols.append(np.sort(rng.choice(k, L, replace=False)).astype(np.uint32))
        rp[i + 1] = rp[i] + L
    a = G.CsrMatrix(len(lens), k, rp, np.concatenate(cols), np.zeros(int(rp[-1]), np.float32))
    G.randomize_values(a, 9)
    for n in (12, 16, 44, 128, 256):
        b = G.make_random_dense(k, n, 3)
        for ht in (0, 30, -1):
            for op in OPS:
                want, warg = _oracle(a, b, op, op in ("max", "min"))
                c, arg = G.native_spmm_arg(a, b, G.KernelVariant.tuned(), G.reduce_op_by_name(op),
                                           exec=G.ExecOptions(hub_threshold=ht),
                                           want_arg=op in ("max", "min"))
                assert first_divergence(c.data, want) is None, (n, ht, op)
                if warg is not None:
                    assert np.array_equal(arg, warg)


def _same_bits_nan_canonical(got, want):
    """Bitwise equality, except that any NaN equals any NaN: the GPU's FMUL/FADD
    emit the canonical NaN (0x7fffffff) where x86 propagates the input payload.
    NaN *positions* must still agree."""
    g, w = bits(got), bits(want)
    gn, wn = np.isnan(got), np.isnan(want)
    return np.array_equal(gn, wn) and np.array_equal(g[~gn], w[~wn])


def test_special_values_nan_inf_signed_zero(cuda):
    """NaN products never enter max/min (strict compare), -inf never beats the
    seed, +0/-0 ties keep the earliest — all exactly as the ordered fold."""
    a = G.gen_uniform_random(G.GraphGenSpec(200, 4000, 3))
    G.randomize_values(a, 4)
    b = G.make_random_dense(200, 64, 5)
    bd = b.data.copy()
    bd[::7, 3] = np.nan
    bd[::5, 4] = -np.inf
    bd[::3, 5] = np.inf
    bd[:, 6] = 0.0
    bd[::2, 7] = -0.0
    bd[1::2, 7] = 0.0
    bs = G.DenseMatrix.of(bd)
    for op in OPS:
        want, warg = _oracle(a, bs, op, op in ("max", "min"))
        for v in ALL_VARIANTS:
            c, arg = G.native_spmm_arg(a, bs, v, G.reduce_op_by_name(op),
                                       want_arg=op in ("max", "min"))
            assert _same_bits_nan_canonical(c.data, want), (op, v)
            if warg is not None:
                assert np.array_equal(arg, warg), (op, v)


def test_empty_shapes_and_errors(golden, cuda):
    # M = 0 -> empty result, no error (native.hpp:109)
    a = G.CsrMatrix.empty(0, 5)
    c = G.native_spmm(a, G.DenseMatrix.zeros(5, 3), G.KernelVariant.tuned(), G.ops.sum())
    assert c.data.shape == (0, 3)
    # all rows empty -> op seeds
    a = G.CsrMatrix.empty(3, 3)
    b = G.make_random_dense(3, 5, 3)
    for v in ALL_VARIANTS:
        assert np.all(G.native_spmm(a, b, v, G.ops.sum()).data == 0.0)
        assert np.all(G.native_spmm(a, b, v, G.ops.max()).data == np.finfo(np.float32).min)
        assert np.all(G.native_spmm(a, b, v, G.ops.min()).data == np.finfo(np.float32).max)
        c, arg = G.native_spmm_arg(a, b, v, G.ops.max(), want_arg=True)
        assert np.all(arg == -1)
    # K = 0
    a = G.CsrMatrix.empty(4, 0)
    c = G.native_spmm(a, G.DenseMatrix.zeros(0, 8), G.KernelVariant.tuned(), G.ops.sum())
    assert np.all(c.data == 0)
    # reference error texts, raised through the device validation
    for case in golden["validation"]:
        a = G.CsrMatrix(case["m"], case["k"], np.array(case["row_ptr"], np.uint32),
                        np.array(case["col_ind"], np.uint32), np.array(case["vals"], np.float32))
        b = G.DenseMatrix.zeros(case["b_rows"], case["n"])
        for v in ALL_VARIANTS:
            if case["error"] is None:
                G.native_spmm(a, b, v, G.ops.sum())
                continue
            with pytest.raises(G.Error) as ei:
                G.native_spmm(a, b, v, G.ops.sum())
            assert str(ei.value) == case["error"], (case["name"], v)
    with pytest.raises(G.Error, match="arg indices"):
        G.native_spmm_arg(G.CsrMatrix.empty(2, 2), G.DenseMatrix.zeros(2, 2),
                          G.KernelVariant.tuned(), G.ops.sum(), want_arg=True)


def test_device_validation_finds_first_violation_in_large_matrix(cuda):
    a = G.gen_uniform_random(G.GraphGenSpec(5000, 200000, 1))
    G.randomize_values(a, 2)
    b = G.make_random_dense(5000, 32, 3)
    for mutate, text in (
        (lambda ci, rp: ci.__setitem__(150000, 7000), "col_ind[150000] = 7000 out of bounds"),
        (lambda ci, rp: ci.__setitem__(int(rp[4000]) + 1, ci[int(rp[4000])]),
         "columns not strictly increasing in row 4000"),
        (lambda ci, rp: rp.__setitem__(2500, rp[2499] - 1), "row_ptr non-decreasing violated at index 2500"),
    ):
        ci, rp = a.col_ind.copy(), a.row_ptr.copy()
        mutate(ci, rp)
        bad = G.CsrMatrix(a.n_rows, a.n_cols, rp, ci, a.vals)
        want_n, want_msg = O.validate(bad.n_rows, bad.n_cols, rp, ci, a.vals)
        assert want_n >= 1 and text in want_msg
        with pytest.raises(G.Error) as ei:
            G.native_spmm(bad, b, G.KernelVariant.tuned(), G.ops.sum())
        assert str(ei.value) == "spmm: matrix is not canonical CSR: " + want_msg


def test_fault_injection_is_detected(cuda):
    """test_kernels.cpp:153-166: SkipTail output differs from the oracle, and
    equals the oracle's own SkipTail restatement (the hook is faithful)."""
    a = G.gen_uniform_random(G.GraphGenSpec(40, 300, 11))
    G.randomize_values(a, 12)
    b = G.make_random_dense(40, 16, 2)
    good, _ = _oracle(a, b, "sum")
    faulty, _ = _oracle(a, b, "sum", skip_tail=True)
    for v in ALL_VARIANTS:
        c = G.native_spmm(a, b, v, G.ops.sum(), exec=G.ExecOptions(fault=G.FaultMode.SkipTail))
        assert first_divergence(c.data, good) is not None
        assert first_divergence(c.data, faulty) is None


def test_fast_mode_within_tolerance(cuda):
    a, b = _powerlaw(2000, 200000, 1999, 3, 128)
    want, _ = _oracle(a, b, "sum")
    absb = G.DenseMatrix.of(np.abs(b.data))
    absa = G.CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, np.abs(a.vals))
    scale, _ = _oracle(absa, absb, "sum")
    for v in ALL_VARIANTS:
        c = G.native_spmm(a, b, v, G.ops.sum(), exec=G.ExecOptions(exact=False))
        err = np.abs(c.data.astype(np.float64) - want)
        assert np.all(err <= 1e-5 * np.maximum(np.abs(want), scale) + 1e-30), v


def test_device_api_plans_and_unaligned_views(cuda):
    import torch
    a, b = _powerlaw(5000, 400000, 4999, 21, 128)
    d = G.DeviceCsr.from_host(a)
    bt = torch.from_numpy(b.data).to(cuda)
    for op in OPS:
        want, warg = _oracle(a, b, op, op in ("max", "min"))
        c, arg = G.spmm(d, bt, op, want_arg=op in ("max", "min"))
        torch.cuda.synchronize()
        assert first_divergence(c.cpu().numpy(), want) is None
        if warg is not None:
            assert np.array_equal(arg.cpu().numpy(), warg)
        plan = G.Plan(d, 128, op)
        assert plan.launches >= 1 and "tuned" in plan.description
        c2 = torch.empty_like(c)
        a2 = torch.empty_like(arg) if arg is not None else None
        for _ in range(2):
            plan.execute(bt, c2, a2)
        torch.cuda.synchronize()
        assert torch.equal(c2, c)
        plan.close()
    # B / C not 16-byte aligned -> scalar-lane fallback shape, same bits
    buf = torch.empty(b.data.size + 1, dtype=torch.float32, device=cuda)
    bview = buf[1:].view(b.data.shape)
    bview.copy_(bt)
    out = torch.empty(a.n_rows * 128 + 1, dtype=torch.float32, device=cuda)[1:].view(a.n_rows, 128)
    c, _ = G.spmm(d, bview, "sum", out=out)
    torch.cuda.synchronize()
    want, _ = _oracle(a, b, "sum")
    assert first_divergence(c.cpu().numpy(), want) is None


@requires_experimental
@pytest.mark.parametrize("n", [64, 128, 256])
def test_hot_column_map_keeps_bits(n, cuda):
    """The frequency-aware L2 map only changes cache hints: forced on (tiny
    budget, so most columns are cold and carry the bit-31 mark through the row
    cache), every op, edge and column args, is bit-identical to the oracle."""
    import torch
    a, b = _powerlaw(6000, 500000, 5000, 31, n)
    d = G.DeviceCsr.from_host(a)
    bt = torch.from_numpy(b.data).to(cuda)
    for op in OPS:
        want_arg = op in ("max", "min")
        for kind, okind in (("edge", O.ARG_EDGE), ("column", O.ARG_COLUMN)):
            if kind == "column" and not want_arg:
                continue
            want, warg = _oracle(a, b, op, want_arg, arg_kind=okind)
            ex = G.ExecOptions(l2_hot_mb=1, arg_kind=kind)
            plan = G.Plan(d, n, op, exec=ex)
            assert "hot map" in plan.description, plan.description
            c = torch.empty((a.n_rows, n), dtype=torch.float32, device=cuda)
            arg = torch.empty((a.n_rows, n), dtype=torch.int32, device=cuda) if want_arg else None
            plan.execute(bt, c, arg)
            torch.cuda.synchronize()
            assert first_divergence(c.cpu().numpy(), want) is None, (op, kind)
            if want_arg:
                assert np.array_equal(arg.cpu().numpy(), warg), (op, kind)
            plan.close()


@requires_experimental
@pytest.mark.parametrize("n", [64, 128, 256, 130])
def test_relocated_hot_rows_keep_bits(n, cuda):
    """Relocated hot rows (hot_rows_mb): the plan gathers the most-gathered
    B rows from its own copy through a remapped col_ind; positions and fold
    order are unchanged, so every op is bit-identical to the oracle, also after
    B moves and changes (the copy is re-placed and refreshed per execute) and
    with hub rows (which gather B through the caller's col_ind)."""
    import torch
    a, b = _powerlaw(6000, 500000, 5000, 37, n)
    d = G.DeviceCsr.from_host(a)
    for op in OPS:
        want_arg = op in ("max", "min")
        plan = G.Plan(d, n, op, exec=G.ExecOptions(hot_rows_mb=1, hub_threshold=2000))
        assert "relocated hot rows" in plan.description, plan.description
        for seed in (0, 1):
            bb = b.data if seed == 0 else -b.data[::-1].copy()
            bt = torch.from_numpy(np.ascontiguousarray(bb)).to(cuda)
            want, warg = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, bb, op,
                                want_arg=want_arg)
            c = torch.empty((a.n_rows, n), dtype=torch.float32, device=cuda)
            arg = torch.empty((a.n_rows, n), dtype=torch.int32, device=cuda) if want_arg else None
            plan.execute(bt, c, arg)
            torch.cuda.synchronize()
            assert first_divergence(c.cpu().numpy(), want) is None, (op, n, seed)
            if want_arg:
                assert np.array_equal(arg.cpu().numpy(), warg), (op, n, seed)
        plan.close()


def test_device_validate_flag(cuda):
    import torch
    a = G.gen_uniform_random(G.GraphGenSpec(100, 1000, 1))
    ci = a.col_ind.copy()
    ci[10] = 1000
    d = G.DeviceCsr.from_host(G.CsrMatrix(100, 100, a.row_ptr, ci, a.vals))
    b = torch.zeros(100, 8, device=cuda)
    with pytest.raises(G.Error, match="out of bounds"):
        G.spmm(d, b, "sum", validate=True)


def _sub_rows(a, rows):
    """CSR of a subset of rows (same columns) for oracle checks at scale."""
    rp = a.row_ptr.astype(np.int64)
    lens = rp[rows + 1] - rp[rows]
    idx = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows])
    sub = G.CsrMatrix(len(rows), a.n_cols, np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32),
                      a.col_ind[idx], a.vals[idx])
    return sub, idx


@pytest.mark.slow
def test_reddit_scale_sum_sampled_rows_and_cross_kernel(cuda):
    """Reddit shape (232,965 rows, 114.8M nnz, N=128): tuned output equals the
    paper's crc-cwm(2) kernel bit-for-bit over the whole matrix, and the oracle on
    every hub row plus 3000 random rows."""
    import torch
    a = G.gen_powerlaw(232965, 114_800_000, 21657, 1.0, 1)
    G.randomize_values(a, 2)
    b = G.make_random_dense(a.n_cols, 128, 42)
    d = G.DeviceCsr.from_host(a)
    bt = torch.from_numpy(b.data).to(cuda)
    c_tuned, _ = G.spmm(d, bt, "sum")
    c_cwm, _ = G.spmm(d, bt, "sum", variant=G.KernelVariant.crc_cwm(2))
    torch.cuda.synchronize()
    assert torch.equal(c_tuned.view(torch.int32), c_cwm.view(torch.int32))
    deg = np.diff(a.row_ptr.astype(np.int64))
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([np.argsort(-deg)[:200], rng.choice(a.n_rows, 3000, False)]))
    sub, _ = _sub_rows(a, rows)
    want, _ = _oracle(sub, b, "sum")
    got = c_tuned[torch.from_numpy(rows).to(cuda)].cpu().numpy()
    assert first_divergence(got, want) is None


@pytest.mark.slow
def test_products_scale_max_arg_sampled_rows(cuda):
    """ogbn-products shape (2.45M rows, 123.7M nnz), N=256 max + argmax."""
    import torch
    a = G.gen_powerlaw(2_449_029, 123_718_280, 17481, 1.0, 1)
    G.randomize_values(a, 2)
    b = G.make_random_dense(a.n_cols, 256, 42)
    d = G.DeviceCsr.from_host(a)
    bt = torch.from_numpy(b.data).to(cuda)
    c, arg = G.spmm(d, bt, "max", want_arg=True)
    torch.cuda.synchronize()
    deg = np.diff(a.row_ptr.astype(np.int64))
    rng = np.random.default_rng(1)
    rows = np.unique(np.concatenate([np.argsort(-deg)[:100], rng.choice(a.n_rows, 2000, False)]))
    sub, idx = _sub_rows(a, rows)
    want, warg = _oracle(sub, b, "max", True)
    sel = torch.from_numpy(rows).to(cuda)
    assert first_divergence(c[sel].cpu().numpy(), want) is None
    got_arg = arg[sel].cpu().numpy()
    # oracle positions are within the sub-CSR; map back to global CSR positions
    mapped = np.where(warg >= 0, idx[np.maximum(warg, 0)], -1)
    assert np.array_equal(got_arg, mapped)


@requires_experimental
@pytest.mark.parametrize("slices", [2, 3, 8])
@pytest.mark.parametrize("n", [64, 100, 256])
def test_column_slices_keep_bits(slices, n, cuda):
    """Slice-major traversal (col_slices) only reorders which columns of B are
    live; every op with edge args stays bit-identical, incl. ragged last slices
    and the hub kernel (threshold forced low)."""
    a, b = _powerlaw(3000, 120000, 2500, 11 + n, n)
    for op in OPS:
        want_arg = op in ("max", "min")
        want, warg = _oracle(a, b, op, want_arg)
        for ht in (0, 300):
            ex = G.ExecOptions(col_slices=slices, hub_threshold=ht)
            c, arg = G.native_spmm_arg(a, b, G.KernelVariant.tuned(), G.reduce_op_by_name(op),
                                       exec=ex, want_arg=want_arg)
            assert first_divergence(c.data, want) is None, (op, ht)
            if want_arg:
                assert np.array_equal(arg, warg), (op, ht)


@pytest.mark.parametrize("rpw", [2, 4, 8])
@pytest.mark.parametrize("n", [32, 64, 100, 128, 200, 256])
def test_rows_per_warp_shapes_keep_bits(rpw, n, cuda):
    """Multi-row warp shapes for low-degree matrices ((4,4,2) ... (4,16,4)): every
    op with args, bit-identical, incl. ragged N and power-law rows spanning many
    chunks (degree-sorted schedule) and low-degree rows (identity schedule)."""
    pl = _powerlaw(3000, 60000, 2000, 17 + n, n)
    un = G.gen_uniform_random(G.GraphGenSpec(5000, 20000, 7))
    G.randomize_values(un, 8)
    for a, b in (pl, (un, G.make_random_dense(5000, n, 9))):
        for op in OPS:
            want_arg = op in ("max", "min")
            want, warg = _oracle(a, b, op, want_arg)
            ex = G.ExecOptions(rows_per_warp=rpw)
            c, arg = G.native_spmm_arg(a, b, G.KernelVariant.tuned(), G.reduce_op_by_name(op),
                                       exec=ex, want_arg=want_arg)
            assert first_divergence(c.data, want) is None, (op, a.n_rows)
            if want_arg:
                assert np.array_equal(arg, warg), (op, a.n_rows)


@pytest.mark.parametrize("share", ["small", "large"])
@pytest.mark.parametrize("op", OPS)
def test_hub_launch_modes_keep_bits(share, op, cuda):
    """Hub rows carrying < 25% of the nonzeros run on the high-priority side
    stream next to the warp kernel; >= 25% run first on the same stream with
    the warp kernel as a programmatic dependent launch.  Both bit-exact, device
    plans and the pipelined host entry."""
    import torch
    a, b = _powerlaw(6000, 400000, 5000, 29, 128)
    deg = np.sort(np.diff(a.row_ptr.astype(np.int64)))[::-1]
    cum = np.cumsum(deg) / deg.sum()
    # threshold = degree of the row where the hub share crosses ~10% / ~60%
    target = 0.10 if share == "small" else 0.60
    thr = int(deg[int(np.searchsorted(cum, target))])
    hub_share = deg[deg >= thr].sum() / deg.sum()
    assert (hub_share < 0.25) if share == "small" else (hub_share >= 0.25)
    want_arg = op in ("max", "min")
    want, warg = _oracle(a, b, op, want_arg)
    ex = G.ExecOptions(hub_threshold=thr)
    c, arg = G.native_spmm_arg(a, b, G.KernelVariant.tuned(), G.reduce_op_by_name(op), exec=ex,
                               want_arg=want_arg)
    assert first_divergence(c.data, want) is None
    if want_arg:
        assert np.array_equal(arg, warg)
    d = G.DeviceCsr.from_host(a, cuda)
    bt = torch.from_numpy(b.data).to(cuda)
    plan = G.Plan(d, 128, op, exec=ex)
    assert f"hub_rows={int((np.diff(a.row_ptr.astype(np.int64)) >= thr).sum())}" in plan.description
    c2 = torch.empty((a.n_rows, 128), device=cuda)
    a2 = torch.empty((a.n_rows, 128), dtype=torch.int32, device=cuda) if want_arg else None
    for _ in range(3):  # repeated launches reuse the persistent-launch counters
        plan.execute(bt, c2, a2)
    torch.cuda.synchronize()
    assert first_divergence(c2.cpu().numpy(), want) is None
    if want_arg:
        assert np.array_equal(a2.cpu().numpy(), warg)
    plan.close()


@pytest.mark.parametrize("n", [64, 128, 130])
def test_fault_injection_through_hub_kernels(n, cuda):
    """SkipTail through the hub kernels (ring-fed k_hub at N % 4 == 0, k_cta at
    130): equal to the oracle's SkipTail restatement, different from the good
    result."""
    a, b = _powerlaw(2000, 80000, 1500, 41, n)
    good, _ = _oracle(a, b, "sum")
    faulty, _ = _oracle(a, b, "sum", skip_tail=True)
    ex = G.ExecOptions(fault=G.FaultMode.SkipTail, hub_threshold=100)
    c = G.native_spmm(a, b, G.KernelVariant.tuned(), G.ops.sum(), exec=ex)
    assert first_divergence(c.data, good) is not None
    assert first_divergence(c.data, faulty) is None


@requires_experimental
@pytest.mark.parametrize("cs", [2, 8, 16])
@pytest.mark.parametrize("op", OPS)
def test_cluster_dsmem_hot_rows_keep_bits(cs, op, cuda):
    """cluster_hot: the most-gathered B rows live in the distributed shared
    memory of CS-CTA clusters and hot gathers go over DSMEM (remapped col_ind);
    every op with edge and column args bit-identical, repeated launches."""
    import torch
    a, b = _powerlaw(20000, 1500000, 9000, 51, 128)
    want_arg = op in ("max", "min")
    d = G.DeviceCsr.from_host(a, cuda)
    bt = torch.from_numpy(b.data).to(cuda)
    for arg_kind in (("edge", "column") if want_arg else ("edge",)):
        want, warg = _oracle(a, b, op, want_arg,
                             arg_kind=O.ARG_COLUMN if arg_kind == "column" else O.ARG_EDGE)
        plan = G.Plan(d, 128, op, exec=G.ExecOptions(cluster_hot=cs, arg_kind=arg_kind))
        assert "cluster DSMEM cache" in plan.description, plan.description
        c = torch.empty((a.n_rows, 128), device=cuda)
        arg = torch.empty((a.n_rows, 128), dtype=torch.int32, device=cuda) if want_arg else None
        for _ in range(2):
            c.fill_(-1.0)
            plan.execute(bt, c, arg)
            torch.cuda.synchronize()
            assert first_divergence(c.cpu().numpy(), want) is None, (cs, op, arg_kind)
            if want_arg:
                assert np.array_equal(arg.cpu().numpy(), warg), (cs, op, arg_kind)
        plan.close()


def _gappy(rows, k, per_row, seed, far_every=0):
    """Sorted random rows over k columns; with far_every, every far_every-th
    row also gets a column near k (a gap >= 65535: an escape code)."""
    rng = np.random.default_rng(seed)
    rp = np.zeros(rows + 1, np.uint32)
    cols = []
    for r in range(rows):
        c = np.sort(rng.choice(k, per_row, replace=False)).astype(np.uint32)
        if far_every and r % far_every == 0:
            c = np.unique(np.concatenate([c, [k - 1 - (r % 7)]])).astype(np.uint32)
        cols.append(c)
        rp[r + 1] = rp[r] + len(c)
    a = G.CsrMatrix(rows, k, rp, np.concatenate(cols), np.zeros(int(rp[-1]), np.float32))
    G.randomize_values(a, seed + 1)
    return a


@pytest.mark.parametrize("kind", ["powerlaw", "uniform", "escapes", "raw_fallback"])
@pytest.mark.parametrize("op", ["sum", "max"])
def test_packed_upload_keeps_bits(kind, op, cuda):
    """Host entry with the col_ind upload as 16-bit gap codes (h2d_pack=1):
    rebuilt on the device by a segmented scan, bit-identical results; escape
    codes for gaps >= 65535 (every 10th row of "escapes"), and blocks with too
    many escapes sent raw ("raw_fallback": gaps ~75k everywhere)."""
    if kind == "powerlaw":
        a = G.gen_powerlaw(6000, 300000, 3000, 1.0, 71)
        G.randomize_values(a, 72)
    elif kind == "uniform":
        a = G.gen_uniform_random(G.GraphGenSpec(8000, 120000, 73))
        G.randomize_values(a, 74)
    elif kind == "escapes":
        a = _gappy(4000, 100_000, 50, 75, far_every=10)
    else:
        a = _gappy(300, 3_000_000, 40, 76)
    b = G.make_random_dense(a.n_cols, 32, 79)
    want, warg = _oracle(a, b, op, op == "max")
    for v in (G.KernelVariant.tuned(), G.KernelVariant.crc_cwm(2)):
        for pack in (1, -1):
            c, arg = G.native_spmm_arg(a, b, v, G.reduce_op_by_name(op),
                                       exec=G.ExecOptions(h2d_pack=pack), want_arg=op == "max")
            assert first_divergence(c.data, want) is None, (kind, pack, v)
            if op == "max":
                assert np.array_equal(arg, warg), (kind, pack, v)


def test_packed_upload_reports_the_same_violations(cuda):
    """Non-canonical inputs travel losslessly (escapes), so the device check
    reports the reference's first violation whether or not the upload is packed."""
    a = G.gen_uniform_random(G.GraphGenSpec(3000, 60000, 81))
    G.randomize_values(a, 82)
    b = G.make_random_dense(3000, 16, 83)
    rp = a.row_ptr.astype(np.int64)
    cases = []
    bad = a.col_ind.copy(); p = int(rp[1500]) + 3; bad[p] = bad[p - 1]          # duplicate
    cases.append(bad)
    bad = a.col_ind.copy(); p = int(rp[2000]) + 2; bad[p], bad[p + 1] = bad[p + 1], bad[p]  # swap
    cases.append(bad)
    bad = a.col_ind.copy(); bad[int(rp[2500]) + 1] = 3000 + 70000                # out of range
    cases.append(bad)
    for ci in cases:
        m = G.CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, ci, a.vals)
        msgs = []
        for pack in (1, -1):
            with pytest.raises(G.Error) as ei:
                G.native_spmm(m, b, G.KernelVariant.tuned(), G.ops.sum(),
                              exec=G.ExecOptions(h2d_pack=pack))
            msgs.append(str(ei.value))
        assert msgs[0] == msgs[1] and "not canonical" in msgs[0]
        want_n, want_msg = O.validate(m.n_rows, m.n_cols, m.row_ptr, m.col_ind, m.vals)
        assert msgs[0] == "spmm: matrix is not canonical CSR: " + want_msg


@pytest.mark.parametrize("ht", [0, 300, -1])
def test_plan_execute_is_graph_capturable(ht, cuda):
    """A plan's execute captured into a CUDA graph and replayed (the GNN-layer
    pattern): hub kernel ahead of the warp kernel as a programmatic dependent
    launch (ht=300), side stream, or warp kernel alone; replays bit-exact, with
    a changed B between replays."""
    import torch
    a, b = _powerlaw(5000, 300000, 4000, 91, 128)
    d = G.DeviceCsr.from_host(a, cuda)
    bt = torch.from_numpy(b.data).to(cuda)
    c = torch.empty((a.n_rows, 128), device=cuda)
    plan = G.Plan(d, 128, "sum", exec=G.ExecOptions(hub_threshold=ht))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.execute(bt, c, stream=s)  # warm-up: policies resolved, attributes set
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plan.execute(bt, c)
    for seed in (92, 93):
        b2 = G.make_random_dense(a.n_cols, 128, seed)
        bt.copy_(torch.from_numpy(b2.data))
        c.fill_(-1.0)
        g.replay()
        torch.cuda.synchronize()
        want, _ = _oracle(a, b2, "sum")
        assert first_divergence(c.cpu().numpy(), want) is None, (ht, seed)
    plan.close()


@pytest.mark.slow
def test_reddit_scale_host_entry_and_shards_equal_device_plan(cuda):
    """Reddit shape, N=128 sum, whole matrix: (1) the pipelined host entry
    (packed col_ind upload, 12 row blocks, block-level hub rows) and (2) the 8
    nnz-balanced row shards of the multi-GPU path (hub rows through k_hub ahead
    of the warp kernel) are both bit-identical to the single device plan."""
    import torch
    from paper_2007_03179_b200 import dist as D
    a = G.gen_powerlaw(232965, 114_800_000, 21657, 1.0, 1)
    G.randomize_values(a, 2)
    b = G.make_random_dense(a.n_cols, 128, 42)
    d = G.DeviceCsr.from_host(a)
    bt = torch.from_numpy(b.data).to(cuda)
    full, _ = G.spmm(d, bt, "sum")
    torch.cuda.synchronize()
    want = full.cpu().numpy()
    c_host = G.native_spmm(a, b, G.KernelVariant.tuned(), G.ops.sum())
    assert first_divergence(c_host.data, want) is None
    bounds = D.partition_rows(a.row_ptr, 8)
    hubs = 0
    for r in range(8):
        sh = D.shard_csr(a, bounds[r], bounds[r + 1])
        plan = G.Plan(G.DeviceCsr.from_host(sh, cuda), 128, "sum")
        hubs += int(plan.description.split("hub_rows=")[1].split(" ")[0])
        c = torch.empty((sh.n_rows, 128), device=cuda)
        plan.execute(bt, c)
        torch.cuda.synchronize()
        assert first_divergence(c.cpu().numpy(), want[bounds[r]:bounds[r + 1]]) is None, r
        plan.close()
    assert hubs > 0  # the shards really went through the hub kernel


@pytest.mark.slow
def test_reddit_scale_hub_threshold_by_width(cuda):
    """The auto hub threshold on the whole Reddit shape: no hub rows at N=128
    (the longest row fits inside the byte-bound launch) and only the very
    longest rows at narrow widths, whose launch is bound per nonzero rather
    than per byte (N=32 took 3.1 ms with ~2600 hub rows, 1.44 ms with the
    per-nonzero floor; profiles/r1_narrow_widths_*.txt).  A sampled row check
    keeps the narrow hub path honest."""
    import torch
    a = G.gen_powerlaw(232965, 114_800_000, 21657, 1.0, 1)
    G.randomize_values(a, 2)
    d = G.DeviceCsr.from_host(a, cuda)

    def hub_rows(desc):
        return int(desc.split("hub_rows=")[1].split(" ")[0])

    p128 = G.Plan(d, 128, "sum")
    assert hub_rows(p128.description) == 0
    p128.close()
    b = G.make_random_dense(a.n_cols, 32, 42)
    bt = torch.from_numpy(b.data).to(cuda)
    p32 = G.Plan(d, 32, "sum")
    h = hub_rows(p32.description)
    assert 0 < h < 2000, p32.description  # deg >= ~10k: the ring-first threshold (alpha rule)
    c = torch.empty((a.n_rows, 32), device=cuda)
    p32.execute(bt, c)
    torch.cuda.synchronize()
    got = c.cpu().numpy()
    p32.close()
    deg = np.diff(a.row_ptr.astype(np.int64))
    rows = np.concatenate([np.argsort(-deg)[:8], np.random.default_rng(5).integers(0, a.n_rows, 24)])
    for r in rows:
        lo, hi = int(a.row_ptr[r]), int(a.row_ptr[r + 1])
        want = np.zeros(32, np.float32)
        for p in range(lo, hi):  # ordered fold v*b then add, as the reference
            want = (want + np.float32(a.vals[p]) * b.data[a.col_ind[p]]).astype(np.float32)
        assert np.array_equal(got[r], want), int(r)


def test_plan_and_spmm_refuse_bad_operands(cuda):
    """Raw pointers reach the kernels only for tensors of exactly the plan's
    shape, dtype, device and layout (no silent out-of-bounds writes)."""
    import torch
    a = G.gen_powerlaw(500, 8000, 400, 1.0, 3)
    G.randomize_values(a, 4)
    d = G.DeviceCsr.from_host(a, cuda)
    p = G.Plan(d, 64, "max")
    b = torch.zeros((500, 64), device=cuda)
    c = torch.empty((500, 64), device=cuda)
    arg = torch.empty((500, 64), dtype=torch.int32, device=cuda)
    p.execute(b, c, arg)
    bad = [
        (torch.zeros((500, 128), device=cuda)[:, :64], c, arg),      # non-contiguous B
        (torch.zeros((499, 64), device=cuda), c, arg),              # short B
        (b, torch.empty((499, 64), device=cuda), arg),              # short C
        (b, torch.empty((500, 64), dtype=torch.float64, device=cuda), arg),
        (b, c, torch.empty((500, 64), dtype=torch.int64, device=cuda)),
        (b.cpu(), c, arg),
    ]
    for bb, cc, aa in bad:
        with pytest.raises(G.Error):
            p.execute(bb, cc, aa)
    with pytest.raises(G.Error):
        G.spmm(d, b, "sum", out=torch.empty((10, 64), device=cuda))
    p.close()


@pytest.mark.slow
def test_experimental_build_suite(cuda):
    """The measured-slower options ship only in libgespmm_exp.so: run their
    parity tests (and the option fuzzers) against that build in a subprocess."""
    import os
    import subprocess
    import sys
    import paper_2007_03179_b200._lib as L
    exp = os.path.join(os.path.dirname(L.__file__), "libgespmm_exp.so")
    if L.experimental_built():
        pytest.skip("this process already runs the experimental build")
    if not os.path.exists(exp):
        pytest.skip("libgespmm_exp.so not built")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GESPMM_EXPERIMENTAL="1", FUZZ_EXAMPLES="25")
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m",
                          "gpu and experimental", "tests/test_gpu_parity.py",
                          "tests/test_gpu_fuzz.py", "tests/test_gpu_peer.py"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=1500)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert " passed" in out.stdout

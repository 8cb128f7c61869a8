"""GPU: randomized parity sweep (hypothesis, fixed seed, bounded examples).
Random canonical CSR shapes (empty rows, single-entry rows, a long row),
random N (odd and even, 1..300), every op with edge/column args, every
kernel variant and the tuned path's options (hub threshold, rows per warp,
column slices, packed upload); exact mode must equal the oracle bit for bit."""
import os

import numpy as np
import pytest
from hypothesis import HealthCheck, given, seed, settings
from hypothesis import strategies as st

import oracle as O
import paper_2007_03179_b200 as G
from conftest import experimental_built, first_divergence

pytestmark = pytest.mark.gpu
# the option fuzzers also run against libgespmm_exp.so
# (test_gpu_parity::test_experimental_build_suite), drawing its options there
EXPERIMENTAL = experimental_built()


def _matrix(rng, m, k, density, long_row):
    rp = [0]
    cols = []
    for r in range(m):
        d = int(rng.binomial(k, density))
        if long_row and r == m // 2:
            d = k
        c = np.sort(rng.choice(k, size=min(d, k), replace=False)) if d else np.zeros(0, np.int64)
        cols.append(c.astype(np.uint32))
        rp.append(rp[-1] + len(c))
    ci = np.concatenate(cols) if cols else np.zeros(0, np.uint32)
    a = G.CsrMatrix(m, k, np.asarray(rp, np.uint32), ci, np.zeros(len(ci), np.float32))
    G.randomize_values(a, int(rng.integers(1 << 30)))
    return a


VARIANTS = [G.KernelVariant.tuned(), G.KernelVariant.naive(), G.KernelVariant.crc(),
            G.KernelVariant.crc_cwm(2), G.KernelVariant.crc_cwm(4), G.KernelVariant.crc_cwm(8)]


@pytest.mark.experimental
@seed(20261017)
@settings(max_examples=int(os.environ.get("FUZZ_EXAMPLES", "60")), deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(m=st.integers(0, 300), k=st.integers(1, 400), density=st.floats(0.0, 0.3),
       long_row=st.booleans(), n=st.integers(1, 300), op=st.sampled_from(["sum", "mean", "max", "min"]),
       column_arg=st.booleans(), vi=st.integers(0, len(VARIANTS) - 1),
       hub=st.sampled_from([0, 1, 5, -1]), rpw=st.sampled_from([0, 1, 2, 4]),
       slices=st.sampled_from([0, 1, 2, 3]), pack=st.sampled_from([0, 1, -1]),
       data=st.integers(0, 1 << 30))
def test_random_shapes_every_path_bit_exact(m, k, density, long_row, n, op, column_arg, vi, hub,
                                            rpw, slices, pack, data):
    if not EXPERIMENTAL:
        slices = min(slices, 1)
    if os.environ.get("FUZZ_LOG"):  # a CUDA fault poisons the context: log before running
        with open(os.environ["FUZZ_LOG"], "a") as f:
            f.write(repr(dict(m=m, k=k, density=density, long_row=long_row, n=n, op=op,
                              column_arg=column_arg, vi=vi, hub=hub, rpw=rpw, slices=slices,
                              pack=pack, data=data)) + "\n")
    rng = np.random.default_rng(data)
    a = _matrix(rng, m, k, density, long_row)
    b = G.make_random_dense(k, n, data + 1)
    want_arg = op in ("max", "min")
    kind = O.ARG_COLUMN if column_arg else O.ARG_EDGE
    want, warg = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b.data, op,
                        want_arg=want_arg, arg_kind=kind)
    ex = G.ExecOptions(arg_kind="column" if column_arg else "edge", hub_threshold=hub,
                       rows_per_warp=rpw, col_slices=slices, h2d_pack=pack)
    try:
        c, arg = G.native_spmm_arg(a, b, VARIANTS[vi], G.reduce_op_by_name(op), exec=ex,
                                   want_arg=want_arg)
    except G.Error as e:
        if os.environ.get("FUZZ_LOG"):
            with open(os.environ["FUZZ_LOG"], "a") as f:
                f.write(f"FAIL {e}\n")
        raise
    assert first_divergence(c.data, want) is None
    if want_arg:
        assert np.array_equal(arg, warg)


@pytest.mark.experimental
@seed(20261018)
@settings(max_examples=int(os.environ.get("FUZZ_EXAMPLES", "60")), deadline=None,
          suppress_health_check=[HealthCheck.too_slow])
@given(m=st.integers(1, 400), k=st.integers(1, 600), density=st.floats(0.0, 0.2),
       long_row=st.booleans(), n=st.one_of(st.integers(1, 300), st.integers(500, 1100)),
       op=st.sampled_from(["sum", "mean", "max", "min"]), column_arg=st.booleans(),
       hub=st.sampled_from([0, 1, 7, -1]), rpw=st.sampled_from([0, 1, 2, 4, 8]),
       slices=st.sampled_from([0, 1, 2, 5]), tuned_cf=st.sampled_from([0, 1, 2, 4]),
       hot=st.sampled_from([0, 1]), replicas=st.sampled_from([1, 1, 3]),
       misalign=st.booleans(), exact=st.sampled_from([True, True, False]),
       cluster=st.sampled_from([0, 0, 0, 2, 8]), overlap=st.booleans(),
       data=st.integers(0, 1 << 30))
def test_random_device_plans_bit_exact(m, k, density, long_row, n, op, column_arg, hub, rpw, slices,
                                       tuned_cf, hot, replicas, misalign, exact, cluster, overlap,
                                       data):
    """Device plans (tuned) over random shapes and options, executed plain or
    with the fused all-gather epilogue into extra replicas; B/C based 4 bytes
    off 16-byte alignment (scalar fallbacks); the cluster-DSMEM cache at N=128;
    fast mode (FFMA) for sum/mean within the documented tolerance."""
    import torch
    if not EXPERIMENTAL:
        slices, hot, cluster = min(slices, 1), 0, 0
    if cluster and n != 128:
        n = 128
    if os.environ.get("FUZZ_LOG"):
        with open(os.environ["FUZZ_LOG"], "a") as f:
            f.write(repr(dict(plan=1, m=m, k=k, density=density, long_row=long_row, n=n, op=op,
                              column_arg=column_arg, hub=hub, rpw=rpw, slices=slices,
                              tuned_cf=tuned_cf, hot=hot, replicas=replicas, misalign=misalign,
                              exact=exact, cluster=cluster, overlap=overlap, data=data)) + "\n")
    rng = np.random.default_rng(data)
    a = _matrix(rng, m, k, density, long_row)
    b = G.make_random_dense(k, n, data + 1)
    want_arg = op in ("max", "min")
    kind = O.ARG_COLUMN if column_arg else O.ARG_EDGE
    want, warg = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b.data, op,
                        want_arg=want_arg, arg_kind=kind)
    dev = torch.device("cuda:0")
    d = G.DeviceCsr.from_host(a, dev)
    sh = 1 if misalign else 0

    def buf(shape, fill, dtype=torch.float32):  # optionally 4 bytes past 16-byte alignment
        flat = torch.full((shape[0] * shape[1] + sh,), fill, dtype=dtype, device=dev)
        return flat[sh:].view(shape)
    bt = buf((k, n), 0.0)
    bt.copy_(torch.from_numpy(b.data))
    fast = not exact and op in ("sum", "mean")
    ex = G.ExecOptions(arg_kind="column" if column_arg else "edge", hub_threshold=hub,
                       rows_per_warp=rpw, col_slices=slices, tuned_cf=tuned_cf, l2_hot_mb=hot,
                       exact=not fast, cluster_hot=cluster, overlap_prev=overlap)
    plan = G.Plan(d, n, op, exec=ex)
    cs = [buf((m, n), -3.0) for _ in range(replicas)]
    args = [buf((m, n), -5, torch.int32) for _ in range(replicas)] if want_arg else None
    try:
        if replicas == 1:
            plan.execute(bt, cs[0], args[0] if args else None)
        else:
            plan.execute_gather(bt, [c.data_ptr() for c in cs],
                                [x.data_ptr() for x in args] if args else None)
        torch.cuda.synchronize()
    except G.Error as e:
        if os.environ.get("FUZZ_LOG"):
            with open(os.environ["FUZZ_LOG"], "a") as f:
                f.write(f"FAIL {e}\n")
        raise
    if fast:  # |delta| <= 1e-5 * max(|want|, sum |v * b|)
        mag, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, np.abs(a.vals),
                        np.abs(b.data), "sum")
        if op == "mean":
            deg = np.maximum(np.diff(a.row_ptr.astype(np.int64)), 1).astype(np.float32)
            mag = mag / deg[:, None]
        for i in range(replicas):
            got = cs[i].cpu().numpy()
            assert np.all(np.abs(got - want) <= 1e-5 * np.maximum(np.abs(want), mag) + 1e-30), i
    else:
        for i in range(replicas):
            assert first_divergence(cs[i].cpu().numpy(), want) is None, i
            if want_arg:
                assert np.array_equal(args[i].cpu().numpy(), warg), i
    plan.close()


@seed(20261019)
@settings(max_examples=int(os.environ.get("FUZZ_EXAMPLES", "60")), deadline=None,
          suppress_health_check=[HealthCheck.too_slow])
@given(m=st.integers(2, 300), k=st.integers(2, 3000), density=st.floats(0.01, 0.2),
       faults=st.lists(st.tuples(st.sampled_from(["oob", "dup", "swap", "big"]),
                                 st.floats(0.0, 1.0)), min_size=1, max_size=4),
       pack=st.sampled_from([1, -1]), data=st.integers(0, 1 << 30))
def test_random_violations_report_the_reference_message(m, k, density, faults, pack, data):
    """Random non-canonical inputs through the host entry (packed upload on or
    off): the error is the reference's first-violation message, or the result
    is correct when the corruption happened to keep the matrix canonical."""
    if os.environ.get("FUZZ_LOG"):
        with open(os.environ["FUZZ_LOG"], "a") as f:
            f.write(repr(dict(viol=1, m=m, k=k, density=density, faults=faults, pack=pack,
                              data=data)) + "\n")
    rng = np.random.default_rng(data)
    a = _matrix(rng, m, k, density, False)
    if a.nnz() < 2:
        return
    ci = a.col_ind.copy()
    for kind, where in faults:
        p = min(int(where * a.nnz()), a.nnz() - 1)
        if kind == "oob":
            ci[p] = k + int(rng.integers(0, 100000))
        elif kind == "big":
            ci[p] = np.uint32(0xFFFFFFF0)
        elif kind == "dup" and p > 0:
            ci[p] = ci[p - 1]
        elif kind == "swap" and p > 0:
            ci[p - 1], ci[p] = ci[p], ci[p - 1]
    bad = G.CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, ci, a.vals)
    b = G.make_random_dense(k, 8, data + 1)
    n_viol, msg = O.validate(bad.n_rows, bad.n_cols, bad.row_ptr, bad.col_ind, bad.vals)
    if n_viol == 0:
        c = G.native_spmm(bad, b, G.KernelVariant.tuned(), G.ops.sum(),
                          exec=G.ExecOptions(h2d_pack=pack))
        want, _ = O.spmm(bad.n_rows, bad.n_cols, bad.row_ptr, bad.col_ind, bad.vals, b.data, "sum")
        assert first_divergence(c.data, want) is None
        return
    with pytest.raises(G.Error) as ei:
        G.native_spmm(bad, b, G.KernelVariant.tuned(), G.ops.sum(),
                      exec=G.ExecOptions(h2d_pack=pack))
    assert str(ei.value) == "spmm: matrix is not canonical CSR: " + msg
    # the device entry with validate=1 checks before any kernel runs
    import torch
    d = G.DeviceCsr.from_host(bad, torch.device("cuda:0"))
    with pytest.raises(G.Error) as ei:
        G.spmm(d, torch.from_numpy(b.data).cuda(), "sum", validate=True)
    assert str(ei.value) == "spmm: matrix is not canonical CSR: " + msg


@seed(20261020)
@settings(max_examples=int(os.environ.get("FUZZ_EXAMPLES", "60")), deadline=None,
          suppress_health_check=[HealthCheck.too_slow])
@given(m=st.integers(0, 500), k=st.integers(1, 700), density=st.floats(0.0, 0.3),
       long_row=st.booleans(), data=st.integers(0, 1 << 30))
def test_random_transpose_matches_numpy_and_round_trips(m, k, density, long_row, data):
    """gespmm_csr_transpose_device on random shapes (empty rows/columns, a
    dense row): equal to a stable numpy transpose, canonical, and its
    transpose is the input again."""
    import torch
    rng = np.random.default_rng(data)
    a = _matrix(rng, m, k, density, long_row) if m else G.CsrMatrix(0, k, np.zeros(1, np.uint32),
                                                                     np.zeros(0, np.uint32),
                                                                     np.zeros(0, np.float32))
    d = G.DeviceCsr.from_host(a, torch.device("cuda:0"))
    t = d.transpose()
    torch.cuda.synchronize()
    th = t.to_host()
    rows = np.repeat(np.arange(m, dtype=np.int64), np.diff(a.row_ptr.astype(np.int64)))
    cols = a.col_ind.astype(np.int64)
    order = np.lexsort((rows, cols))  # by column, then row: the canonical transpose
    want_rp = np.concatenate([[0], np.cumsum(np.bincount(cols, minlength=k))]).astype(np.uint32)
    assert th.n_rows == k and th.n_cols == m
    assert np.array_equal(th.row_ptr, want_rp)
    assert np.array_equal(th.col_ind[:a.nnz()], rows[order].astype(np.uint32))
    assert np.array_equal(th.vals[:a.nnz()].view(np.uint32), a.vals[order].view(np.uint32))
    back = t.transpose().to_host()
    assert np.array_equal(back.row_ptr, a.row_ptr)
    assert np.array_equal(back.col_ind[:a.nnz()], a.col_ind)
    assert np.array_equal(back.vals[:a.nnz()].view(np.uint32), a.vals.view(np.uint32))


@seed(20261021)
@settings(max_examples=int(os.environ.get("FUZZ_EXAMPLES", "60")), deadline=None,
          suppress_health_check=[HealthCheck.too_slow])
@given(rows=st.integers(0, 400), cols=st.integers(1, 5000), count=st.integers(0, 20000),
       dup=st.floats(0.0, 0.9), policy=st.sampled_from(["sum", "last"]), bad=st.booleans(),
       data=st.integers(0, 1 << 30))
def test_random_from_coo_device_equals_host(rows, cols, count, dup, policy, bad, data):
    """gespmm_from_coo_device on random triples (duplicate runs of any length,
    empty rows, an out-of-bounds triple): the same CSR, bit for bit, or the
    same error text, as the host from_coo (itself pinned to the reference's,
    tests/test_host_api.py)."""
    import torch
    rng = np.random.default_rng(data)
    if rows == 0:
        count = 0
    r = rng.integers(0, max(rows, 1), count).astype(np.uint32)
    c = rng.integers(0, cols, count).astype(np.uint32)
    if count and dup > 0:  # copy earlier coordinates forward: duplicate runs
        idx = np.nonzero(rng.random(count) < dup)[0]
        src = (rng.random(len(idx)) * np.maximum(idx, 1)).astype(np.int64)
        r[idx], c[idx] = r[src], c[src]
    v = rng.standard_normal(count).astype(np.float32)
    if bad and count:
        i = int(rng.integers(0, count))
        if rng.random() < 0.5:
            r[i] = rows + int(rng.integers(0, 7))
        else:
            c[i] = cols + int(rng.integers(0, 7))
    t = lambda x: torch.from_numpy(x.view(np.int32) if x.dtype == np.uint32 else x).cuda()  # noqa: E731
    try:
        want = G.from_coo(rows, cols, (r, c, v), policy)
    except G.Error as e:
        with pytest.raises(G.Error) as ei:
            G.DeviceCsr.from_coo(rows, cols, t(r), t(c), t(v), policy=policy)
        assert str(ei.value) == str(e)
        return
    got = G.DeviceCsr.from_coo(rows, cols, t(r), t(c), t(v), policy=policy)
    assert np.array_equal(got.row_ptr.cpu().numpy().view(np.uint32), want.row_ptr)
    assert np.array_equal(got.col_ind.cpu().numpy().view(np.uint32), want.col_ind)
    assert np.array_equal(got.vals.cpu().numpy().view(np.uint32), want.vals.view(np.uint32))

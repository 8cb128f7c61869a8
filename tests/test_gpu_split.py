"""GPU: split hub rows (a hub row's nonzeros folded in segments by k_warp into
partial rows, then an ordered combine) — the path plans take instead of the
k_hub ring when the fold does not depend on the order of its partials:
max/min always (strict compare, earliest position among ties: bit-identical
to the sequential fold, arg included), sum/mean in fast mode (tolerance).
Hub rows are forced with a small hub threshold so every segment boundary,
tie and special value crosses the combine."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2007_03179_b200 as G
from conftest import first_divergence

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _graph(rows=3000, nnz=150000, maxdeg=2900, seed=31):
    a = G.gen_powerlaw(rows, nnz, maxdeg, 1.0, seed)
    G.randomize_values(a, seed + 1)
    return a


def _run(a, x, op, ex, arg_kind="edge"):
    d = G.DeviceCsr.from_host(a, DEV)
    plan = G.Plan(d, x.shape[1], op, exec=G.ExecOptions(arg_kind=arg_kind, **ex))
    c = torch.empty((a.n_rows, x.shape[1]), device=DEV)
    arg = (torch.empty((a.n_rows, x.shape[1]), dtype=torch.int32, device=DEV)
           if op in ("max", "min") else None)
    plan.execute(torch.from_numpy(np.ascontiguousarray(x)).to(DEV), c, arg)
    torch.cuda.synchronize()
    desc, launches = plan.description, plan.launches
    plan.close()
    return c.cpu().numpy(), (arg.cpu().numpy() if arg is not None else None), desc, launches


@pytest.mark.parametrize("n", [256, 128, 64, 32, 30, 7])
@pytest.mark.parametrize("op", ["max", "min"])
@pytest.mark.parametrize("arg_kind", ["edge", "column"])
def test_split_max_min_bit_exact(n, op, arg_kind):
    a = _graph()
    x = G.make_random_dense(a.n_cols, n, 33).data
    want, warg = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, x, op, want_arg=True,
                        arg_kind=O.ARG_COLUMN if arg_kind == "column" else O.ARG_EDGE)
    c, arg, desc, launches = _run(a, x, op, {"hub_threshold": 300}, arg_kind)
    assert "split" in desc and launches == 3, desc
    assert first_divergence(c, want) is None
    assert np.array_equal(arg, warg)


@pytest.mark.parametrize("op", ["max", "min"])
def test_split_ties_and_special_values(op):
    """Few distinct products (values +-1, B on a 4-value grid, zeros of both
    signs, NaN/inf columns): equal maxima across segment boundaries must keep
    the earliest position and its exact bits, NaN never enters."""
    a = _graph(seed=41)
    rng = np.random.default_rng(42)
    a = G.CsrMatrix(a.n_rows, a.n_cols, a.row_ptr, a.col_ind,
                    np.where(rng.random(len(a.vals)) < 0.5, -1.0, 1.0).astype(np.float32))
    x = rng.integers(-2, 2, (a.n_cols, 64)).astype(np.float32)
    x[:, 5] = 0.0
    x[::2, 6] = -0.0
    x[1::2, 6] = 0.0
    x[::9, 7] = np.nan
    x[::4, 8] = np.inf
    x[::3, 9] = -np.inf
    want, warg = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, x, op, want_arg=True)
    c, arg, desc, _ = _run(a, x, op, {"hub_threshold": 300})
    assert "split" in desc
    gn, wn = np.isnan(c), np.isnan(want)
    assert np.array_equal(gn, wn)
    assert np.array_equal(c[~gn].view(np.uint32), want[~wn].view(np.uint32))
    assert np.array_equal(arg, warg)


@pytest.mark.parametrize("op", ["sum", "mean"])
def test_split_fast_sum_mean_within_tolerance(op):
    a = _graph(seed=51)
    x = G.make_random_dense(a.n_cols, 128, 53).data
    want, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, x, op)
    scale, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, np.abs(a.vals), np.abs(x), op)
    c, _, desc, _ = _run(a, x, op, {"hub_threshold": 300, "exact": False})
    assert "split" in desc
    err = np.abs(c.astype(np.float64) - want)
    assert np.all(err <= 1e-5 * np.maximum(np.abs(want), scale) + 1e-30)


def test_exact_sum_keeps_the_ring():
    """Exact sum never splits (reassociation would change bits)."""
    a = _graph(seed=61)
    x = G.make_random_dense(a.n_cols, 128, 63).data
    want, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, x, "sum")
    c, _, desc, _ = _run(a, x, "sum", {"hub_threshold": 300})
    assert "split" not in desc
    assert first_divergence(c, want) is None


def test_split_replicas_equal_oracle():
    """The fused all-gather epilogue: the combine stores hub rows into every
    replica, k_warp the rest."""
    a = _graph(seed=71)
    x = G.make_random_dense(a.n_cols, 64, 73).data
    want, warg = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, x, "max", want_arg=True)
    d = G.DeviceCsr.from_host(a, DEV)
    plan = G.Plan(d, 64, "max", exec=G.ExecOptions(hub_threshold=300))
    assert "split" in plan.description
    reps = [torch.full((a.n_rows, 64), 7.0, device=DEV) for _ in range(3)]
    args = [torch.full((a.n_rows, 64), -7, dtype=torch.int32, device=DEV) for _ in range(3)]
    plan.execute_gather(torch.from_numpy(x).to(DEV), [r.data_ptr() for r in reps],
                        [g.data_ptr() for g in args])
    torch.cuda.synchronize()
    for r, g in zip(reps, args):
        assert first_divergence(r.cpu().numpy(), want) is None
        assert np.array_equal(g.cpu().numpy(), warg)
    plan.close()


@pytest.mark.parametrize("op", ["max", "sum"])
def test_cached_split_plan_follows_row_ptr_changed_in_place(op):
    """The plan-less entry caches plans by the CSR's pointers and shape; a
    split plan's virtual row_ptr over hub-row segments holds row_ptr values,
    so a cache hit must rebuild it from the live row_ptr.  Overwrite A in
    place with another matrix of the same shape and nnz (what a recycled
    allocation looks like) and check the second call against the oracle."""
    a1, a2 = _graph(seed=61), _graph(seed=62)
    assert a1.nnz() == a2.nnz() and not np.array_equal(a1.row_ptr, a2.row_ptr)
    x = G.make_random_dense(a1.n_cols, 64, 63).data
    xd = torch.from_numpy(np.ascontiguousarray(x)).to(DEV)
    ex = G.ExecOptions(hub_threshold=300, exact=(op != "sum"))
    d = G.DeviceCsr.from_host(a1, DEV)
    for a in (a1, a2, a1):
        src = G.DeviceCsr.from_host(a, DEV)
        d.row_ptr.copy_(src.row_ptr)
        d.col_ind.copy_(src.col_ind)
        d.vals.copy_(src.vals)
        c, arg = G.spmm(d, xd, op, want_arg=(op == "max"), exec=ex, validate=False)
        torch.cuda.synchronize()
        want, warg = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, x, op,
                            want_arg=(op == "max"))
        if op == "max":
            assert first_divergence(c.cpu().numpy(), want) is None
            assert np.array_equal(arg.cpu().numpy(), warg)
        else:  # fast-mode sum: the north_star's 1e-5 relative tolerance
            scale, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, np.abs(a.vals),
                              np.abs(x), op)
            err = np.abs(c.cpu().numpy().astype(np.float64) - want)
            assert np.all(err <= 1e-5 * np.maximum(np.abs(want), scale) + 1e-30)


def test_plan_less_calls_on_two_streams_do_not_share_scratch():
    """Back-to-back plan-less calls on two streams with the same CSR: each
    stream gets its own cached plan (split partials and hub counters are
    per-execute scratch), so concurrently running executes never mix."""
    a = _graph(seed=81)
    d = G.DeviceCsr.from_host(a, DEV)
    ex = G.ExecOptions(hub_threshold=300)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    xs = [G.make_random_dense(a.n_cols, 64, 90 + i).data for i in range(6)]
    xds = [torch.from_numpy(np.ascontiguousarray(x)).to(DEV) for x in xs]
    torch.cuda.synchronize()
    outs = []
    for i, xd in enumerate(xds):
        s = streams[i % 2]
        with torch.cuda.stream(s):
            outs.append(G.spmm(d, xd, "max", want_arg=True, exec=ex, validate=False, stream=s))
    torch.cuda.synchronize()
    for x, (c, arg) in zip(xs, outs):
        want, warg = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, x, "max",
                            want_arg=True)
        assert first_divergence(c.cpu().numpy(), want) is None
        assert np.array_equal(arg.cpu().numpy(), warg)


@pytest.mark.parametrize("explicit", [False, True])
def test_low_degree_plan_stays_correct_when_a_gets_long_rows(explicit):
    """A plan made for a low-degree matrix (identity row order, several rows
    per warp) only orders rows: overwrite A in place with a power-law matrix of
    the same shape and nnz (rows far longer than the plan saw) and both the
    explicit plan and the plan-less call still match the oracle bit for bit."""
    lo = G.gen_uniform_random(G.GraphGenSpec(3000, 30000, 5))
    G.randomize_values(lo, 6)
    hi = G.gen_powerlaw(3000, 30000, 2900, 1.0, 7)
    G.randomize_values(hi, 8)
    assert lo.nnz() == hi.nnz()
    x = G.make_random_dense(3000, 128, 9).data
    xd = torch.from_numpy(np.ascontiguousarray(x)).to(DEV)
    d = G.DeviceCsr.from_host(lo, DEV)
    plan = G.Plan(d, 128, "sum") if explicit else None
    for a in (lo, hi):
        src = G.DeviceCsr.from_host(a, DEV)
        d.row_ptr.copy_(src.row_ptr)
        d.col_ind.copy_(src.col_ind)
        d.vals.copy_(src.vals)
        if explicit:
            c = torch.empty((3000, 128), device=DEV)
            plan.execute(xd, c)
        else:
            c, _ = G.spmm(d, xd, "sum", validate=False)
        torch.cuda.synchronize()
        want, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, x, "sum")
        assert first_divergence(c.cpu().numpy(), want) is None
    if plan is not None:
        plan.close()

"""GPU: overlap_prev plans (programmatic dependent launch onto the previous
kernel: the A-side prologue runs before griddepcontrol.wait, B reads and C
writes after it).  Chained ping-pong hops H_{t+1} = A H_t — each SpMM reads
what the previous one wrote and overwrites what it read — must stay
bit-identical to the oracle, eagerly and replayed from a CUDA graph."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2007_03179_b200 as G

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _graph(kind, m, nnz):
    if kind == "uniform":
        return G.gen_uniform_random(G.GraphGenSpec(m, nnz, 5))
    return G.gen_powerlaw(m, nnz, 300, 1.0, 5)


def _oracle_hops(a, x, hops, op):
    h, args = x, None
    for _ in range(hops):
        h, args = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, h, op,
                         want_arg=op in ("max", "min"))
    return h, args


@pytest.mark.parametrize("kind,m,nnz,n,op", [
    ("uniform", 19717, 88648, 128, "sum"),   # Pubmed shape, the small-config chain
    ("uniform", 2708, 10556, 16, "sum"),     # Cora shape
    ("powerlaw", 6000, 90000, 64, "max"),
    ("uniform", 5000, 40000, 32, "mean"),
])
@pytest.mark.parametrize("graph", [False, True])
def test_overlap_chain_equals_oracle(kind, m, nnz, n, op, graph):
    a = _graph(kind, m, nnz)
    G.randomize_values(a, 6)
    x = G.make_random_dense(m, n, 7).data
    d = G.DeviceCsr.from_host(a, DEV)
    plan = G.Plan(d, n, op, exec=G.ExecOptions(overlap_prev=True))
    assert plan.launches == 1
    bufs = [torch.from_numpy(x).to(DEV), torch.empty((m, n), device=DEV)]
    arg = torch.empty((m, n), dtype=torch.int32, device=DEV) if op in ("max", "min") else None
    hops = 6
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        plan.execute(bufs[0], bufs[1], arg)  # setup outside any capture
    torch.cuda.synchronize()
    bufs[1].zero_()
    torch.cuda.synchronize()

    def run():
        for t in range(hops):
            plan.execute(bufs[t % 2], bufs[(t + 1) % 2], arg)

    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            run()
        bufs[0].copy_(torch.from_numpy(x).to(DEV))
        torch.cuda.synchronize()
        g.replay()
    else:
        with torch.cuda.stream(st):
            run()
    torch.cuda.synchronize()
    want, wargs = _oracle_hops(a, x, hops, op)
    got = bufs[hops % 2].cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    if arg is not None:
        assert np.array_equal(arg.cpu().numpy(), wargs)
    plan.close()


def test_overlap_ignored_by_hub_plans():
    """A plan whose execute is two kernels (hub rows) never chains; results
    unchanged."""
    a = G.gen_powerlaw(4000, 120000, 3000, 1.0, 9)
    G.randomize_values(a, 10)
    x = G.make_random_dense(4000, 128, 11).data
    d = G.DeviceCsr.from_host(a, DEV)
    plan = G.Plan(d, 128, "sum", exec=G.ExecOptions(overlap_prev=True, hub_threshold=500))
    assert plan.launches == 2
    c = torch.empty((4000, 128), device=DEV)
    plan.execute(torch.from_numpy(x).to(DEV), c)
    want, _ = O.spmm(4000, 4000, a.row_ptr, a.col_ind, a.vals, x, "sum")
    assert np.array_equal(c.cpu().numpy().view(np.uint32), want.view(np.uint32))
    plan.close()

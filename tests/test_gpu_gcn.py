"""GPU: CSR transpose and the two-layer GCN driver (config 5 of BASELINE.json)."""
import numpy as np
import pytest

import oracle as O
import paper_2007_03179_b200 as G
from paper_2007_03179_b200 import gcn
from conftest import first_divergence

pytestmark = pytest.mark.gpu


def _host_transpose(a):
    """Stable counting-sort transpose (test-side checker)."""
    rows = np.repeat(np.arange(a.n_rows, dtype=np.uint32), np.diff(a.row_ptr.astype(np.int64)))
    order = np.argsort(a.col_ind, kind="stable")
    rp = np.zeros(a.n_cols + 1, np.int64)
    np.add.at(rp, a.col_ind.astype(np.int64) + 1, 1)
    return G.CsrMatrix(a.n_cols, a.n_rows, np.cumsum(rp).astype(np.uint32), rows[order],
                       a.vals[order])


@pytest.mark.parametrize("shape", [(1, 1, 0), (5, 7, 0), (300, 200, 4000), (3000, 3000, 120000)])
def test_csr_transpose_matches_host(shape, cuda):
    m, k, nnz = shape
    if m == k and nnz:
        a = G.gen_powerlaw(m, nnz, m - 1, 1.0, 5)
    elif nnz:
        rng = np.random.default_rng(0)
        flat = np.sort(rng.choice(m * k, nnz, replace=False))
        r, c = flat // k, flat % k
        rp = np.zeros(m + 1, np.int64)
        np.add.at(rp, r + 1, 1)
        a = G.CsrMatrix(m, k, np.cumsum(rp).astype(np.uint32), c.astype(np.uint32),
                        np.ones(nnz, np.float32))
    else:
        a = G.CsrMatrix.empty(m, k)
    G.randomize_values(a, 3)
    t = G.DeviceCsr.from_host(a).transpose().to_host()
    want = _host_transpose(a)
    assert np.array_equal(t.row_ptr, want.row_ptr)
    assert np.array_equal(t.col_ind, want.col_ind)
    assert np.array_equal(t.vals.view(np.uint32), want.vals.view(np.uint32))
    # A^T is canonical and (A^T)^T == A
    n, _ = O.validate(t.n_rows, t.n_cols, t.row_ptr, t.col_ind, t.vals)
    assert n == 0
    tt = G.DeviceCsr.from_host(t).transpose().to_host()
    assert np.array_equal(tt.row_ptr, a.row_ptr) and np.array_equal(tt.col_ind, a.col_ind)


def test_transpose_spmm_is_the_adjoint(cuda):
    """<A x, y> == <x, A^T y> (float64 accumulation of float32 results)."""
    import torch
    a = G.gen_powerlaw(4000, 200000, 3000, 1.0, 9)
    G.randomize_values(a, 10)
    d = G.DeviceCsr.from_host(a)
    t = d.transpose()
    x = torch.from_numpy(G.make_random_dense(4000, 16, 1).data).to(cuda)
    y = torch.from_numpy(G.make_random_dense(4000, 16, 2).data).to(cuda)
    ax, _ = G.spmm(d, x, "sum")
    aty, _ = G.spmm(t, y, "sum")
    lhs = (ax.double() * y.double()).sum().item()
    rhs = (x.double() * aty.double()).sum().item()
    assert abs(lhs - rhs) <= 1e-4 * max(1.0, abs(lhs))


def _dense_reference_step(a, h, y, w1, w2):
    import torch
    A = torch.zeros(a.n_rows, a.n_cols, dtype=torch.float64)
    rows = np.repeat(np.arange(a.n_rows), np.diff(a.row_ptr.astype(np.int64)))
    A[torch.from_numpy(rows), torch.from_numpy(a.col_ind.astype(np.int64))] = \
        torch.from_numpy(a.vals.astype(np.float64))
    w1 = w1.detach().cpu().double().requires_grad_(True)
    w2 = w2.detach().cpu().double().requires_grad_(True)
    hd = torch.from_numpy(h).double()
    z2 = A @ (torch.relu(A @ (hd @ w1)) @ w2)
    loss = torch.nn.functional.cross_entropy(z2, torch.from_numpy(y), reduction="sum") / a.n_rows
    loss.backward()
    return z2.detach(), loss.item(), w1.grad, w2.grad


def test_gcn_step_matches_dense_float64_reference(cuda):
    import torch
    a = gcn.normalize_adjacency(G.gen_powerlaw(1500, 60000, 1000, 1.0, 4))
    cfg = gcn.GCNConfig(in_features=24, hidden=64, classes=7, lr=0.5)
    h, y = gcn.synthetic_features(a.n_rows, cfg.in_features, cfg.classes)
    adj, info = gcn.build_adjacency(a, cuda)
    model = gcn.GCN(cfg, cuda)
    ht = torch.from_numpy(h).to(cuda)
    yt = torch.from_numpy(y).to(cuda)
    # the model pads W2 to 8 zero-filled columns (float4 SpMM lanes); the
    # reference is the unpadded 7-class model
    assert model.w2.shape[1] == cfg.classes_padded == 8
    z_ref, loss_ref, g1_ref, g2_ref = _dense_reference_step(a, h, y, model.w1,
                                                            model.w2[:, :cfg.classes])
    z = model.forward(ht, adj)
    assert torch.allclose(z.double().cpu(), z_ref, rtol=1e-4, atol=1e-4)
    w1_before = model.w1.detach().clone()
    loss = model.step(ht, yt, adj)
    assert abs(loss.item() - loss_ref) <= 1e-4 * max(1.0, abs(loss_ref))
    g1 = (w1_before - model.w1.detach()) / cfg.lr
    assert torch.allclose(g1.double().cpu(), g1_ref, rtol=2e-3, atol=1e-5)
    # a few steps reduce the loss
    losses = [model.step(ht, yt, adj).item() for _ in range(10)]
    assert losses[-1] < loss.item()
    assert (model.w2.detach()[:, cfg.classes:] == 0).all()  # padding never trains
    assert np.isfinite(losses).all()
    adj.close()

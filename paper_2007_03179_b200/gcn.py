"""Two-layer GCN on the GE-SpMM kernels (BASELINE.json config 5).

    Z1 = A · (H W1),  H1 = relu(Z1),  Z2 = A · (H1 W2),  loss = CE(Z2[train], y)

Aggregation is the tuned SpMM (sum); its backward is the SpMM with A^T
(built once on the device by gespmm_csr_transpose_device).  The dense
transforms are plain torch matmuls (cuBLAS — library GEMMs).  The paper's
integration into GNN frameworks (§IV-B) is exactly this: SpMM-like as
an autograd op.

Multi-GPU (one process per GPU): nodes are row-sharded by nnz
(dist.partition_rows); rank r holds rows [lo, hi) of A and of A^T.  Each layer
all-gathers the transformed features before aggregating (forward) and the
incoming gradient before the A^T aggregation (backward) — the per-layer NCCL
all-gather of the north_star, one in-place ncclAllGather into a padded buffer
that the local blocks' column ids index directly (dist.pad_columns: no
concatenation); weight gradients are all-reduced.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, Optional, Tuple

import numpy as np

from . import api
from .api import CsrMatrix, DeviceCsr, ExecOptions, Plan
from . import dist as D


class Adjacency:
    """A (rows lo..hi of the graph) and A^T (rows lo..hi of the transpose) on
    one device, with cached plans per feature width."""

    def __init__(self, a_rows: DeviceCsr, at_rows: DeviceCsr, exec: ExecOptions = ExecOptions()):
        self.a, self.at = a_rows, at_rows
        self.exec = exec
        self._plans: Dict[Tuple[bool, int], Plan] = {}

    def plan(self, transposed: bool, n: int) -> Plan:
        key = (transposed, n)
        if key not in self._plans:
            self._plans[key] = Plan(self.at if transposed else self.a, n, "sum", exec=self.exec)
        return self._plans[key]

    def close(self):
        for p in self._plans.values():
            p.close()
        self._plans.clear()


def build_adjacency(a: CsrMatrix, device, rank: int = 0, world: int = 1,
                    exec: ExecOptions = ExecOptions()):
    """Shard A by nnz-balanced rows; build A^T on the device from the full A and
    keep the same node range of it.  Returns (Adjacency, ShardInfo)."""
    import torch
    bounds = D.partition_rows(a.row_ptr, world)
    info = D.ShardInfo(rank, world, bounds)
    full = DeviceCsr.from_host(a, device)
    at_full = full.transpose()
    torch.cuda.synchronize(device)
    if world == 1:
        return Adjacency(full, at_full, exec), info
    # column ids of the local blocks index the padded all-gather buffer
    # (dist.pad_columns), so each layer's exchange feeds the SpMM directly
    a_loc = DeviceCsr.from_host(D.pad_columns(D.shard_csr(a, info.lo, info.hi), info), device)
    at_host = at_full.to_host()
    at_loc = DeviceCsr.from_host(D.pad_columns(D.shard_csr(at_host, info.lo, info.hi), info),
                                 device)
    del full, at_full
    return Adjacency(a_loc, at_loc, exec), info


# When a list, every per-layer exchange appends its (start, end) CUDA events,
# so bench.py can report the all-gather time apart from the step.
EXCHANGE_EVENTS = None


def _gather(x, info: Optional[D.ShardInfo]):
    """The per-layer exchange: one in-place ncclAllGather into the padded buffer
    the local A / A^T blocks are column-indexed by (build_adjacency)."""
    if info is None or info.world == 1:
        return x
    import torch
    ev = None
    if EXCHANGE_EVENTS is not None:
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
    out = torch.empty((info.world * info.max_rows, x.shape[1]), dtype=x.dtype, device=x.device)
    D.allgather_padded(x.contiguous(), info, out=out)
    if ev is not None:
        ev[1].record()
        EXCHANGE_EVENTS.append(ev)
    return out


class _Aggregate:
    """torch.autograd.Function: Y_local = A_local · gather(X_local); dX_local = A^T_local · gather(dY_local)."""

    @staticmethod
    def make():
        import torch

        class Aggregate(torch.autograd.Function):
            @staticmethod
            def forward(ctx, x, adj: Adjacency, info):
                x_full = _gather(x, info).contiguous()
                out = torch.empty((adj.a.n_rows, x.shape[1]), dtype=x.dtype, device=x.device)
                adj.plan(False, x.shape[1]).execute(x_full, out)
                ctx.adj, ctx.info = adj, info
                return out

            @staticmethod
            def backward(ctx, grad):
                g_full = _gather(grad.contiguous(), ctx.info).contiguous()
                adj = ctx.adj
                out = torch.empty((adj.at.n_rows, grad.shape[1]), dtype=grad.dtype,
                                  device=grad.device)
                adj.plan(True, grad.shape[1]).execute(g_full, out)
                return out, None, None

        return Aggregate


_AGG = None


def aggregate(x, adj: Adjacency, info: Optional[D.ShardInfo] = None):
    global _AGG
    if _AGG is None:
        _AGG = _Aggregate.make()
    return _AGG.apply(x, adj, info)


@dataclasses.dataclass
class GCNConfig:
    in_features: int = 602     # Reddit
    hidden: int = 256          # BASELINE config 5
    classes: int = 41
    lr: float = 0.01
    seed: int = 0
    # aggregated widths are padded to a multiple of this with zero weight
    # columns: N % 4 == 0 rows are 16-byte aligned, so the SpMM uses float4
    # lanes (41 classes -> 44: 2.4 -> ~1 ms per Reddit SpMM); the padded
    # logits are sliced off before the loss, so the model is unchanged
    pad_to: int = 4

    @property
    def classes_padded(self) -> int:
        q = max(1, self.pad_to)
        return (self.classes + q - 1) // q * q


class GCN:
    """Two GCN layers with explicit parameters (no nn.Module magic needed)."""

    def __init__(self, cfg: GCNConfig, device):
        import torch
        g = torch.Generator(device="cpu").manual_seed(cfg.seed)
        s1 = (6.0 / (cfg.in_features + cfg.hidden)) ** 0.5
        s2 = (6.0 / (cfg.hidden + cfg.classes)) ** 0.5
        self.w1 = ((torch.rand(cfg.in_features, cfg.hidden, generator=g) * 2 - 1) * s1).to(device)
        w2 = torch.zeros(cfg.hidden, cfg.classes_padded)
        w2[:, :cfg.classes] = (torch.rand(cfg.hidden, cfg.classes, generator=g) * 2 - 1) * s2
        self.w2 = w2.to(device)
        self.w1.requires_grad_(True)
        self.w2.requires_grad_(True)
        self.cfg = cfg

    def params(self):
        return [self.w1, self.w2]

    def forward(self, h, adj: Adjacency, info=None):
        import torch
        z1 = aggregate(h @ self.w1, adj, info)
        h1 = torch.relu(z1)
        return aggregate(h1 @ self.w2, adj, info)[:, :self.cfg.classes]

    def step(self, h, labels, adj: Adjacency, info=None, n_total: Optional[int] = None):
        """One full-batch training step (forward, backward, SGD); returns the loss."""
        import torch
        import torch.nn.functional as F
        logits = self.forward(h, adj, info)
        n_total = n_total if n_total is not None else h.shape[0]
        loss = F.cross_entropy(logits, labels, reduction="sum") / n_total
        for p in self.params():
            p.grad = None
        loss.backward()
        if info is not None and info.world > 1:
            import torch.distributed as dist
            for p in self.params():
                dist.all_reduce(p.grad)
            lt = loss.detach().clone()
            dist.all_reduce(lt)
            loss = lt
        with torch.no_grad():
            for p in self.params():
                p -= self.cfg.lr * p.grad
        return loss.detach()


def sgc_features(a: CsrMatrix, x0, hops: int, info: Optional[D.ShardInfo], device,
                 exchange: str = "fused", group=None, exec: Optional[ExecOptions] = None):
    """SGC-style propagated features S^K X (Wu et al. 2019: the K stacked
    aggregations of a GCN without the per-layer transforms, then one linear
    layer).  The hops are stacked SpMM layers whose outputs are the next hop's
    gathered operand, so the per-hop exchange can be fused into the SpMM
    epilogue: ``exchange="fused"`` runs dist.fused_propagate (peer stores over
    NVLink + one device barrier per hop), ``"nccl"`` dist.nccl_propagate (SpMM
    into the padded slot + in-place all-gather).  Both return the full M x F
    result on every rank, bit-identical (each element is folded by one thread
    in CSR order either way).  x0: the full M x F input on `device`."""
    info = info or D.ShardInfo(0, 1, [0, a.n_rows])
    if exchange == "fused":
        return D.fused_propagate(a, x0, hops, info, device, "sum", group=group, exec=exec)
    if exchange == "nccl":
        return D.nccl_propagate(a, x0, hops, info, device, "sum", group=group, exec=exec)
    raise ValueError(f"exchange must be 'fused' or 'nccl', not {exchange!r}")


def normalize_adjacency(a: CsrMatrix, add_self_loops: bool = True) -> CsrMatrix:
    """GCN propagation matrix D^-1/2 (A + I) D^-1/2 on A's pattern (values
    ignored), as a canonical CSR (Kipf & Welling; the normalisation GE-SpMM's
    GCN experiments use through PyG/DGL, §V-E)."""
    m = a.n_rows
    rp = a.row_ptr.astype(np.int64)
    rows = np.repeat(np.arange(m, dtype=np.int64), np.diff(rp))
    cols = a.col_ind.astype(np.int64)
    if add_self_loops and m == a.n_cols:
        # insert (i, i) where missing, keeping rows sorted (vectorised merge)
        has = np.zeros(m, bool)
        has[rows[cols == rows]] = True
        need = ~has
        before = np.bincount(rows[cols < rows], minlength=m)         # entries left of the diagonal
        shift = np.concatenate([[0], np.cumsum(need)])               # inserted before row i
        new_pos = np.arange(len(rows)) + shift[rows] + (need[rows] & (cols > rows))
        diag_rows = np.nonzero(need)[0]
        diag_pos = rp[diag_rows] + before[diag_rows] + shift[diag_rows]
        total = len(rows) + len(diag_rows)
        r2 = np.empty(total, np.int64)
        c2 = np.empty(total, np.int64)
        r2[new_pos], c2[new_pos] = rows, cols
        r2[diag_pos], c2[diag_pos] = diag_rows, diag_rows
        rows, cols = r2, c2
    deg_r = np.bincount(rows, minlength=m).astype(np.float64)
    deg_c = np.bincount(cols, minlength=a.n_cols).astype(np.float64)
    vals = (1.0 / np.sqrt(deg_r[rows] * deg_c[cols])).astype(np.float32)
    new_rp = np.zeros(m + 1, np.int64)
    np.add.at(new_rp, rows + 1, 1)
    return CsrMatrix(m, a.n_cols, np.cumsum(new_rp).astype(np.uint32), cols.astype(np.uint32), vals)


def synthetic_features(m: int, f: int, classes: int, seed: int = 3):
    """Deterministic node features (reference make_random_dense) and labels."""
    h = api.make_random_dense(m, f, seed).data
    rng = np.random.default_rng(seed)
    y = rng.integers(0, classes, m).astype(np.int64)
    return h, y


def spmm_flops_per_step(nnz: int, cfg: GCNConfig) -> int:
    """4 SpMMs per step: A·X1 (hidden), A·X2 (classes), and the two A^T ones.
    Counted at the model's widths (the padding columns are not counted)."""
    return 2 * nnz * (2 * cfg.hidden + 2 * cfg.classes)

"""Multi-GPU layer: nnz-balanced row shards, B replicated once, C row blocks
re-assembled for stacked layers.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch on the box,
gloo on CPU for tests).  The SpMM itself needs no exchange: output row i
depends only on CSR row i and B, so each rank runs the local
kernel on its shard.  Collectives appear only where the path really moves
data:

* ``broadcast_dense`` — the dense operand B, once per B (north_star: "replicated
  once via NCCL broadcast");
* ``allgather_rows`` — variable-size C row blocks for the next layer
  (padded to the largest shard, as ncclAllGather needs equal counts).

The compute callable is injected, so the plumbing is tested on CPU (gloo)
with the oracle as the per-shard compute, and runs the CUDA path on the box.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, List, Sequence

import numpy as np

from .api import CsrMatrix


def partition_rows(row_ptr: np.ndarray, parts: int) -> List[int]:
    """Contiguous row ranges with ~equal nnz: boundary g is the first row whose
    prefix reaches g*nnz/parts (binary search on row_ptr).  Returns parts+1
    boundaries b[0]=0 <= ... <= b[parts]=M; every row lands in exactly one shard."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    rp = np.asarray(row_ptr, np.int64)
    m = len(rp) - 1
    nnz = int(rp[-1])
    bounds = [0]
    for g in range(1, parts):
        target = (nnz * g) // parts
        r = int(np.searchsorted(rp, target, side="left"))
        r = min(max(r, bounds[-1]), m)
        bounds.append(r)
    bounds.append(m)
    return bounds


def shard_csr(a: CsrMatrix, lo: int, hi: int) -> CsrMatrix:
    """Rows [lo, hi) of A with a rebased row_ptr; the column space is unchanged."""
    rp = np.asarray(a.row_ptr, np.int64)
    s, e = int(rp[lo]), int(rp[hi])
    return CsrMatrix(hi - lo, a.n_cols, (rp[lo:hi + 1] - s).astype(np.uint32),
                     np.ascontiguousarray(a.col_ind[s:e]), np.ascontiguousarray(a.vals[s:e]))


@dataclasses.dataclass
class ShardInfo:
    rank: int
    world: int
    bounds: List[int]

    @property
    def lo(self) -> int:
        return self.bounds[self.rank]

    @property
    def hi(self) -> int:
        return self.bounds[self.rank + 1]

    @property
    def rows(self) -> int:
        return self.hi - self.lo

    @property
    def max_rows(self) -> int:
        return max(self.bounds[i + 1] - self.bounds[i] for i in range(self.world))


def broadcast_dense(tensor, src: int = 0, group=None):
    """Replicate B from ``src`` to every rank (NCCL broadcast on GPUs)."""
    import torch.distributed as dist
    dist.broadcast(tensor, src=src, group=group)
    return tensor


def allgather_rows(local, info: ShardInfo, group=None):
    """Assemble the full M x N output from per-rank row blocks of unequal height.
    Each block is padded to the largest shard, all-gathered, then unpadded."""
    import torch
    import torch.distributed as dist
    n = local.shape[1]
    pad = info.max_rows
    buf = torch.zeros((pad, n), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]].copy_(local)
    gathered = [torch.empty_like(buf) for _ in range(info.world)]
    dist.all_gather(gathered, buf, group=group)
    parts = [gathered[r][: info.bounds[r + 1] - info.bounds[r]] for r in range(info.world)]
    return torch.cat(parts, dim=0)


def distributed_spmm(a: CsrMatrix, b, rank: int, world: int,
                     compute: Callable[[CsrMatrix, object], object], gather: bool = True,
                     group=None):
    """Row-sharded SpMM-like: B is broadcast from rank 0, each rank computes
    its nnz-balanced shard with ``compute(shard, B)``; optionally all-gather C."""
    bounds = partition_rows(a.row_ptr, world)
    info = ShardInfo(rank, world, bounds)
    broadcast_dense(b, 0, group)
    local = compute(shard_csr(a, info.lo, info.hi), b)
    if not gather:
        return local, info
    return allgather_rows(local, info, group), info


def shard_balance(row_ptr: Sequence[int], bounds: Sequence[int]) -> float:
    """max shard nnz / mean shard nnz (1.0 = perfect)."""
    rp = np.asarray(row_ptr, np.int64)
    loads = [int(rp[bounds[i + 1]] - rp[bounds[i]]) for i in range(len(bounds) - 1)]
    mean = sum(loads) / len(loads)
    return max(loads) / mean if mean else 1.0

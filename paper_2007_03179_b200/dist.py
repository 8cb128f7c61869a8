"""Multi-GPU layer: nnz-balanced row shards, B replicated once, C row blocks
re-assembled for stacked layers.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch on the box,
gloo on CPU for tests).  The SpMM itself needs no exchange: output row i
depends only on CSR row i and B, so each rank runs the local
kernel on its shard.  Collectives appear only where the path really moves
data:

* ``broadcast_dense`` — the dense operand B, once per B (north_star: "replicated
  once via NCCL broadcast");
* ``allgather_padded`` — variable-size C row blocks for the next layer, one
  in-place ncclAllGather into a buffer padded to the largest shard (equal
  counts); ``pad_columns`` re-indexes a shard's columns into that buffer so
  the next SpMM reads it directly (``allgather_rows`` compacts it instead).

The compute callable is injected, so the plumbing is tested on CPU (gloo)
with the oracle as the per-shard compute, and runs the CUDA path on the box.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, List, Optional, Sequence

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


def allgather_padded(local, info: ShardInfo, out=None, group=None):
    """Per-layer exchange into ONE padded buffer: rank r's block lands at rows
    [r*pad, r*pad + rows_r) of ``out`` (world*pad x N), pad = the largest shard.
    One in-place all_gather_into_tensor (ncclAllGather), no per-rank buffers and
    no concatenation.  ``local`` may already be ``out``'s own slot (zero-copy);
    otherwise it is copied in.  Returns ``out``.  Pair it with
    ``pad_columns`` so the next SpMM reads the padded buffer directly."""
    import torch
    import torch.distributed as dist
    n = local.shape[1]
    pad = info.max_rows
    if out is None:
        out = torch.zeros((info.world * pad, n), dtype=local.dtype, device=local.device)
    slot = out[info.rank * pad:(info.rank + 1) * pad]
    if local.data_ptr() != slot.data_ptr():
        slot[: local.shape[0]].copy_(local)
    dist.all_gather_into_tensor(out, slot, group=group)
    return out


def padded_row(info: ShardInfo, rows):
    """Global row ids -> their rows in the padded all-gather buffer."""
    b = np.asarray(info.bounds, np.int64)
    rows = np.asarray(rows, np.int64)
    owner = np.searchsorted(b, rows, side="right") - 1
    return owner * info.max_rows + (rows - b[owner])


def pad_columns(a: CsrMatrix, info: ShardInfo) -> CsrMatrix:
    """A copy of ``a`` whose column ids index the padded all-gather buffer
    (column c -> padded_row(c)).  The map is increasing, so rows stay sorted
    and the fold order (ascending CSR position) is unchanged: results are
    bit-identical to the SpMM on the compact operand."""
    ci = padded_row(info, a.col_ind).astype(np.uint32)
    return CsrMatrix(a.n_rows, info.world * info.max_rows, a.row_ptr.copy(), ci, a.vals.copy())


def allgather_rows(local, info: ShardInfo, group=None):
    """Assemble the full M x N output (compact rows) from per-rank row blocks
    of unequal height: allgather_padded, then one gather of the valid rows."""
    import torch
    buf = allgather_padded(local, info, group=group)
    if info.max_rows * info.world == info.bounds[-1]:
        return buf
    idx = torch.from_numpy(padded_row(info, np.arange(info.bounds[-1]))).to(buf.device)
    return buf.index_select(0, idx)


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


# ---------------------------------------------------------------------------
# Fused all-gather: the SpMM epilogue writes every output row into every
# rank's full-height buffer over peer memory (gespmm_plan_execute_gather), and
# one cross-rank barrier (gespmm_peer_barrier) replaces ncclAllGather.
# ---------------------------------------------------------------------------

class _CudaArray:
    """__cuda_array_interface__ view of a raw device allocation (no ownership)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None, "stream": None}


def _align(x: int, a: int = 256) -> int:
    return (x + a - 1) // a * a


class PeerRows:
    """A full-height M x N f32 buffer (+ optional int32 arg buffer) on every
    rank, mapped into every rank's process, with `world` signal words for the
    barrier.  Rank r's shard lands at rows [lo_r, hi_r) of EVERY rank's copy.

    Allocation: gespmm_peer_alloc (cudaMalloc base pointers), handles exchanged
    with ``all_gather_object`` (any backend: gloo on one shared GPU in the
    tests, NCCL on an NVSwitch box), opened with CUDA IPC (NVLink P2P mappings
    between GPUs).  ``full`` is a torch view of the local copy; it is valid
    while this object is open."""

    def __init__(self, m: int, n: int, info: ShardInfo, device, arg: bool = False, group=None):
        import ctypes as C
        import torch
        import torch.distributed as dist
        from . import _lib
        if info.world > _lib.MAX_GATHER_DSTS:
            raise ValueError(f"fused all-gather supports at most {_lib.MAX_GATHER_DSTS} ranks")
        self.m, self.n, self.info, self.device = int(m), int(n), info, torch.device(device)
        self._L = _lib.lib()
        self._data_bytes = _align(4 * self.m * self.n)
        self._arg_off = self._data_bytes
        self._sig_off = self._arg_off + (self._data_bytes if arg else 0)
        total = self._sig_off + _align(4 * info.world)
        with torch.cuda.device(self.device):
            p = C.c_void_p()
            st = self._L.gespmm_peer_alloc(total, C.byref(p))
            if st != _lib.OK:
                raise RuntimeError(_lib.last_error())
            self._base = int(p.value)
            torch.cuda.synchronize(self.device)
            # zero the signal words (epoch counting starts at 1)
            sig = torch.as_tensor(_CudaArray(self._base + self._sig_off, (info.world,), "<u4"),
                                  device=self.device)
            sig.zero_()
            torch.cuda.synchronize(self.device)
            bases = [self._base] * info.world
            self._opened = []
            if info.world > 1:
                h = C.create_string_buffer(64)
                st = self._L.gespmm_ipc_get_handle(self._base, h)
                if st != _lib.OK:
                    raise RuntimeError(_lib.last_error())
                handles = [None] * info.world
                dist.all_gather_object(handles, bytes(h.raw), group=group)
                for r in range(info.world):
                    if r == info.rank:
                        continue
                    q = C.c_void_p()
                    st = self._L.gespmm_ipc_open_handle(handles[r], C.byref(q))
                    if st != _lib.OK:
                        raise RuntimeError(_lib.last_error())
                    bases[r] = int(q.value)
                    self._opened.append(bases[r])
        self._bases = bases
        self.has_arg = arg
        self.epoch = 0
        self.full = torch.as_tensor(_CudaArray(self._base, (self.m, self.n), "<f4"),
                                    device=self.device)
        self.full_arg = (torch.as_tensor(_CudaArray(self._base + self._arg_off, (self.m, self.n),
                                                    "<i4"), device=self.device)
                         if arg else None)
        self._err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._sigs = (C.c_void_p * info.world)(*[b + self._sig_off for b in bases])

    def dsts(self, rank: Optional[int] = None):
        """(c_dsts, arg_dsts): where shard `rank`'s row 0 lands in every copy,
        this process's own copy first."""
        r = self.info.rank if rank is None else rank
        off = 4 * self.info.bounds[r] * self.n
        order = [self.info.rank] + [p for p in range(self.info.world) if p != self.info.rank]
        c = [self._bases[p] + off for p in order]
        a = [self._bases[p] + self._arg_off + off for p in order] if self.has_arg else None
        return c, a

    def local_rows(self):
        """This rank's shard rows of the local copy (a view)."""
        return self.full[self.info.lo:self.info.hi]

    def barrier(self, stream=None, timeout_ms: int = 60000):
        """Every rank's stores issued before this call (on their streams) are
        visible to every rank's work enqueued after it (device-side barrier)."""
        from . import _lib
        from .api import _stream_ptr
        self.epoch = (self.epoch + 1) & 0xffffffff or 1
        st = self._L.gespmm_peer_barrier(self._sigs, self.info.rank, self.info.world, self.epoch,
                                         timeout_ms, self._err.data_ptr(), _stream_ptr(stream))
        if st != _lib.OK:
            raise RuntimeError(_lib.last_error())

    def check(self):
        """Raises if a barrier timed out (synchronises)."""
        if int(self._err.item()):
            raise RuntimeError("peer barrier timed out (a rank did not arrive)")

    def close(self):
        import torch
        if getattr(self, "_base", None) is None:
            return
        torch.cuda.synchronize(self.device)
        self.full = self.full_arg = None
        for q in self._opened:
            self._L.gespmm_ipc_close(q)
        self._opened = []
        self._L.gespmm_peer_free(self._base)
        self._base = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fused_propagate(a: CsrMatrix, x0, hops: int, info: ShardInfo, device, op: str = "sum",
                    group=None, exec=None, keep_buffers: bool = False):
    """Stacked SpMM layers H_{t+1} = A (x) H_t (SGC/APPNP-style propagation,
    the "stacked layers" of SURVEY.md §8e.4) on nnz-balanced row shards, with
    the per-layer all-gather fused into the SpMM epilogue: each rank's kernel
    stores its rows into every rank's next-layer buffer over NVLink, then one
    device barrier.  Two PeerRows buffers ping-pong.  x0: the full M x N input
    (torch, on `device`, identical on every rank — e.g. after broadcast_dense).
    Returns the full H_hops (a torch tensor owned by the caller)."""
    import torch
    from .api import DeviceCsr, ExecOptions, Plan
    m, n = a.n_rows, int(x0.shape[1])
    if a.n_rows != a.n_cols:
        raise ValueError("propagation needs a square A")
    local = DeviceCsr.from_host(shard_csr(a, info.lo, info.hi), device)
    plan = Plan(local, n, op, exec=exec or ExecOptions())
    bufs = [PeerRows(m, n, info, device, group=group), PeerRows(m, n, info, device, group=group)]
    try:
        # H_0 only feeds this rank's own kernel; peers first write bufs[0] at hop 1,
        # after the hop-0 barrier that this rank reaches only after this copy.
        bufs[0].full.copy_(x0)
        for t in range(hops):
            src, dst = bufs[t % 2], bufs[(t + 1) % 2]
            c_dsts, _ = dst.dsts()
            if info.hi > info.lo:
                plan.execute_gather(src.full, c_dsts)
            dst.barrier()
        out = bufs[hops % 2].full.clone()
        torch.cuda.synchronize(device)
        for bf in bufs:
            bf.check()
        return (out, bufs) if keep_buffers else out
    finally:
        if not keep_buffers:
            for bf in bufs:
                bf.close()
        plan.close()


def nccl_propagate(a: CsrMatrix, x0, hops: int, info: ShardInfo, device, op: str = "sum",
                   group=None, exec=None):
    """The same propagation with the unfused exchange: local SpMM into this
    rank's slot of a padded buffer, then one in-place ncclAllGather
    (allgather_padded); the local block's columns index that buffer
    (pad_columns).  The baseline fused_propagate replaces."""
    from .api import DeviceCsr, ExecOptions, Plan
    import torch
    n = int(x0.shape[1])
    m = a.n_rows
    if info.world == 1:
        local = DeviceCsr.from_host(a, device)
        plan = Plan(local, n, op, exec=exec or ExecOptions())
        h = x0.contiguous()
        try:
            for _ in range(hops):
                y = torch.empty((m, n), dtype=torch.float32, device=device)
                plan.execute(h, y)
                h = y
            return h
        finally:
            plan.close()
    pad = info.max_rows
    local = DeviceCsr.from_host(pad_columns(shard_csr(a, info.lo, info.hi), info), device)
    plan = Plan(local, n, op, exec=exec or ExecOptions())
    idx = torch.from_numpy(padded_row(info, np.arange(m))).to(device)
    bufs = [torch.zeros((info.world * pad, n), dtype=torch.float32, device=device)
            for _ in range(2)]
    bufs[0].index_copy_(0, idx, x0.contiguous())
    try:
        for t in range(hops):
            src, dst = bufs[t % 2], bufs[(t + 1) % 2]
            slot = dst[info.rank * pad:(info.rank + 1) * pad]
            if info.rows:
                plan.execute(src, slot[:info.rows])
            allgather_padded(slot, info, out=dst, group=group)
        return bufs[hops % 2].index_select(0, idx)
    finally:
        plan.close()

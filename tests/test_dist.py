"""CPU, world_size 2 over gloo: the multi-GPU plumbing (nnz-balanced shards,
B broadcast once, variable-height C row all-gather) with the oracle as the
per-shard compute — the CUDA path replaces only that callable on the box."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2007_03179_b200 as G
from paper_2007_03179_b200 import dist as D


def test_partition_rows_balances_nnz_and_covers_all_rows():
    a = G.gen_powerlaw(20000, 800000, 5000, 1.0, 3)
    for parts in (1, 2, 3, 4, 8):
        b = D.partition_rows(a.row_ptr, parts)
        assert b[0] == 0 and b[-1] == a.n_rows and len(b) == parts + 1
        assert all(b[i] <= b[i + 1] for i in range(parts))
        # each shard within one max-degree row of the ideal split
        loads = np.diff(a.row_ptr.astype(np.int64)[b])
        assert loads.sum() == a.nnz()
        assert loads.max() - a.nnz() / parts <= 5000
    assert D.shard_balance(a.row_ptr, D.partition_rows(a.row_ptr, 8)) < 1.06


def test_partition_edge_cases():
    rp = np.array([0, 0, 0, 10, 10], np.uint32)  # one heavy row, empty rows
    b = D.partition_rows(rp, 4)
    assert b[0] == 0 and b[-1] == 4 and sorted(b) == b
    empty = D.partition_rows(np.zeros(1, np.uint32), 3)
    assert empty == [0, 0, 0, 0]
    with pytest.raises(ValueError):
        D.partition_rows(rp, 0)


def test_shard_csr_rebases_rows():
    a = G.gen_uniform_random(G.GraphGenSpec(50, 600, 2))
    s = D.shard_csr(a, 10, 30)
    assert s.n_rows == 20 and s.row_ptr[0] == 0
    assert s.nnz() == int(a.row_ptr[30] - a.row_ptr[10])
    assert np.array_equal(s.col_ind, a.col_ind[a.row_ptr[10]:a.row_ptr[30]])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, op, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = G.gen_powerlaw(3000, 90000, 1500, 1.0, 11)
    G.randomize_values(a, 12)
    if rank == 0:
        b = torch.from_numpy(G.make_random_dense(3000, 24, 13).data.copy())
    else:
        b = torch.zeros(3000, 24)

    def compute(shard, bt):
        c, _ = O.spmm(shard.n_rows, shard.n_cols, shard.row_ptr, shard.col_ind, shard.vals,
                      bt.numpy(), op)
        return torch.from_numpy(c)

    full, info = D.distributed_spmm(a, b, rank, world, compute)
    np.save(os.path.join(result_dir, f"rank{rank}.npy"), full.numpy())
    np.save(os.path.join(result_dir, f"b{rank}.npy"), b.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("op", ["sum", "max"])
def test_two_rank_gloo_spmm_equals_single_process(tmp_path, op):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), op, str(tmp_path)), nprocs=world, join=True)
    a = G.gen_powerlaw(3000, 90000, 1500, 1.0, 11)
    G.randomize_values(a, 12)
    b = G.make_random_dense(3000, 24, 13)
    want, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b.data, op)
    for r in range(world):
        got = np.load(tmp_path / f"rank{r}.npy")
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
        assert np.array_equal(np.load(tmp_path / f"b{r}.npy"), b.data)  # broadcast reached rank 1


def _padded_worker(rank, world, port, result_dir):
    """Two stacked layers on shards whose columns index the padded all-gather
    buffer (dist.pad_columns + allgather_padded), oracle as the compute."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = G.gen_powerlaw(2500, 60000, 1200, 1.0, 31)
    G.randomize_values(a, 32)
    x0 = G.make_random_dense(2500, 12, 33).data
    info = D.ShardInfo(rank, world, D.partition_rows(a.row_ptr, world))
    local = D.pad_columns(D.shard_csr(a, info.lo, info.hi), info)
    pad = info.max_rows
    buf = torch.zeros((world * pad, 12))
    buf[torch.from_numpy(D.padded_row(info, np.arange(2500)))] = torch.from_numpy(x0)
    for _ in range(2):
        y, _ = O.spmm(local.n_rows, local.n_cols, local.row_ptr, local.col_ind, local.vals,
                      buf.numpy(), "sum")
        nxt = torch.zeros_like(buf)
        D.allgather_padded(torch.from_numpy(y), info, out=nxt)
        buf = nxt
    full = D.allgather_rows(torch.from_numpy(y), info)  # the compacting form
    np.save(os.path.join(result_dir, f"pad_rank{rank}.npy"),
            buf[torch.from_numpy(D.padded_row(info, np.arange(2500)))].numpy())
    np.save(os.path.join(result_dir, f"compact_rank{rank}.npy"), full.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_padded_allgather_two_layers_gloo(tmp_path, world):
    mp.spawn(_padded_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    a = G.gen_powerlaw(2500, 60000, 1200, 1.0, 31)
    G.randomize_values(a, 32)
    x = G.make_random_dense(2500, 12, 33).data
    for _ in range(2):
        x, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, x, "sum")
    for r in range(world):
        for name in ("pad", "compact"):
            got = np.load(tmp_path / f"{name}_rank{r}.npy")
            assert np.array_equal(got.view(np.uint32), x.view(np.uint32)), (name, r)


def test_pad_columns_keeps_rows_sorted():
    a = G.gen_powerlaw(4000, 100000, 2000, 1.0, 5)
    info = D.ShardInfo(0, 3, D.partition_rows(a.row_ptr, 3))
    p = D.pad_columns(a, info)
    assert p.n_cols == 3 * info.max_rows
    rp = p.row_ptr.astype(np.int64)
    d = np.diff(p.col_ind.astype(np.int64))
    inner = np.ones(p.nnz(), bool)
    inner[rp[:-1][rp[:-1] < rp[1:]]] = False  # row starts
    assert np.all(d[inner[1:]] > 0)
    assert np.array_equal(D.padded_row(info, a.col_ind), p.col_ind)


def _cuda_worker(rank, world, port, op, result_dir):
    """Two ranks sharing cuda:0 over gloo: the library's CUDA kernels as the
    per-shard compute, B broadcast and C all-gathered as CUDA tensors."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    a = G.gen_powerlaw(6000, 300000, 3000, 1.0, 21)
    G.randomize_values(a, 22)
    if rank == 0:
        b = torch.from_numpy(G.make_random_dense(6000, 128, 23).data.copy()).to(dev)
    else:
        b = torch.zeros(6000, 128, device=dev)

    def compute(shard, bt):
        c, arg = G.spmm(G.DeviceCsr.from_host(shard, dev), bt, op, want_arg=op == "max")
        torch.cuda.synchronize()
        return c

    full, info = D.distributed_spmm(a, b, rank, world, compute)
    np.save(os.path.join(result_dir, f"cuda_rank{rank}.npy"), full.cpu().numpy())
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("op", ["sum", "max"])
def test_two_rank_cuda_shards_equal_oracle(tmp_path, op):
    world = 2
    mp.spawn(_cuda_worker, args=(world, _free_port(), op, str(tmp_path)), nprocs=world,
             join=True)
    a = G.gen_powerlaw(6000, 300000, 3000, 1.0, 21)
    G.randomize_values(a, 22)
    b = G.make_random_dense(6000, 128, 23)
    want, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b.data, op)
    for r in range(world):
        got = np.load(tmp_path / f"cuda_rank{r}.npy")
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


from hypothesis import given, seed, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@seed(20261022)
@settings(max_examples=200, deadline=None)
@given(degs=st.lists(st.integers(0, 5000), min_size=0, max_size=400), parts=st.integers(1, 16))
def test_partition_rows_properties_random(degs, parts):
    """Every row in exactly one contiguous shard; each shard's nonzeros within
    one max-degree row of the ideal nnz/parts split."""
    rp = np.concatenate([[0], np.cumsum(np.asarray(degs, np.int64))]).astype(np.uint32)
    b = D.partition_rows(rp, parts)
    m = len(degs)
    assert len(b) == parts + 1 and b[0] == 0 and b[-1] == m
    assert all(b[i] <= b[i + 1] for i in range(parts))
    nnz = int(rp[-1])
    maxd = max(degs) if degs else 0
    loads = np.diff(rp.astype(np.int64)[b])
    assert loads.sum() == nnz
    assert np.all(loads <= nnz / parts + maxd + 1)

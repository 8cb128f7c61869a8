"""GPU: the fused all-gather epilogue (gespmm_plan_execute_gather) and the
device barrier (gespmm_peer_barrier).  On the one-GPU box the "peers" are
other buffers of the same device (one process) or IPC mappings between two
processes sharing cuda:0 — the same code path an NVSwitch box runs, with
NVLink replaced by the local memory system.  Every replica must equal the
oracle bit for bit."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2007_03179_b200 as G
from paper_2007_03179_b200 import _lib
from paper_2007_03179_b200 import dist as D

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _oracle_hops(a, x, hops, op="sum"):
    h = x
    for _ in range(hops):
        h, _ = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, h, op)
    return h


@pytest.mark.parametrize("op,n,opts", [
    ("sum", 128, {}),
    ("max", 128, {}),
    ("min", 64, {"hub_threshold": 400}),      # hub rows through the row-per-CTA kernel
    pytest.param("mean", 96, {"col_slices": 2},  # slice offsets applied to every replica
                 marks=[pytest.mark.experimental,
                        pytest.mark.skipif("not __import__('conftest').experimental_built()",
                                           reason="default build: col_slices not compiled")]),
    ("sum", 30, {}),                          # scalar lanes (N % 4 != 0)
])
def test_execute_gather_replicas_equal_oracle(op, n, opts):
    a = G.gen_powerlaw(4000, 160000, 1200, 1.0, 31)
    G.randomize_values(a, 32)
    b = G.make_random_dense(4000, n, 33).data
    want, warg = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b, op,
                        want_arg=op in ("max", "min"))
    # rows [lo, hi) of A computed, landing at rows lo.. of four full-height replicas
    lo, hi = 700, 3100
    shard = D.shard_csr(a, lo, hi)
    d = G.DeviceCsr.from_host(shard, DEV)
    bt = torch.from_numpy(b).to(DEV)
    plan = G.Plan(d, n, op, exec=G.ExecOptions(**opts))
    has_arg = op in ("max", "min")
    reps = [torch.full((a.n_rows, n), -7.0, device=DEV) for _ in range(4)]
    args = [torch.full((a.n_rows, n), -9, dtype=torch.int32, device=DEV) for _ in range(4)] \
        if has_arg else None
    c_d = [r.data_ptr() + 4 * lo * n for r in reps]
    a_d = [x.data_ptr() + 4 * lo * n for x in args] if has_arg else None
    before = G.launch_count()
    plan.execute_gather(bt, c_d, a_d)
    torch.cuda.synchronize()
    assert G.launch_count() > before
    for i, r in enumerate(reps):
        got = r.cpu().numpy()
        assert np.array_equal(got[lo:hi].view(np.uint32), want[lo:hi].view(np.uint32)), i
        assert (got[:lo] == -7.0).all() and (got[hi:] == -7.0).all(), "wrote outside the shard"
        if has_arg:
            ga = args[i].cpu().numpy()
            # the shard's arg positions are shard-local CSR positions
            off = int(a.row_ptr[lo])
            wa = warg[lo:hi].copy()
            wa[wa >= 0] -= off
            assert np.array_equal(ga[lo:hi], wa), i
    plan.close()


def test_execute_gather_rejects_bad_requests():
    a = G.gen_powerlaw(500, 5000, 100, 1.0, 3)
    d = G.DeviceCsr.from_host(a, DEV)
    bt = torch.zeros(500, 32, device=DEV)
    c = torch.empty(500, 32, device=DEV)
    plan = G.Plan(d, 32, "sum")
    with pytest.raises(G.Error, match="n_dsts"):
        plan.execute_gather(bt, [c.data_ptr()] * 9)
    with pytest.raises(G.Error, match="alignment"):
        plan.execute_gather(bt, [c.data_ptr(), c.data_ptr() + 4])
    plan.close()
    naive = G.Plan(d, 32, "sum", variant=G.KernelVariant.naive())
    with pytest.raises(G.Error, match="tuned plan"):
        naive.execute_gather(bt, [c.data_ptr()])
    naive.close()


def test_fused_propagate_single_rank_equals_oracle():
    a = G.gen_powerlaw(3000, 60000, 800, 1.0, 41)
    G.randomize_values(a, 42)
    x = G.make_random_dense(3000, 32, 43).data
    info = D.ShardInfo(0, 1, D.partition_rows(a.row_ptr, 1))
    got = D.fused_propagate(a, torch.from_numpy(x).to(DEV), 3, info, DEV)
    want = _oracle_hops(a, x, 3)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("exchange", ["fused", "nccl"])
def test_sgc_features_equal_oracle(exchange):
    """gcn.sgc_features: the K stacked aggregations of an SGC model through
    either exchange, on the GCN-normalised adjacency, bit-identical to the
    oracle's hops."""
    from paper_2007_03179_b200 import gcn
    a = gcn.normalize_adjacency(G.gen_powerlaw(2500, 40000, 600, 1.0, 7))
    x = G.make_random_dense(2500, 64, 8).data
    got = gcn.sgc_features(a, torch.from_numpy(x).to(DEV), 2, None, DEV, exchange=exchange)
    want = _oracle_hops(a, x, 2)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), want.view(np.uint32))


def test_peer_barrier_times_out_instead_of_hanging():
    L = _lib.lib()
    mine = torch.zeros(2, dtype=torch.int32, device=DEV)    # rank 0's signal words
    theirs = torch.zeros(2, dtype=torch.int32, device=DEV)  # "rank 1"'s, never signalling
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    stream = torch.cuda.current_stream().cuda_stream
    sigs = (C.c_void_p * 2)(mine.data_ptr(), theirs.data_ptr())
    assert L.gespmm_peer_barrier(sigs, 0, 2, 5, 200, err.data_ptr(), stream) == 0
    torch.cuda.synchronize()
    assert int(err.item()) == 1
    assert mine.cpu().tolist() == [5, 0] and theirs.cpu().tolist() == [5, 0]
    # a lone rank passes its own barrier
    err.zero_()
    one = (C.c_void_p * 1)(mine.data_ptr())
    assert L.gespmm_peer_barrier(one, 0, 1, 9, 200, err.data_ptr(), stream) == 0
    torch.cuda.synchronize()
    assert int(err.item()) == 0 and int(mine[0].item()) == 9
    with pytest.raises(Exception):
        D.PeerRows  # noqa: B018  (module attribute exists)
        if L.gespmm_peer_barrier(sigs, 2, 2, 1, 10, None, stream) != 0:
            raise RuntimeError(_lib.last_error())


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _prop_worker(rank, world, port, hops, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    a = G.gen_powerlaw(5000, 150000, 2000, 1.0, 51)
    G.randomize_values(a, 52)
    x = torch.from_numpy(G.make_random_dense(5000, 64, 53).data.copy()).to(dev)
    info = D.ShardInfo(rank, world, D.partition_rows(a.row_ptr, world))
    fused = D.fused_propagate(a, x, hops, info, dev)
    ref = D.nccl_propagate(a, x, hops, info, dev)
    np.save(os.path.join(result_dir, f"fused{rank}.npy"), fused.cpu().numpy())
    np.save(os.path.join(result_dir, f"ref{rank}.npy"), ref.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_fused_propagate_over_ipc(tmp_path):
    """Two ranks (processes) sharing cuda:0: buffers mapped with CUDA IPC, the
    epilogue storing into the other process's buffer, the device barrier
    between processes; equal to the oracle and to the NCCL-style path."""
    world, hops = 2, 3
    mp.spawn(_prop_worker, args=(world, _free_port(), hops, str(tmp_path)), nprocs=world,
             join=True)
    a = G.gen_powerlaw(5000, 150000, 2000, 1.0, 51)
    G.randomize_values(a, 52)
    want = _oracle_hops(a, G.make_random_dense(5000, 64, 53).data, hops)
    for r in range(world):
        got = np.load(tmp_path / f"fused{r}.npy")
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), r
        assert np.array_equal(np.load(tmp_path / f"ref{r}.npy").view(np.uint32),
                              want.view(np.uint32)), r


@pytest.mark.parametrize("op,n", [("sum", 128), ("max", 128), ("mean", 64), ("sum", 30)])
def test_multicast_epilogue_on_one_device(op, n):
    """NVLS multicast: the epilogue's multimem.st through a multicast object
    bound to this device's memory lands every output row (and arg) in the
    bound allocation, bit-identical to the oracle.  Skips where the device or
    driver has no multicast."""
    L = _lib.lib()
    a = G.gen_powerlaw(3000, 90000, 900, 1.0, 61)
    G.randomize_values(a, 62)
    b = G.make_random_dense(3000, n, 63).data
    has_arg = op in ("max", "min")
    want, warg = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b, op, want_arg=has_arg)
    bytes_c = 4 * a.n_rows * n
    total = 2 * bytes_c if has_arg else bytes_c
    uc, mc = C.c_void_p(), C.c_void_p()
    st = L.gespmm_multicast_alloc(total, C.byref(uc), C.byref(mc))
    if st == _lib.EUNSUPPORTED:
        pytest.skip(_lib.last_error())
    assert st == 0, _lib.last_error()
    try:
        full = torch.as_tensor(D._CudaArray(uc.value, (a.n_rows, n), "<f4"), device=DEV)
        full.fill_(-5.0)
        full_arg = (torch.as_tensor(D._CudaArray(uc.value + bytes_c, (a.n_rows, n), "<i4"),
                                    device=DEV) if has_arg else None)
        if has_arg:
            full_arg.fill_(-9)
        d = G.DeviceCsr.from_host(a, DEV)
        bt = torch.from_numpy(b).to(DEV)
        local = torch.empty((a.n_rows, n), device=DEV)
        local_arg = torch.empty((a.n_rows, n), dtype=torch.int32, device=DEV) if has_arg else None
        plan = G.Plan(d, n, op, exec=G.ExecOptions(hub_threshold=300))
        plan.execute_gather(bt, [local.data_ptr()],
                            [local_arg.data_ptr()] if has_arg else None,
                            c_multicast=mc.value,
                            arg_multicast=(mc.value + bytes_c) if has_arg else None)
        torch.cuda.synchronize()
        for got in (local, full):
            assert np.array_equal(got.cpu().numpy().view(np.uint32), want.view(np.uint32))
        if has_arg:
            assert np.array_equal(local_arg.cpu().numpy(), warg)
            assert np.array_equal(full_arg.cpu().numpy(), warg)
        plan.close()
        del full, full_arg
    finally:
        assert L.gespmm_multicast_free(uc) == 0

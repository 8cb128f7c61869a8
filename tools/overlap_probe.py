import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import bench, paper_2007_03179_b200 as G
from paper_2007_03179_b200 import dist as D
dev = torch.device("cuda", 0)
a = bench.make_inputs(bench.CONFIGS["reddit"])
b = torch.from_numpy(G.make_random_dense(a.n_cols, 128, 42).data).to(dev)
bounds = D.partition_rows(a.row_ptr, 8)
sh = D.shard_csr(a, bounds[0], bounds[1])
d = G.DeviceCsr.from_host(sh, dev)
c = torch.empty((sh.n_rows, 128), device=dev)
flush = torch.empty(128 * 1024 * 1024, device=dev)
import numpy as np
deg = np.diff(sh.row_ptr.astype(np.int64))
hub = np.sort(np.nonzero(deg >= 2946)[0]); rest = np.sort(np.nonzero(deg < 2946)[0])
def sub(rows):
    rp = sh.row_ptr.astype(np.int64)
    idx = np.concatenate([np.arange(rp[r], rp[r+1]) for r in rows])
    return G.CsrMatrix(len(rows), sh.n_cols, np.concatenate([[0], np.cumsum(deg[rows])]).astype(np.uint32), sh.col_ind[idx], sh.vals[idx])
def t(plan, cc):
    ts=[]
    for i in range(9):
        flush.zero_()
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); plan.execute(b, cc); e1.record(); torch.cuda.synchronize()
        if i>=2: ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)
full = G.Plan(d, 128, "sum")
print("full shard (auto):", t(full, c), full.description[-60:])
hs = sub(hub); dh = G.DeviceCsr.from_host(hs, dev); ch = torch.empty((hs.n_rows,128), device=dev)
rs = sub(rest); dr = G.DeviceCsr.from_host(rs, dev); cr = torch.empty((rs.n_rows,128), device=dev)
print("hub rows only via k_hub:", t(G.Plan(dh, 128, "sum", exec=G.ExecOptions(hub_threshold=1)), ch), hs.nnz())
print("hub rows only via k_warp:", t(G.Plan(dh, 128, "sum", exec=G.ExecOptions(hub_threshold=-1)), ch))
print("rest rows via k_warp:", t(G.Plan(dr, 128, "sum", exec=G.ExecOptions(hub_threshold=-1)), cr), rs.nnz())
print("full shard no hub:", t(G.Plan(d, 128, "sum", exec=G.ExecOptions(hub_threshold=-1)), c))

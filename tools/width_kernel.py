"""A few back-to-back launches of one SpMM width on the Reddit shape — the
target for an ncu capture of the narrow-width k_warp (GCN class width).

    python tools/width_kernel.py [N] [hub_threshold]
"""
import os
import sys

sys.path.insert(0, os.getcwd())

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2007_03179_b200 as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 44
ht = int(sys.argv[2]) if len(sys.argv) > 2 else -1
dev = torch.device("cuda", 0)
a = bench.make_inputs(bench.CONFIGS["reddit"])
d = G.DeviceCsr.from_host(a, dev)
b = torch.randn(a.n_cols, n, device=dev)
c = torch.empty(a.n_rows, n, device=dev)
p = G.Plan(d, n, "sum", exec=G.ExecOptions(hub_threshold=ht))
print(p.description, flush=True)
flush = torch.empty(128 * 1024 * 1024, device=dev)
for i in range(5):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    p.execute(b, c)
    e1.record()
    torch.cuda.synchronize()
    print(n, ht, round(e0.elapsed_time(e1), 3), flush=True)
p.close()

import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import bench, paper_2007_03179_b200 as G
from paper_2007_03179_b200 import gcn
dev = torch.device("cuda", 0)
a = gcn.normalize_adjacency(bench.make_inputs(bench.CONFIGS["reddit"]))
d = G.DeviceCsr.from_host(a, dev)
flush = torch.empty(128 * 1024 * 1024, device=dev)
cases = [(44, -1, 0), (44, 8000, 0), (44, 12000, 0), (44, 16000, 0), (44, 19000, 0), (256, 0, 0)]
if os.environ.get("PROBE_CASES"):
    cases = [tuple(int(v) for v in c.split(":")) for c in os.environ["PROBE_CASES"].split(",")]
for case in cases:
    n, ht, rpw = case[:3]
    slices = case[3] if len(case) > 3 else 0
    b = torch.randn(a.n_cols, n, device=dev)
    c = torch.empty(a.n_rows, n, device=dev)
    if True:
        p = G.Plan(d, n, "sum", exec=G.ExecOptions(hub_threshold=ht, rows_per_warp=rpw,
                                                   col_slices=slices))
        ts = []
        for i in range(8):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); p.execute(b, c); e1.record(); torch.cuda.synchronize()
            if i >= 2: ts.append(e0.elapsed_time(e1))
        print(n, ht, rpw, slices, round(statistics.median(ts), 3), p.description[-80:], flush=True)
        p.close()

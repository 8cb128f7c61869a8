#!/usr/bin/env python
"""Floor of a cold-L2 Pubmed-sized step: after the bench's L2 flush, time
(a) an empty launch, (b) a 10 MB device copy (B-sized read + C-sized write),
(c) the tuned SpMM plan (Pubmed N=128 sum), each with CUDA events, median."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    import paper_2007_03179_b200 as G
    dev = torch.device("cuda", 0)
    cfg = bench.CONFIGS["pubmed"]
    a = bench.make_inputs(cfg)
    n = 128
    b = torch.from_numpy(G.make_random_dense(a.n_cols, n, 42).data).to(dev)
    c = torch.empty((a.n_rows, n), device=dev)
    d = G.DeviceCsr.from_host(a, dev)
    flush = torch.empty(256 * 1024 * 1024 // 4 * 2, dtype=torch.float32, device=dev)
    small = torch.empty(1, device=dev)
    res = {}
    plans = {f"rpw{r}": G.Plan(d, n, "sum", exec=G.ExecOptions(rows_per_warp=r)) for r in (1, 2, 4, 8)}
    cases = {"empty": lambda: small.add_(1.0), "copy10MB": lambda: c.copy_(b)}
    for k, p in plans.items():
        cases[k] = (lambda p=p: p.execute(b, c))
    for cold in (True, False):
        for name, fn in cases.items():
            ts = []
            for i in range(25):
                if cold:
                    flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                if i >= 5:
                    ts.append(e0.elapsed_time(e1) * 1e3)
            res[(name, cold)] = statistics.median(ts)
            print(f"{'cold' if cold else 'warm'} {name:10s} median {res[(name, cold)]:7.2f} us  "
                  f"min {min(ts):7.2f} us", flush=True)
    for p in plans.values():
        print(p.description)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Probe: hub-row kernels on B200.  R rows of degree D (uniform random
columns over a Reddit-sized B, N=128 fp32, sum): the TMA-ring row-per-CTA
kernel (k_hub, hub_threshold=1) vs one warp per row (k_warp, threshold off).
R=1 measures a hub row's critical path, R=148*k the throughput per SM."""
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import argparse
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default=None, help="R,D: one case only")
    ap.add_argument("--only", default=None, choices=["warp", "hub"])
    ap.add_argument("--reps", type=int, default=9)
    args = ap.parse_args()
    import paper_2007_03179_b200 as G
    dev = torch.device("cuda", 0)
    K, n = 232_965, 128
    b = torch.from_numpy(G.make_random_dense(K, n, 42).data).to(dev)
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device=dev)
    rng = np.random.default_rng(0)
    cases = [(1, 21657), (1, 4000), (148, 21657), (296, 8000), (1000, 4000), (4000, 2000)]
    if args.case:
        cases = [tuple(int(x) for x in args.case.split(","))]
    for r, d in cases:
        cols = np.concatenate([np.sort(rng.choice(K, d, replace=False)) for _ in range(r)])
        a = G.CsrMatrix(r, K, (np.arange(r + 1, dtype=np.int64) * d).astype(np.uint32),
                        cols.astype(np.uint32), np.ones(r * d, np.float32))
        G.randomize_values(a, 3)
        dc = G.DeviceCsr.from_host(a, dev)
        c = torch.empty((r, n), device=dev)
        res = {}
        for name, ht in (("warp", -1), ("hub", 1)):
            if args.only and name != args.only:
                res[name] = float("nan")
                continue
            plan = G.Plan(dc, n, "sum", exec=G.ExecOptions(hub_threshold=ht))
            ts = []
            for i in range(args.reps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                plan.execute(b, c)
                e1.record()
                torch.cuda.synchronize()
                if i >= 2:
                    ts.append(e0.elapsed_time(e1))
            res[name] = statistics.median(ts)
            plan.close()
        gb = r * d * n * 4 / 1e9
        print(f"R={r:5d} D={d:6d}: warp {res['warp']:8.3f} ms ({gb / res['warp']:6.2f} TB/s)  "
              f"hub {res['hub']:8.3f} ms ({gb / res['hub']:6.2f} TB/s)", flush=True)


if __name__ == "__main__":
    main()

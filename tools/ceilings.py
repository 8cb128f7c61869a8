#!/usr/bin/env python
"""Measured ceilings for the roofline report (run on the B200 box).

Gather ceiling: gespmm_diag_gather reads one 512-byte B row (N=128 fp32) per
index into registers — the SpMM's L2->SM traffic without its arithmetic,
output or row structure.  Run on the Reddit-shape matrix's own col_ind (CSR
order) and on synthetic index streams that isolate L2 vs L1 behaviour.

    python tools/ceilings.py [--json out.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_2007_03179_b200 as G
    from paper_2007_03179_b200 import _lib

    p = argparse.ArgumentParser()
    p.add_argument("--json", default=None)
    p.add_argument("--reps", type=int, default=10)
    args = p.parse_args()
    dev = torch.device("cuda", 0)
    cfg = bench.CONFIGS["reddit"]
    a = bench.make_inputs(cfg)
    k, n = a.n_cols, 128
    b = torch.from_numpy(G.make_random_dense(k, n, 42).data).to(dev)
    count = a.nnz()
    rng = np.random.default_rng(0)
    streams = {
        "reddit_col_ind_csr_order": a.col_ind,
        "uniform_random_over_K": rng.integers(0, k, count, dtype=np.uint32),
        "reddit_col_ind_sorted": np.sort(a.col_ind),
        "uniform_random_over_2048_rows": rng.integers(0, 2048, count, dtype=np.uint32),
        "all_row_0": np.zeros(count, np.uint32),
    }
    L = _lib.lib()
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device=dev)
    out = {}
    for blocks in (148 * 3, 148 * 6):
        sink = torch.empty(blocks * 256, dtype=torch.float32, device=dev)
        for name, idx in streams.items():
            for hints in (1, 0):
                if blocks != 148 * 3 and (hints == 0 or name != "reddit_col_ind_csr_order"):
                    continue
                d_idx = torch.from_numpy(np.ascontiguousarray(idx).view(np.int32)).to(dev)
                st = torch.cuda.current_stream()
                times = []
                for r in range(args.reps + 2):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    rc = L.gespmm_diag_gather(d_idx.data_ptr(), count, b.data_ptr(), n,
                                              sink.data_ptr(), blocks, hints, st.cuda_stream)
                    assert rc == 0, _lib.last_error()
                    e1.record(st)
                    torch.cuda.synchronize()
                    if r >= 2:
                        times.append(e0.elapsed_time(e1))
                ms = float(np.median(times))
                gbs = count * n * 4 / (ms * 1e-3) / 1e9
                key = f"{name}|hints={hints}|blocks={blocks}"
                out[key] = {"ms": round(ms, 4), "gather_GBps": round(gbs, 1)}
                print(f"{key:60s} {ms:8.3f} ms  {gbs:9.1f} GB/s", flush=True)
                del d_idx
    info = G.device_info()
    out["device"] = info
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()

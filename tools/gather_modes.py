#!/usr/bin/env python
"""Gather ceiling by B-row load path (gespmm_diag_gather_mode), on the
Reddit-shape col_ind stream and on synthetic streams; N = 128.

    python tools/gather_modes.py [--json out.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MODES = {0: "LDG.128 L1-alloc", 1: "LDG.128 L1::no_allocate", 2: "cp.async.cg -> smem",
         3: "cp.async.bulk 512B -> smem"}


def main():
    import torch

    import bench
    import paper_2007_03179_b200 as G
    from paper_2007_03179_b200 import _lib

    p = argparse.ArgumentParser()
    p.add_argument("--json", default=None)
    p.add_argument("--reps", type=int, default=8)
    args = p.parse_args()
    dev = torch.device("cuda", 0)
    a = bench.make_inputs(bench.CONFIGS["reddit"])
    k, n = a.n_cols, 128
    b = torch.from_numpy(G.make_random_dense(k, n, 42).data).to(dev)
    count = a.nnz()
    rng = np.random.default_rng(0)
    streams = {"reddit_col_ind_csr_order": a.col_ind,
               "uniform_random_over_2048_rows": rng.integers(0, 2048, count, dtype=np.uint32)}
    L = _lib.lib()
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device=dev)
    out = {}
    for name, idx in streams.items():
        d_idx = torch.from_numpy(np.ascontiguousarray(idx).view(np.int32)).to(dev)
        for mode in MODES:
            for blocks in (148 * 2, 148 * 3, 148 * 4):
                sink = torch.empty(blocks * 256, dtype=torch.float32, device=dev)
                st = torch.cuda.current_stream()
                times = []
                for r in range(args.reps + 2):
                    flush.zero_()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    rc = L.gespmm_diag_gather_mode(d_idx.data_ptr(), count, b.data_ptr(),
                                                   sink.data_ptr(), blocks, mode, st.cuda_stream)
                    assert rc == 0, _lib.last_error()
                    e1.record(st)
                    torch.cuda.synchronize()
                    if r >= 2:
                        times.append(e0.elapsed_time(e1))
                ms = float(np.median(times))
                key = f"{name}|mode={mode} {MODES[mode]}|blocks={blocks}"
                out[key] = {"ms": round(ms, 4), "gather_GBps": round(count * n * 4 / ms / 1e6, 1),
                            "checksum": float(sink.double().sum().item())}
                print(f"{key:72s} {ms:8.3f} ms {out[key]['gather_GBps']:9.1f} GB/s "
                      f"sum={out[key]['checksum']:.6e}", flush=True)
        del d_idx
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()

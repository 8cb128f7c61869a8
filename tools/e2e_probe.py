#!/usr/bin/env python
"""Time the host-buffer entry point (gespmm_spmm_host) under option variants,
next to raw pinned H2D/D2H copy bandwidth, to attribute the e2e time."""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench
    import paper_2007_03179_b200 as G
    from paper_2007_03179_b200 import _lib

    a = bench.make_inputs(bench.CONFIGS["reddit"])
    n = 128
    b = G.make_random_dense(a.n_cols, n, 42).data
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()  # noqa: E731
    rp, ci, v, bh = pin(a.row_ptr.view(np.int32)), pin(a.col_ind.view(np.int32)), pin(a.vals), pin(b)
    ch = torch.empty((a.n_rows, n), dtype=torch.float32).pin_memory()
    dev = torch.device("cuda", 0)
    # raw copy bandwidth
    big = torch.empty(ci.numel(), dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    big.copy_(ci, non_blocking=True)
    torch.cuda.synchronize()
    t_h2d = time.perf_counter() - t0
    t0 = time.perf_counter()
    ci_back = torch.empty_like(ci).pin_memory()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ci_back.copy_(big, non_blocking=True)
    torch.cuda.synchronize()
    t_d2h = time.perf_counter() - t0
    print(f"pinned H2D {ci.numel() * 4 / t_h2d / 1e9:.1f} GB/s, D2H {ci.numel() * 4 / t_d2h / 1e9:.1f} GB/s")
    csr = _lib.Csr(a.n_rows, a.n_cols, a.nnz(), rp.data_ptr(), ci.data_ptr(), v.data_ptr())
    L = _lib.lib()
    for name, kw in [("tuned validate", {}), ("tuned novalidate", {"validate": 0}),
                     ("crc-cwm2 novalidate", {"validate": 0, "variant": 3, "cf": 2}),
                     ("tuned validate pageable", {"pageable": True})]:
        pageable = kw.pop("pageable", False)
        o = _lib.default_options(**kw)
        if pageable:
            cs = _lib.Csr(a.n_rows, a.n_cols, a.nnz(), a.row_ptr.ctypes.data, a.col_ind.ctypes.data,
                          a.vals.ctypes.data)
            bp, cp = b, np.empty((a.n_rows, n), np.float32)
            args = (ctypes.byref(cs), bp.ctypes.data, a.n_cols, n, 0, cp.ctypes.data, None,
                    ctypes.byref(o))
        else:
            args = (ctypes.byref(csr), bh.data_ptr(), a.n_cols, n, 0, ch.data_ptr(), None,
                    ctypes.byref(o))
        L.gespmm_spmm_host(*args)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            st = L.gespmm_spmm_host(*args)
            ts.append(time.perf_counter() - t0)
            assert st == 0, _lib.last_error()
        print(f"{name:28s} {1e3 * min(ts):8.2f} ms (min of 3) {[round(1e3 * t, 2) for t in ts]}")


if __name__ == "__main__":
    main()

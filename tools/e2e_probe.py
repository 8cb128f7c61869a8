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
    # raw copy bandwidth: the whole H2D payload of one step, best of 5
    big = torch.empty(ci.numel(), dtype=torch.int32, device=dev)
    ci_back = torch.empty_like(ci).pin_memory()

    def best(fn, reps=5):
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return min(ts)
    t_h2d = best(lambda: big.copy_(ci, non_blocking=True))
    t_d2h = best(lambda: ci_back.copy_(big, non_blocking=True))
    both = best(lambda: (big.copy_(ci, non_blocking=True), ci_back.copy_(big, non_blocking=True)))
    print(f"pinned H2D {ci.numel() * 4 / t_h2d / 1e9:.1f} GB/s, D2H {ci.numel() * 4 / t_d2h / 1e9:.1f} GB/s "
          f"(best of 5, {ci.numel() * 4 / 1e6:.0f} MB)")
    step_in = 4 * (a.n_rows + 1) + 8 * a.nnz() + 4 * a.n_cols * n
    print(f"H2D floor for one step ({step_in / 1e9:.3f} GB): {1e3 * step_in / (ci.numel() * 4 / t_h2d):.2f} ms")
    del both
    csr = _lib.Csr(a.n_rows, a.n_cols, a.nnz(), rp.data_ptr(), ci.data_ptr(), v.data_ptr())
    L = _lib.lib()
    runs = [("tuned validate", {}), ("tuned novalidate", {"validate": 0})]
    for nch in (4, 12, 16):
        runs.append((f"tuned validate chunks={nch}", {"chunks": nch}))
    for name, kw in runs + [
                     ("crc-cwm2 novalidate", {"validate": 0, "variant": 3, "cf": 2}),
                     ("tuned validate pageable", {"pageable": True})]:
        pageable = kw.pop("pageable", False)
        chunks = kw.pop("chunks", None)
        if chunks:
            os.environ["GESPMM_CHUNKS"] = str(chunks)
        else:
            os.environ.pop("GESPMM_CHUNKS", None)
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
        print(f"{name:28s} {1e3 * min(ts):8.2f} ms (min of 3) {[round(1e3 * t, 2) for t in ts]}",
              flush=True)
    os.environ["GESPMM_TRACE"] = "1"
    for nch in os.environ.get("PROBE_TRACE_CHUNKS", "8,16").split(","):
        os.environ["GESPMM_CHUNKS"] = nch
        o = _lib.default_options()
        for rep in range(2):  # the second call is the warm one
            print(f"traced call chunks={nch} rep {rep}:", flush=True)
            sys.stdout.flush()
            L.gespmm_spmm_host(ctypes.byref(csr), bh.data_ptr(), a.n_cols, n, 0, ch.data_ptr(),
                               None, ctypes.byref(o))
            sys.stderr.flush()


if __name__ == "__main__":
    main()

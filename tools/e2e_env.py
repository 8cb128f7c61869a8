#!/usr/bin/env python
"""Time gespmm_spmm_host on the Reddit shape under the current environment
(GESPMM_* / OMP_* knobs are read once per process): min / median of 7 calls,
optionally one traced call (E2E_TRACE=1)."""
import ctypes
import os
import statistics
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
    torch.zeros(1, device="cuda:0")
    csr = _lib.Csr(a.n_rows, a.n_cols, a.nnz(), rp.data_ptr(), ci.data_ptr(), v.data_ptr())
    L = _lib.lib()
    o = _lib.default_options()
    args = (ctypes.byref(csr), bh.data_ptr(), a.n_cols, n, 0, ch.data_ptr(), None, ctypes.byref(o))
    L.gespmm_spmm_host(*args)
    ts = []
    for _ in range(7):
        t0 = time.perf_counter()
        assert L.gespmm_spmm_host(*args) == 0, _lib.last_error()
        ts.append(1e3 * (time.perf_counter() - t0))
    env = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items())
                   if k.startswith(("GESPMM_", "OMP_", "GOMP_")))
    print(f"{env or 'default'}: min {min(ts):.2f} median {statistics.median(ts):.2f} ms "
          f"{[round(t, 2) for t in ts]}", flush=True)


if __name__ == "__main__":
    main()

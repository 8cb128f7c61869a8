#!/usr/bin/env python
"""Host-entry (packed upload) time vs host packing threads: OMP_NUM_THREADS
is read once per process, so run one process per setting; prints the median
of CALLS calls of gespmm_spmm_host on the Reddit shape (pinned buffers)."""
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
    csr = _lib.Csr(a.n_rows, a.n_cols, a.nnz(), rp.data_ptr(), ci.data_ptr(), v.data_ptr())
    o = _lib.default_options()
    L = _lib.lib()
    ts = []
    for i in range(int(os.environ.get("CALLS", "12"))):
        t0 = time.perf_counter()
        assert L.gespmm_spmm_host(ctypes.byref(csr), bh.data_ptr(), a.n_cols, n, 0, ch.data_ptr(),
                                  None, ctypes.byref(o)) == 0, _lib.last_error()
        ts.append(1e3 * (time.perf_counter() - t0))
    print(f"OMP_NUM_THREADS={os.environ.get('OMP_NUM_THREADS', '-')}: median {statistics.median(ts[2:]):.2f} ms "
          f"min {min(ts[2:]):.2f} ({' '.join(f'{t:.1f}' for t in ts)})", flush=True)


if __name__ == "__main__":
    main()

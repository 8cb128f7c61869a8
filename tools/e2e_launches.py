#!/usr/bin/env python
"""One host-entry call (Reddit shape, pinned buffers) for an ncu launch list:
which kernels the per-block compute of gespmm_spmm_host consists of."""
import ctypes
import os
import sys

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
    for _ in range(int(os.environ.get("CALLS", "2"))):
        assert L.gespmm_spmm_host(ctypes.byref(csr), bh.data_ptr(), a.n_cols, n, 0, ch.data_ptr(),
                                  None, ctypes.byref(o)) == 0, _lib.last_error()


if __name__ == "__main__":
    main()

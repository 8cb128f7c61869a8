#!/usr/bin/env python
"""Probe: does a static shared-memory hub cache beat L1/L2 gathers on B200?

Synthetic index streams over a Reddit-sized B (232,965 x 128 fp32): a fraction
f of the gathers hit rows [0, 400) (the "hub"), the rest are uniform over the
other rows.  Each stream runs through gespmm_diag_gather_hub with the hub in
shared memory (hub_rows=400) and without (hub_rows=0: hub rows come through
L1/L2), plus the plain gather kernel.  Prints ms and gathered TB/s.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2007_03179_b200 as G
    from paper_2007_03179_b200 import _lib
    dev = torch.device("cuda", 0)
    K, n, H = 232_965, 128, 400
    count = 60_000_000
    b = torch.from_numpy(G.make_random_dense(K, n, 42).data).to(dev)
    L = _lib.lib()
    sink = torch.empty(148 * 1024 * 4, dtype=torch.float32, device=dev)
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(0)
    st = torch.cuda.current_stream()

    def timeit(fn, reps=5):
        ts = []
        for r in range(reps + 2):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            assert fn() == 0, _lib.last_error()
            e1.record(st)
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(e0.elapsed_time(e1))
        return float(np.median(ts))

    for f in (0.0, 0.1, 0.25, 0.35, 0.5, 0.75, 1.0):
        u = torch.rand(count, device=dev, generator=gen)
        hub = torch.randint(0, H, (count,), device=dev, generator=gen, dtype=torch.int32)
        rest = torch.randint(H, K, (count,), device=dev, generator=gen, dtype=torch.int32)
        idx = torch.where(u < f, hub, rest).contiguous()
        del u, hub, rest
        gb = count * n * 4 / 1e9
        t_smem = timeit(lambda: L.gespmm_diag_gather_hub(idx.data_ptr(), count, b.data_ptr(), H,
                                                         sink.data_ptr(), 148, st.cuda_stream))
        t_l1 = timeit(lambda: L.gespmm_diag_gather_hub(idx.data_ptr(), count, b.data_ptr(), 0,
                                                       sink.data_ptr(), 148, st.cuda_stream))
        t_plain = timeit(lambda: L.gespmm_diag_gather(idx.data_ptr(), count, b.data_ptr(), n,
                                                      sink.data_ptr(), 444, 1, st.cuda_stream))
        print(f"hub frac {f:4.2f}: smem-hub {t_smem:7.3f} ms ({gb / t_smem:6.1f} TB/s)  "
              f"L1/L2 persistent {t_l1:7.3f} ms ({gb / t_l1:6.1f})  plain {t_plain:7.3f} ms "
              f"({gb / t_plain:6.1f})", flush=True)
        del idx


if __name__ == "__main__":
    main()

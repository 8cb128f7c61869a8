#!/usr/bin/env python
"""Time COO -> CSR on the benchmark graphs: the device builder
(gespmm_from_coo_device, triples already in HBM, CUDA events) against the
reference's from_coo (oracle/_ref, one host thread, triples in host memory),
on the shuffled edge list of the Reddit-shaped graph (and products with
--products).  Prints one JSON line per graph."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    import oracle as O
    import paper_2007_03179_b200 as G
    names = ["reddit"] + (["products"] if "--products" in sys.argv else [])
    for name in names:
        a = bench.make_inputs(bench.CONFIGS[name])
        d = G.DeviceCsr.from_host(a, "cuda:0")
        r, c, v = d.to_coo()
        perm = torch.randperm(r.numel(), device="cuda:0", generator=torch.Generator("cuda:0").manual_seed(0))
        r, c, v = r[perm].contiguous(), c[perm].contiguous(), v[perm].contiguous()
        del perm, d
        ts = []
        for _ in range(4):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = G.DeviceCsr.from_coo(a.n_rows, a.n_cols, r, c, v)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ok = (np.array_equal(out.col_ind.cpu().numpy().view(np.uint32), a.col_ind)
              and np.array_equal(out.vals.cpu().numpy(), a.vals))
        rh, ch, vh = (x.cpu().numpy() for x in (r, c, v))
        ref_s = None
        if O.ref_available():
            t0 = time.perf_counter()
            O.ref_from_coo(a.n_rows, a.n_cols, rh.view(np.uint32), ch.view(np.uint32), vh)
            ref_s = time.perf_counter() - t0
        print(json.dumps({"graph": name, "triples": int(a.nnz()), "device_ms": round(min(ts[1:]), 3),
                          "device_ms_first": round(ts[0], 3), "equal_to_generator_csr": bool(ok),
                          "reference_from_coo_s": round(ref_s, 3) if ref_s else None,
                          "speedup": round(ref_s * 1e3 / min(ts[1:]), 1) if ref_s else None}),
              flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""One small invocation of every kernel family of libgespmm.so, each result
checked against the oracle, sized so the whole run finishes in about a minute
under compute-sanitizer (which replays every memory access):

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck \
        python tools/sanitize_driver.py

SURVEY §5 "race detection": the reference relies on disjoint output ownership
and has no sanitizer runs; here the kernels with shared-memory staging
(k_warp's per-warp tiles, k_hub's mbarrier ring, k_cta, the unpack scan),
the fused replica epilogue, the overlap (programmatic dependent launch) chain,
the validation, transpose and COO builders all go through the tools.
Exits non-zero on a parity failure; the tool's own report is the verdict on
memory/race/sync errors."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import oracle as O
    import paper_2007_03179_b200 as G

    dev = "cuda:0"
    fails = []

    def same(tag, got, want):
        g = np.ascontiguousarray(got).view(np.uint32)
        w = np.ascontiguousarray(want).view(np.uint32)
        if not np.array_equal(g, w):
            fails.append(tag)
            print(f"MISMATCH {tag}", flush=True)

    a = G.gen_powerlaw(1500, 40000, 900, 1.0, 3)  # a few hub-sized rows
    G.randomize_values(a, 4)
    d = G.DeviceCsr.from_host(a, dev)
    for n, op, ex in [(128, "sum", {}), (64, "max", {}), (44, "mean", {}), (32, "min", {}),
                      (16, "sum", {}), (7, "max", {}), (256, "sum", {"tuned_cf": 2}),
                      (128, "sum", {"hub_threshold": 300}), (96, "max", {"hub_threshold": 300}),
                      (128, "sum", {"rows_per_warp": 4}), (128, "sum", {"exact": False})]:
        x = G.make_random_dense(a.n_cols, n, 5).data
        want, wa = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, x, op,
                          want_arg=op in ("max", "min"))
        c, arg = G.spmm(d, torch.from_numpy(x).to(dev), op, want_arg=op in ("max", "min"),
                        exec=G.ExecOptions(**ex))
        torch.cuda.synchronize()
        if ex.get("exact", True):
            same(f"tuned n={n} {op} {ex}", c.cpu().numpy(), want)
            if arg is not None:
                same(f"tuned arg n={n} {op} {ex}", arg.cpu().numpy(), wa)
        print(f"ok tuned n={n} {op} {ex}", flush=True)
    # hub rows through the LDG row-per-CTA kernel (N % 4 != 0 forces k_cta)
    x = G.make_random_dense(a.n_cols, 30, 6).data
    c, _ = G.spmm(d, torch.from_numpy(x).to(dev), "sum", exec=G.ExecOptions(hub_threshold=300))
    same("k_cta n=30", c.cpu().numpy(), O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals,
                                               x, "sum")[0])
    print("ok k_cta", flush=True)
    # the paper's Algorithms 1-3
    x = G.make_random_dense(a.n_cols, 64, 7).data
    want = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, x, "sum")[0]
    for v in (G.KernelVariant.naive(), G.KernelVariant.crc(), G.KernelVariant.crc_cwm(2),
              G.KernelVariant.crc_cwm(4)):
        c, _ = G.spmm(d, torch.from_numpy(x).to(dev), "sum", variant=v)
        same(f"faithful {v}", c.cpu().numpy(), want)
    print("ok faithful", flush=True)
    # host entry: pipelined blocks, packed upload, device validation
    b = G.DenseMatrix.of(G.make_random_dense(a.n_cols, 128, 8).data)
    want = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b.data, "sum")[0]
    got = G.native_spmm(a, b, G.KernelVariant.tuned(), G.ops.sum(), exec=G.ExecOptions(h2d_pack=1))
    same("host entry packed", got.data, want)
    print("ok host entry", flush=True)
    # fused all-gather epilogue into local replicas
    plan = G.Plan(d, 64, "sum")
    x = G.make_random_dense(a.n_cols, 64, 9).data
    bt = torch.from_numpy(x).to(dev)
    reps = [torch.empty((a.n_rows, 64), device=dev) for _ in range(3)]
    plan.execute_gather(bt, [r.data_ptr() for r in reps])
    want = O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, x, "sum")[0]
    for i, r in enumerate(reps):
        same(f"replica {i}", r.cpu().numpy(), want)
    plan.close()
    print("ok replicas", flush=True)
    # overlap_prev chain (programmatic dependent launches), ping-pong hops
    u = G.gen_uniform_random(G.GraphGenSpec(3000, 15000, 10))
    G.randomize_values(u, 11)
    du = G.DeviceCsr.from_host(u, dev)
    pl = G.Plan(du, 128, "sum", exec=G.ExecOptions(overlap_prev=True))
    x = G.make_random_dense(3000, 128, 12).data
    bufs = [torch.from_numpy(x).to(dev), torch.empty((3000, 128), device=dev)]
    for t in range(4):
        pl.execute(bufs[t % 2], bufs[(t + 1) % 2])
    h = x
    for _ in range(4):
        h = O.spmm(3000, 3000, u.row_ptr, u.col_ind, u.vals, h, "sum")[0]
    same("overlap chain", bufs[0].cpu().numpy(), h)
    pl.close()
    print("ok overlap chain", flush=True)
    # transpose, COO builders, validation
    t = d.transpose()
    th = t.to_host()
    rows = np.repeat(np.arange(a.n_rows, dtype=np.uint32), np.diff(a.row_ptr.astype(np.int64)))
    order = np.lexsort((rows, a.col_ind))
    same("transpose cols", th.col_ind, rows[order])
    rr, cc, vv = d.to_coo()
    perm = torch.randperm(rr.numel(), device=dev, generator=torch.Generator(dev).manual_seed(1))
    back = G.DeviceCsr.from_coo(a.n_rows, a.n_cols, rr[perm].contiguous(), cc[perm].contiguous(),
                                vv[perm].contiguous())
    same("from_coo cols", back.col_ind.cpu().numpy(), a.col_ind)
    same("from_coo vals", back.vals.cpu().numpy(), a.vals)
    bad = G.DeviceCsr(a.n_rows, a.n_cols, d.row_ptr, d.col_ind.clone(), d.vals)
    bad.col_ind[5] = a.n_cols + 3
    try:
        G.spmm(bad, torch.zeros((a.n_cols, 32), device=dev), "sum")
        fails.append("validation did not reject")
    except G.Error:
        pass
    print("ok transpose/coo/validate", flush=True)
    torch.cuda.synchronize()
    print(f"sanitize driver: {len(fails)} parity failures", flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()

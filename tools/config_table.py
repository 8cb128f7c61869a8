#!/usr/bin/env python
"""Every BASELINE.json config measured in one run on the
B200 box: GPU kernel time (cold L2 = flushed before each launch, and warm =
back-to-back launches), GFLOP/s, minimum-traffic roofline fraction, the
reference CPU path on the same inputs (oracle/_ref spmm::native_spmm for
sum/max, all host threads; the restatement for mean), and the bitwise parity
of the two results (FNV-1a checksum, dense.hpp:62-72, plus memcmp).

    python tools/config_table.py [--json out.json] [--md out.md] [--big]

Without --big only Cora and the Pubmed sweep run (seconds); --big adds the
Reddit N=128 sum and products N=256 max+arg lines.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SMALL = [("cora", dict(kind="uniform", rows=2708, nnz=10556), [16], ["sum", "max"]),
         ("pubmed", dict(kind="uniform", rows=19717, nnz=88648), [32, 64, 128],
          ["sum", "mean", "max"])]


def gen(spec):
    import bench
    import paper_2007_03179_b200 as G
    if spec["kind"] == "powerlaw":
        a = G.gen_powerlaw(spec["rows"], spec["nnz"], spec["maxdeg"], spec["exponent"],
                           bench.GEN_SEED)
    else:
        a = G.gen_uniform_random(G.GraphGenSpec(spec["rows"], spec["nnz"], bench.GEN_SEED))
    G.randomize_values(a, bench.VAL_SEED)
    return a


def time_gpu(plan, bt, c, arg, flush, cold_reps=20, warm_reps=200):
    import torch
    st = torch.cuda.current_stream()
    for _ in range(3):
        plan.execute(bt, c, arg)
    torch.cuda.synchronize()
    cold = []
    for _ in range(cold_reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        plan.execute(bt, c, arg)
        e1.record(st)
        torch.cuda.synchronize()
        cold.append(e0.elapsed_time(e1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = warm_reps if cold and statistics.median(cold) < 1.0 else 10
    e0.record(st)
    for _ in range(reps):
        plan.execute(bt, c, arg)
    e1.record(st)
    torch.cuda.synchronize()
    return statistics.median(cold), e0.elapsed_time(e1) / reps


def time_cpu(a, b, op):
    import oracle as O
    use_ref = O.ref_available() and op in ("sum", "max")
    threads = O.ref_hardware_concurrency() if O.ref_available() else (os.cpu_count() or 1)
    n = b.shape[1]
    variant, cf = ("crc", 1) if n <= 32 else ("crc-cwm", 2)
    want_arg = op in ("max", "min")

    def run():
        if use_ref:
            return O.ref_native_spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b, op,
                                     variant, cf, 0), None
        return O.spmm(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b, op,
                      want_arg=want_arg, threads=threads)

    t0 = time.perf_counter()
    out = run()
    first = time.perf_counter() - t0
    reps = 1 if first > 2.0 else (3 if first > 0.2 else 9)  # reference bench: median of repeats
    times = [first]
    for _ in range(reps - 1):
        t0 = time.perf_counter()
        out = run()
        times.append(time.perf_counter() - t0)
    c = out[0] if isinstance(out, tuple) else out
    kind = "reference spmm::native_spmm " + (variant if n <= 32 else f"{variant}{cf}") \
        if use_ref else "oracle restatement (no reference op)"
    return statistics.median(times), c, kind, threads


def main():
    import torch

    import bench
    import oracle as O
    import paper_2007_03179_b200 as G

    p = argparse.ArgumentParser()
    p.add_argument("--json", default=None)
    p.add_argument("--md", default=None)
    p.add_argument("--big", action="store_true")
    args = p.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device=dev)  # 512 MB
    peak, peak_src = bench.hbm_peak()
    jobs = list(SMALL)
    if args.big:
        r, pr = bench.CONFIGS["reddit"], bench.CONFIGS["products"]
        jobs.append(("reddit", r, [128], ["sum"]))
        jobs.append(("products", pr, [256], ["max+arg"]))
    rows = []
    for name, spec, ns, ops in jobs:
        a = gen(spec)
        d = G.DeviceCsr.from_host(a, dev)
        for n in ns:
            b = G.make_random_dense(a.n_cols, n, bench.B_SEED).data
            bt = torch.from_numpy(b).to(dev)
            for opname in ops:
                op = opname.split("+")[0]
                want_arg = opname.endswith("+arg")
                plan = G.Plan(d, n, op)
                c = torch.empty((a.n_rows, n), dtype=torch.float32, device=dev)
                arg = torch.empty((a.n_rows, n), dtype=torch.int32, device=dev) if want_arg else None
                cold, warm = time_gpu(plan, bt, c, arg, flush)
                got = c.cpu().numpy()
                cpu_s, want, kind, threads = time_cpu(a, b, op)
                exact = bool(np.array_equal(got.view(np.uint32), want.view(np.uint32)))
                alg, uniq = bench.algorithmic_bytes(a, n, want_arg)
                flops = 2 * a.nnz() * n
                row = {"config": name, "rows": a.n_rows, "nnz": a.nnz(), "n": n, "op": opname,
                       "gpu_ms_cold": round(cold, 5), "gpu_ms_warm": round(warm, 5),
                       "gflops_cold": round(flops / cold / 1e6, 1),
                       "gflops_warm": round(flops / warm / 1e6, 1),
                       "alg_bytes": alg, "hbm_frac_cold": round(alg / cold / 1e6 / peak, 4),
                       "cpu_s": round(cpu_s, 5), "cpu_gflops": round(flops / cpu_s / 1e9, 3),
                       "cpu_kind": kind, "cpu_threads": threads,
                       "speedup_cold": round(cpu_s * 1e3 / cold, 1),
                       "bit_exact": exact, "checksum_gpu": f"{O.checksum(got):016x}",
                       "checksum_cpu": f"{O.checksum(want):016x}", "plan": plan.description}
                rows.append(row)
                print(json.dumps(row), flush=True)
                plan.close()
                del c
        del d
    info = {"device": G.device_info(), "peak_gbs": peak, "peak_source": peak_src,
            "l2": "cold = 512 MB flush before each launch; warm = back-to-back launches",
            "rows": rows}
    if args.json:
        with open(args.json, "w") as f:
            json.dump(info, f, indent=1)
    if args.md:
        with open(args.md, "w") as f:
            f.write("| config | N | op | GPU cold ms | GPU warm ms | GFLOP/s cold | HBM frac cold | "
                    "CPU ref s | CPU kind (threads) | speed-up | bit-exact | checksum |\n")
            f.write("|---|---|---|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                f.write(f"| {r['config']} | {r['n']} | {r['op']} | {r['gpu_ms_cold']:.4f} | "
                        f"{r['gpu_ms_warm']:.4f} | {r['gflops_cold']:.0f} | {r['hbm_frac_cold']:.3f} | "
                        f"{r['cpu_s']:.4f} | {r['cpu_kind']} ({r['cpu_threads']}) | "
                        f"{r['speedup_cold']:.0f}x | {'yes' if r['bit_exact'] else 'NO'} | "
                        f"{r['checksum_gpu']} |\n")


if __name__ == "__main__":
    main()

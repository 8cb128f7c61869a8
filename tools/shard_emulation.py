#!/usr/bin/env python
"""Row-sharded multi-GPU step time, emulated on one B200.

The sharded path has no data-path collective: at G GPUs, rank
g runs the plan of its nnz-balanced row shard on its own GPU with B
replicated, and the step time is the max over ranks.  Each shard's kernel time
is therefore measurable alone on one GPU: this tool times every shard of
every G in --shards (L2 flushed before each launch, CUDA events, median of
--reps) and prints the emulated step time max_g t_g, the aggregate GFLOP/s and
the efficiency vs G x the 1-GPU value.  What it cannot see: the one-time B
broadcast (outside the step) and any cross-GPU interference (none: separate
HBM and L2 per GPU).

    python tools/shard_emulation.py [--config reddit] [--shards 1,2,4,8]
                                    [--hub-threshold T] [--json out.json]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench
    import paper_2007_03179_b200 as G
    from paper_2007_03179_b200 import dist as D

    p = argparse.ArgumentParser()
    p.add_argument("--config", default="reddit", choices=sorted(bench.CONFIGS))
    p.add_argument("--shards", default="1,2,4,8")
    p.add_argument("--hub-threshold", type=int, default=0)
    p.add_argument("--reps", type=int, default=7)
    p.add_argument("--json", default=None)
    p.add_argument("--only-shard", type=int, default=None, help="time only this shard index")
    p.add_argument("--fast", action="store_true", help="fast mode (FFMA sum, split hub rows)")
    args = p.parse_args()
    cfg = bench.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    a = bench.make_inputs(cfg)
    n, op, want_arg = cfg["n"], cfg["op"], bool(cfg.get("arg"))
    b = torch.from_numpy(G.make_random_dense(a.n_cols, n, bench.B_SEED).data).to(dev)
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device=dev)  # 512 MB
    ex = G.ExecOptions(hub_threshold=args.hub_threshold, exact=not args.fast)
    flops = 2 * a.nnz() * n
    out = {"config": args.config, "hub_threshold": args.hub_threshold, "runs": []}
    base = None
    for g in [int(x) for x in args.shards.split(",")]:
        bounds = D.partition_rows(a.row_ptr, g)
        times, descs, alg = [], [], 0
        for r in range(g):
            if args.only_shard is not None and r != args.only_shard:
                continue
            sh = D.shard_csr(a, bounds[r], bounds[r + 1]) if g > 1 else a
            alg += bench.algorithmic_bytes(sh, n, want_arg)[0]
            d = G.DeviceCsr.from_host(sh, dev)
            c = torch.empty((sh.n_rows, n), dtype=torch.float32, device=dev)
            arg = torch.empty((sh.n_rows, n), dtype=torch.int32, device=dev) if want_arg else None
            plan = G.Plan(d, n, op, exec=ex)
            ts = []
            for i in range(args.reps + 2):
                flush.zero_()
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record()
                plan.execute(b, c, arg)
                s1.record()
                torch.cuda.synchronize()
                if i >= 2:
                    ts.append(s0.elapsed_time(s1))
            times.append(statistics.median(ts))
            descs.append(plan.description)
            plan.close()
            del d, c, arg
        step = max(times)
        gf = flops / (step * 1e-3) / 1e9
        if g == 1:
            base = gf
        eff = gf / (g * base) if base else None
        peak, _ = bench.hbm_peak()
        hbm = alg / (step * 1e-3) / 1e9  # minimum-traffic bytes of all shards / step
        run = {"gpus": g, "shard_ms": [round(t, 4) for t in times], "step_ms": round(step, 4),
               "gflops": round(gf, 1), "efficiency_vs_1gpu": round(eff, 3) if eff else None,
               "hbm_gbs": round(hbm, 1), "roofline_frac": round(hbm / (g * peak), 4),
               "plan_shard0": descs[0]}
        out["runs"].append(run)
        print(json.dumps(run), flush=True)
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()

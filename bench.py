#!/usr/bin/env python
"""GE-SpMM on B200: the BASELINE.json headline metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config reddit|products|pubmed]

Default workload (BASELINE.json configs[2], the one the metric is quoted on):
Reddit-shaped power-law CSR (232,965 rows, 114.8M nnz, max degree 21,657,
seeded Chung-Lu generator), dense B of N=128 fp32, sum reduce.  A step is one
SpMM over the matrix with inputs resident in HBM; L2 is flushed between steps
(the inputs, 1.16 GB, are also larger than L2).  For N>1 (torchrun) every rank
takes an nnz-balanced row shard of the same matrix, B is broadcast once (NCCL),
and the step time is the max over ranks: total work is fixed -> "strong".

The JSON line adds ``roofline`` (minimum-traffic HBM model),
``cpu_baseline`` (the reference's own native_spmm from oracle/_ref on this
host, bounded row sample), ``e2e`` (the host-buffer C-ABI call with H2D/D2H in
the timed region), ``clocks`` and ``gpu_launches``.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CSR SpMM GFLOP/s + HBM GB/s vs roofline, Reddit-shape N=128, 1/2/4/8 B200"

CONFIGS = {
    "reddit": dict(kind="powerlaw", rows=232_965, nnz=114_800_000, maxdeg=21_657, exponent=1.0,
                   n=128, op="sum",
                   desc="Reddit-shaped power-law CSR (232965 rows, 114.8M nnz, max degree "
                        "21657) x dense fp32 N=128, sum"),
    "products": dict(kind="powerlaw", rows=2_449_029, nnz=123_718_280, maxdeg=17_481,
                     exponent=1.0, n=256, op="max", arg=True,
                     desc="ogbn-products-shaped power-law CSR (2449029 rows, 123.7M nnz) x "
                          "dense fp32 N=256, max + argmax"),
    "pubmed": dict(kind="uniform", rows=19_717, nnz=88_648, n=128, op="sum",
                   desc="Pubmed-shaped uniform CSR (19717 rows, 88648 nnz) x dense fp32 N=128, sum"),
    "cora": dict(kind="uniform", rows=2_708, nnz=10_556, n=16, op="sum",
                 desc="Cora-shaped uniform CSR (2708 rows, 10556 nnz) x dense fp32 N=16, sum"),
}
# BASELINE config 2 sweeps Pubmed over N in {32, 64, 128} x {sum, mean, max}:
# --n / --op override a config's width and reduce op (the workload text follows)
SMALL_BYTES = 64 << 20  # below this many algorithmic bytes a step is launch/latency-bound
GEN_SEED, VAL_SEED, B_SEED = 1, 2, 42
DATA_DESC = "synthetic (seeded power-law / uniform generator, reference value and B generators)"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# inputs
# ---------------------------------------------------------------------------

def make_inputs(cfg):
    """Our arm's inputs, from the product library's generators (bit-identical to
    the oracle restatements the reference arm uses, tests/test_oracle.py)."""
    import paper_2007_03179_b200 as G
    t0 = time.perf_counter()
    if cfg["kind"] == "powerlaw":
        a = G.gen_powerlaw(cfg["rows"], cfg["nnz"], cfg["maxdeg"], cfg["exponent"], GEN_SEED)
    else:
        a = G.gen_uniform_random(G.GraphGenSpec(cfg["rows"], cfg["nnz"], GEN_SEED))
    G.randomize_values(a, VAL_SEED)
    log(f"[bench] generated {a.n_rows} rows / {a.nnz()} nnz in {time.perf_counter() - t0:.1f}s")
    return a


class HostCsr:
    """Plain-array CSR for the reference arm (no product types)."""

    def __init__(self, n_rows, n_cols, row_ptr, col_ind, vals):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.row_ptr, self.col_ind, self.vals = row_ptr, col_ind, vals

    def nnz(self):
        return int(len(self.col_ind))


def make_inputs_reference(cfg):
    """The reference arm's inputs, built WITHOUT the product library: the
    reference's own gen_uniform_random (oracle/_ref) for the uniform shape, the
    oracle's C restatement of the power-law generator otherwise, then the
    value / B generators restated from the reference (oracle/powerlaw_oracle.c)."""
    import oracle as O
    t0 = time.perf_counter()
    if cfg["kind"] == "powerlaw":
        rp, ci, v = O.gen_powerlaw(cfg["rows"], cfg["nnz"], cfg["maxdeg"], cfg["exponent"],
                                   GEN_SEED)
    elif O.ref_available():
        rp, ci, v = O.ref_gen_uniform(cfg["rows"], cfg["nnz"], GEN_SEED)
    else:
        raise SystemExit("bench.py --impl reference: oracle/_ref not built (uniform generator)")
    v = np.ascontiguousarray(v, np.float32)
    O.randomize_values(v, VAL_SEED)
    a = HostCsr(cfg["rows"], cfg["rows"], rp, ci, v)
    b = O.make_random_dense(a.n_cols, cfg["n"], B_SEED)
    log(f"[bench] reference inputs {a.n_rows} rows / {a.nnz()} nnz in "
        f"{time.perf_counter() - t0:.1f}s (oracle generators, no product library)")
    return a, b


def config_of(cfg, world, exact=True):
    """The `config` object, identical in both arms for the same workload."""
    return {"workload": cfg["desc"], "rows": cfg["rows"], "nnz": cfg["nnz"], "n": cfg["n"],
            "op": cfg["op"], "arg": bool(cfg.get("arg")), "exact": bool(exact),
            "parallelism": f"row-shard x{world}",
            "l2": "flushed between steps (512 MB write)"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def algorithmic_bytes(a, n, arg):
    """4(M+1) + 8 nnz + 4 U N + 4 M N (+ 4 M N for arg), U = distinct columns."""
    u = int(np.count_nonzero(np.bincount(a.col_ind, minlength=a.n_cols))) if a.nnz() else 0
    m = a.n_rows
    return 4 * (m + 1) + 8 * a.nnz() + 4 * u * n + 4 * m * n * (2 if arg else 1), u


def sample_rows(a, frac, seed=0):
    """Strided row sample (keeps the degree mix) as a standalone plain-array CSR."""
    m = a.n_rows
    step = max(1, int(round(1.0 / max(frac, 1e-9))))
    if step == 1:
        return HostCsr(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals)
    rows = np.arange(seed % step, m, step, dtype=np.int64)
    rp = a.row_ptr.astype(np.int64)
    lens = rp[rows + 1] - rp[rows]
    idx = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows]) if len(rows) else \
        np.zeros(0, np.int64)
    return HostCsr(len(rows), a.n_cols, np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32),
                   np.ascontiguousarray(a.col_ind[idx]), np.ascontiguousarray(a.vals[idx]))


# ---------------------------------------------------------------------------
# clocks / peaks
# ---------------------------------------------------------------------------

class ClockSampler:
    """SM clock / power / throttle reasons sampled through NVML every ~10 ms on a
    thread; only samples taken inside the timed region (mark_start..mark_end)
    count.  Falls back to the nvidia-smi CLI when pynvml is missing."""
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4), ("hw_power_brake", 0x80))

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []  # (t, sm_mhz, mem_mhz, power_w, reasons_mask)
        self.t0 = self.t1 = None
        self._stop = threading.Event()
        self.thread = None
        self.error = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001 - report, do not fail the bench
            self.error = f"nvml unavailable: {e}"
            return

        def run():
            while not self._stop.is_set():
                try:
                    t = time.perf_counter()
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    mem = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)
                    pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((t, sm, mem, pw, rs))
                except Exception as e:  # noqa: BLE001
                    self.error = str(e)
                    return
                time.sleep(0.01)

        self.thread = threading.Thread(target=run, daemon=True)
        self.thread.start()

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_end(self):
        self.t1 = time.perf_counter()

    def stop(self):
        if self.thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.error or "not sampled"]}
        time.sleep(0.25)  # NVML readings lag: keep sampling briefly after the region
        self._stop.set()
        self.thread.join(timeout=2)
        t0 = self.t0 if self.t0 is not None else -1e30
        t1 = self.t1 if self.t1 is not None else 1e30
        inside = [x for x in self.samples if t0 <= x[0] <= t1]
        if not inside and self.samples:  # region shorter than one sample period
            inside = [min(self.samples, key=lambda x: abs(x[0] - t1))]
        if os.environ.get("GESPMM_CLOCK_LOG"):
            with open(os.environ["GESPMM_CLOCK_LOG"], "w") as f:
                for x in self.samples:
                    f.write(f"{x[0] - t0:.4f},{x[1]},{x[2]},{x[3]:.1f},{x[4]:#x},"
                            f"{int(t0 <= x[0] <= t1)}\n")
        reasons = sorted({name for x in inside for name, bit in self.REASONS if x[4] & bit})
        after = [x for x in self.samples if t1 < x[0] <= t1 + 0.25]
        reasons_after = sorted({name for x in after for name, bit in self.REASONS if x[4] & bit})
        sm = [x[1] for x in inside]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_min_mhz": min(sm) if sm else None,
                "sm_max_mhz": self.max_sm,
                "mem_mhz": statistics.median([x[2] for x in inside]) if inside else None,
                "power_w_max": max(x[3] for x in inside) if inside else None,
                "samples": len(inside), "source": "nvml, timed region only",
                "reasons": reasons,
                "reasons_next_250ms": reasons_after,
                "sm_mhz_next_250ms": statistics.median([x[1] for x in after]) if after else None}


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(config):
    """(dram bytes per step, source, bound counters) of the committed ncu
    capture of this config's kernel (profiles/ncu_<config>.json)."""
    p = os.path.join(ROOT, "profiles", f"ncu_{config}.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_step"), d.get("source"), d.get("bound_counters")
    except (OSError, ValueError):
        return None, None, None


# ---------------------------------------------------------------------------
# CPU baseline: the reference's own native_spmm (oracle/_ref) or the restatement
# ---------------------------------------------------------------------------

def _cpu_runner(sub, b, op, threads):
    """One CPU SpMM step over `sub`: the reference's spmm::bench window
    (oracle/_ref, RefSession, repeats=1) for the ops it has, else the oracle's
    C restatement of the same fold (mean / min / arg have no reference code)."""
    import oracle as O
    use_ref = O.ref_available() and op in ("sum", "max")
    variant, cf = ("crc", 1) if b.shape[1] <= 32 else ("crc-cwm", 2)
    if use_ref:
        sess = O.RefSession(sub.n_rows, sub.n_cols, sub.row_ptr, sub.col_ind, sub.vals, b)

        def run():
            return sess.bench(op, variant, cf, 0, 1)["median_s"]
        what = f"spmm::bench(native_spmm {variant}{'' if variant == 'crc' else f'({cf})'}, " \
               f"repeats=1) window, oracle/_ref"
    else:
        def run():
            t0 = time.perf_counter()
            O.spmm(sub.n_rows, sub.n_cols, sub.row_ptr, sub.col_ind, sub.vals, b, op,
                   want_arg=op in ("max", "min"), threads=threads)
            return time.perf_counter() - t0
        what = "oracle C restatement of the fold (no reference implementation of this op)"
    return run, ("reference" if use_ref else "port"), what


def cpu_sample_run(a, b, op, target_s=12.0):
    """The reported cpu_baseline: the reference on this host's cores, over the
    whole matrix when one pass fits `target_s`, else a strided row sample."""
    import oracle as O
    threads = O.ref_hardware_concurrency() if O.ref_available() else (os.cpu_count() or 1)
    frac = 1.0 / 512
    while True:
        sub = sample_rows(a, frac)
        run, kind, what = _cpu_runner(sub, b, op, threads)
        t = run()
        if t >= 0.5 or frac >= 1.0:
            break
        frac = min(1.0, frac * 4)
    if t < target_s and frac < 1.0:
        frac = min(1.0, frac * target_s / max(t, 1e-9))
        sub = sample_rows(a, frac)
        run, kind, what = _cpu_runner(sub, b, op, threads)
    reps = max(1, min(5, int(target_s / max(t, 1e-3))))
    ts = sorted(run() for _ in range(reps))
    t = ts[(len(ts) - 1) // 2]
    gflops = 2 * b.shape[1] * sub.nnz() / t / 1e9
    return {"value": round(gflops, 4), "unit": "GFLOP/s", "cores": threads, "kind": kind,
            "cpu_model": cpu_model(),
            "sample": f"every {int(round(1 / frac))}th row: {sub.n_rows} rows / {sub.nnz()} nnz "
                      f"({100.0 * sub.nnz() / max(a.nnz(), 1):.2f}% of nnz); {what}; median of "
                      f"{reps}", "seconds": round(t, 3)}


# ---------------------------------------------------------------------------
# arms
# ---------------------------------------------------------------------------

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def init_dist(world, local):
    """One process per GPU: pick the device, and for world > 1 join the NCCL
    group.  GESPMM_DIST_BACKEND=gloo (with ranks sharing a device, local %
    device_count) exercises the multi-rank path on a single-GPU box."""
    import torch
    dev = torch.device("cuda", local % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("GESPMM_DIST_BACKEND", "nccl")
        if backend == "nccl":
            if world > torch.cuda.device_count():
                raise SystemExit(f"bench.py: {world} NCCL ranks but {torch.cuda.device_count()} "
                                 "GPU(s); GESPMM_DIST_BACKEND=gloo shares one device")
            # communicator lines (nRanks, NVLS/NVLink transports) in each rank's stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    return dev


def run_reference(args, cfg):
    """The reference arm: the reference's own CPU native_spmm (oracle/_ref,
    unmodified headers) on this host's cores, inside its own spmm::bench
    timing window, on inputs built without the product library.  Rank 0
    only; other ranks exit without work."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle as O
    a, b = make_inputs_reference(cfg)
    op = cfg["op"]
    threads = O.ref_hardware_concurrency() if O.ref_available() else (os.cpu_count() or 1)
    # one step over the whole matrix when (warmup + steps) of them take ~2 min,
    # else a strided row sample sized to that budget
    per_step = max(0.2, 120.0 / max(1, args.steps + args.warmup))
    frac = 1.0
    sub = a
    run, kind, what = _cpu_runner(sub, b, op, threads)
    t = run()
    if t > per_step:
        frac = max(1.0 / 4096, per_step / t)
        sub = sample_rows(a, frac, seed=1)
        run, kind, what = _cpu_runner(sub, b, op, threads)
    for _ in range(args.warmup):
        run()
    times = [run() for _ in range(args.steps)]
    total = float(sum(times))
    flops = 2 * sub.nnz() * cfg["n"]
    value = flops * args.steps / total / 1e9
    sample = (f"{'whole matrix' if sub is a else f'every {int(round(1 / frac))}th row'}: "
              f"{sub.n_rows} rows / {sub.nnz()} nnz per step; {what}"
              + ("; max only (the reference has no argmax)" if cfg.get("arg") else ""))
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / args.steps, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": DATA_DESC,
        "config": config_of(cfg, world),
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": threads,
                         "kind": kind, "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "step_s": {"min": round(min(times), 4), "median": round(statistics.median(times), 4),
                   "max": round(max(times), 4)},
    }
    print(json.dumps(line), flush=True)
    return 0


def small_step_timings(plan, bt, c, arg, l2_flush, stream, reps=25, graph_len=64,
                       plan_overlap=None):
    """Launch/latency-bound configs (Pubmed, Cora): the step replayed from a
    captured CUDA graph, cold (after the L2 flush, as the timed steps) and warm
    (graph_len back-to-back SpMMs in one graph, per SpMM), next to two floors
    timed the same way: an empty kernel and a device copy of the step's dense
    bytes (B read, a B-sized write).  Event-timed on `stream`, medians in us."""
    import torch

    def timed(fn, cold, per=1):
        ts = []
        for i in range(reps + 5):
            if cold:
                l2_flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            if i >= 5:
                ts.append(e0.elapsed_time(e1) * 1e3 / per)
        return round(float(statistics.median(ts)), 2)

    cap = torch.cuda.Stream()
    cap.wait_stream(stream)
    with torch.cuda.stream(cap):
        plan.execute(bt, c, arg)  # first-call setup (policies) outside the capture
    torch.cuda.synchronize()
    g1, gr = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g1, stream=cap):
        plan.execute(bt, c, arg)
    with torch.cuda.graph(gr, stream=cap):
        for _ in range(graph_len):
            plan.execute(bt, c, arg)
    go = None
    if plan_overlap is not None:  # the same chain, each SpMM a programmatic dependent launch
        with torch.cuda.stream(cap):
            plan_overlap.execute(bt, c, arg)
        torch.cuda.synchronize()
        go = torch.cuda.CUDAGraph()
        with torch.cuda.graph(go, stream=cap):
            for _ in range(graph_len):
                plan_overlap.execute(bt, c, arg)
    torch.cuda.synchronize()
    one = torch.zeros(1, device=bt.device)
    dst = torch.empty_like(bt)
    with torch.cuda.stream(stream):
        out = {
            "cold_graph_us": timed(g1.replay, True),
            "cold_launch_us": timed(lambda: plan.execute(bt, c, arg), True),
            "warm_graph_us_per_spmm": timed(gr.replay, False, per=graph_len),
            "warm_graph_overlap_us_per_spmm": (timed(go.replay, False, per=graph_len)
                                               if go is not None else None),
            "floor_cold_empty_kernel_us": timed(lambda: one.add_(1.0), True),
            "floor_cold_copy_us": timed(lambda: dst.copy_(bt), True),
            "floor_copy_bytes": int(2 * bt.numel() * 4),
            "note": "cold = after the 512 MB L2 flush (the timed steps' condition); warm = "
                    f"{graph_len} SpMMs back to back in one CUDA graph, inputs L2-resident; "
                    "floors: an empty kernel and a device copy of B, timed the same way; "
                    "overlap = the plan with overlap_prev (each SpMM a programmatic dependent "
                    "launch of the previous one: its CTAs start and read A while it drains)",
        }
    return out


def run_ours(args, cfg):
    import torch
    import paper_2007_03179_b200 as G
    from paper_2007_03179_b200 import dist as D

    world, rank, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device")
    dev = init_dist(world, local)

    a = make_inputs(cfg)
    n, op, want_arg = cfg["n"], cfg["op"], bool(cfg.get("arg"))
    total_flops = 2 * a.nnz() * n
    bounds = D.partition_rows(a.row_ptr, world)
    info = D.ShardInfo(rank, world, bounds)
    shard = D.shard_csr(a, info.lo, info.hi) if world > 1 else a

    # B: generated on rank 0, replicated once over NCCL (timed apart from the step)
    if rank == 0:
        b_host = G.make_random_dense(a.n_cols, n, B_SEED).data
        bt = torch.from_numpy(b_host).to(dev)
    else:
        b_host = None
        bt = torch.empty((a.n_cols, n), dtype=torch.float32, device=dev)
    setup = None
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        D.broadcast_dense(bt, 0)
        e1.record()
        torch.cuda.synchronize()
        bms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        dist.all_reduce(bms, op=dist.ReduceOp.MAX)
        setup = {"b_broadcast_ms": round(float(bms.item()), 3),
                 "b_broadcast_bytes": int(bt.numel() * 4),
                 "backend": dist.get_backend(),
                 "note": "one-time replication of B (not in the step), max over ranks"}
    d = G.DeviceCsr.from_host(shard, dev)
    c = torch.empty((shard.n_rows, n), dtype=torch.float32, device=dev)
    arg = torch.empty((shard.n_rows, n), dtype=torch.int32, device=dev) if want_arg else None
    hints = 0 if args.no_hints else args.hints
    ex = G.ExecOptions(hub_threshold=args.hub_threshold, exact=not args.fast,
                       l2_persist=args.l2_persist, l2_hints=hints, l2_hot_mb=args.l2_hot_mb,
                       tuned_cf=args.tuned_cf, col_slices=args.col_slices,
                       rows_per_warp=args.rows_per_warp, cluster_hot=args.cluster_hot,
                       hot_rows_mb=args.hot_rows_mb)
    variant = G.variant_by_name(args.variant, args.cf)
    plan = G.Plan(d, n, op, variant=variant, exec=ex)
    log(f"[bench] rank {rank}: rows [{info.lo},{info.hi}) nnz {shard.nnz()} plan: {plan.description}")
    stream = torch.cuda.current_stream()
    flush_mb = int(os.environ.get("GESPMM_FLUSH_MB", "512"))  # A/B: flush size (> L2)
    l2_flush = torch.empty(flush_mb * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        plan.execute(bt, c, arg)

    nvtx = torch.cuda.nvtx
    nvtx.range_push("bench: warmup")
    for _ in range(max(args.warmup, 1)):
        l2_flush.zero_()
        step()
    torch.cuda.synchronize()
    nvtx.range_pop()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    sampler = ClockSampler(local) if rank == 0 else None
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    if sampler and not os.environ.get("GESPMM_NO_CLOCKS"):
        sampler.start()
        time.sleep(0.05)
    launches0 = G.launch_count()
    if sampler:
        sampler.mark_start()
    nvtx.range_push("bench: timed steps")
    for i in range(args.steps):
        if not args.no_flush:
            l2_flush.zero_()  # outside the events: L2 flushed between steps
        starts[i].record(stream)
        nvtx.range_push(f"step {i}")
        step()
        nvtx.range_pop()
        ends[i].record(stream)
    torch.cuda.synchronize()
    nvtx.range_pop()
    if sampler:
        sampler.mark_end()
    launches = G.launch_count() - launches0
    clocks = sampler.stop() if sampler else None
    per_step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    log("[bench] per-step ms: " + " ".join(f"{x:.3f}" for x in per_step_ms))
    total_ms = float(sum(per_step_ms))
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = total_flops * args.steps / (total_ms * 1e-3) / 1e9

    # roofline for this rank's SpMM step (plan.execute: warp kernel ∥ hub kernel)
    alg_bytes, uniq = algorithmic_bytes(shard, n, want_arg)
    my_ms = float(np.mean(per_step_ms))
    achieved = alg_bytes / (my_ms * 1e-3) / 1e9
    peak, peak_src = hbm_peak()
    traffic, traffic_src, bound_counters = ncu_traffic(args.config)

    # gather ceilings on this box, now (outside the timed region): the same
    # index stream through gespmm_diag_gather (one 512-B B row per nonzero into
    # registers, no arithmetic/output/row structure), and every gather hitting
    # one row (the L1/LSU data path alone).  N = 128 only (the diag kernel's).
    gather_ceiling = None
    if n == 128 and rank == 0 and not args.no_ceiling:
        from paper_2007_03179_b200 import _lib as _L
        Lg = _L.lib()
        blocks = 148 * 3
        sink = torch.empty(blocks * 256, dtype=torch.float32, device=dev)
        cnt = shard.nnz()
        res = {}
        for name, idx in (("csr_order", d.col_ind), ("one_row", torch.zeros_like(d.col_ind))):
            ts = []
            for r in range(5):
                l2_flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                rc = Lg.gespmm_diag_gather(idx.data_ptr(), cnt, bt.data_ptr(), n, sink.data_ptr(),
                                           blocks, 1, stream.cuda_stream)
                e1.record(stream)
                torch.cuda.synchronize()
                if rc != 0:
                    raise RuntimeError(_L.last_error())
                if r >= 2:
                    ts.append(e0.elapsed_time(e1))
            res[name] = round(float(statistics.median(ts)), 4)
        kernel_ms = float(statistics.median(per_step_ms))
        gather_ceiling = {
            "bound": "L2->SM / LSU data path: one 512-B B row per nonzero",
            "index_stream_ms": res["csr_order"], "one_row_ms": res["one_row"],
            "kernel_median_ms": round(kernel_ms, 4),
            "kernel_vs_index_stream": round(res["csr_order"] / kernel_ms, 3),
            "kernel_vs_one_row": round(res["one_row"] / kernel_ms, 3),
            "gathered_GBps": round(cnt * n * 4 / (kernel_ms * 1e-3) / 1e9, 1),
            "note": "gespmm_diag_gather on the matrix's own col_ind (L2 flushed) and on an "
                    "all-zero index stream (every gather an L1 hit); ratio > 1 = kernel faster"}

    small = None
    if alg_bytes < SMALL_BYTES and rank == 0:
        import dataclasses
        ov = (G.Plan(d, n, op, variant=variant, exec=dataclasses.replace(ex, overlap_prev=True))
              if variant.kind == G.KernelVariant.tuned().kind else None)
        small = small_step_timings(plan, bt, c, arg, l2_flush, stream, plan_overlap=ov)
        if ov is not None:
            ov.close()

    # end to end: the C-ABI host-buffer call, pinned host buffers, H2D + D2H inside
    e2e = None
    if not args.no_e2e:
        pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory()  # noqa: E731
        if b_host is None:
            b_host = bt.cpu().numpy()
        rp_h, ci_h = pin(shard.row_ptr.view(np.int32)), pin(shard.col_ind.view(np.int32))
        v_h, b_h = pin(shard.vals), pin(b_host)
        c_h = torch.empty((shard.n_rows, n), dtype=torch.float32).pin_memory()
        arg_h = torch.empty((shard.n_rows, n), dtype=torch.int32).pin_memory() if want_arg else None
        import ctypes
        from paper_2007_03179_b200 import _lib
        csr = _lib.Csr(shard.n_rows, shard.n_cols, shard.nnz(), rp_h.data_ptr(), ci_h.data_ptr(),
                       v_h.data_ptr())
        o = _lib.default_options(variant=int(variant.kind), cf=args.cf,
                                 hub_threshold=args.hub_threshold, exact=int(not args.fast),
                                 l2_persist=int(args.l2_persist), l2_hints=hints,
                                 l2_hot_mb=args.l2_hot_mb, tuned_cf=args.tuned_cf,
                                 col_slices=args.col_slices, rows_per_warp=args.rows_per_warp)
        L = _lib.lib()

        def host_call():
            st = L.gespmm_spmm_host(ctypes.byref(csr), b_h.data_ptr(), a.n_cols, n,
                                    _lib.REDUCE[op], c_h.data_ptr(),
                                    arg_h.data_ptr() if arg_h is not None else None,
                                    ctypes.byref(o))
            if st != 0:
                raise RuntimeError(_lib.last_error())

        host_call()
        e2e_steps = max(3, min(10, args.steps))
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        e2e_each = []
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            t1 = time.perf_counter()
            host_call()
            e2e_each.append(1e3 * (time.perf_counter() - t1))
        e2e_s = time.perf_counter() - t0
        log("[bench] e2e per-step ms: " + " ".join(f"{x:.2f}" for x in e2e_each))
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        h2d_user = 4 * (shard.n_rows + 1) + 8 * shard.nnz() + 4 * a.n_cols * n
        h2d = h2d_user
        if shard.nnz() >= (8 << 20):  # packed upload: 2-byte codes + 8-byte escapes
            rp64 = shard.row_ptr.astype(np.int64)
            ci64 = shard.col_ind.astype(np.int64)
            first = np.zeros(shard.nnz(), bool)
            first[rp64[:-1][rp64[:-1] < rp64[1:]]] = True
            gap = np.empty_like(ci64)
            gap[0] = ci64[0]
            gap[1:] = ci64[1:] - ci64[:-1] - 1
            gap[first] = ci64[first]
            n_esc = int(np.count_nonzero((gap < 0) | (gap >= 0xFFFF)))
            h2d = 4 * (shard.n_rows + 1) + 6 * shard.nnz() + 8 * n_esc + 4 * a.n_cols * n
        d2h = 4 * shard.n_rows * n * (2 if want_arg else 1)
        e2e = {"value": round(total_flops * e2e_steps / e2e_s / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "input_bytes_per_step": h2d_user,
               "ms_per_step": round(1e3 * e2e_s / e2e_steps, 3), "steps": e2e_steps,
               "step_ms": {"min": round(min(e2e_each), 3),
                           "median": round(statistics.median(e2e_each), 3),
                           "max": round(max(e2e_each), 3)},
               "path": "gespmm_spmm_host: row_ptr+B H2D, then 12 nnz-balanced row blocks pipelined "
                       "(host packs col_ind to 16-bit gap codes | codes+vals H2D | device unpack+"
                       "validate+kernel | C D2H); h2d_bytes = bytes that crossed PCIe, "
                       "input_bytes = the caller's CSR + B"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_sample_run(a, b_host if b_host is not None else bt.cpu().numpy(), op)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": DATA_DESC,
            "config": config_of(cfg, world, exact=not args.fast),
            "variant": args.variant, "plan": plan.description,
            "shards": {"kind": "nnz-balanced contiguous rows", "bounds": [int(x) for x in bounds]},
            "setup": setup,
            "hbm_gbs": round(achieved, 1),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": peak_src,
                         # what actually binds the kernel (ncu): the L2->SM return
                         # path and the L1 data pipe, not HBM
                         "bound_counters": bound_counters,
                         "kernel": "gespmm tuned SpMM step (warp-row kernel k_warp; hub "
                                   "rows, if any, through k_hub alongside)",
                         "algorithmic_bytes": alg_bytes, "unique_cols": uniq,
                         "model": "4(M+1)+8nnz+4UN+4MN[+4MN arg], per step"},
            "gather_ceiling": gather_ceiling,
            "small_step": small,
            "gpu_launches": int(launches),
            "step_ms": {"min": round(min(per_step_ms), 4),
                        "median": round(statistics.median(per_step_ms), 4),
                        "max": round(max(per_step_ms), 4)},
            "launches_per_step": plan.launches,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if args.dump_c:
        # per-rank shard of C (and arg) for the parity tests; rank 0 adds the bounds
        np.save(f"{args.dump_c}.rank{rank}.npy", c.cpu().numpy())
        if arg is not None:
            np.save(f"{args.dump_c}.arg.rank{rank}.npy", arg.cpu().numpy())
        if rank == 0:
            with open(f"{args.dump_c}.bounds.json", "w") as f:
                json.dump({"bounds": [int(x) for x in bounds], "world": world}, f)
    plan.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def run_gcn(args):
    """BASELINE config 5: two-layer GCN on the Reddit shape, hidden 256 — one
    full-batch training step (2 SpMM with A, 2 with A^T, 4 GEMMs, SGD) per step;
    under torchrun the nodes are row-sharded and each layer all-gathers."""
    import torch
    from paper_2007_03179_b200 import gcn
    import paper_2007_03179_b200 as G

    world, rank, local = dist_env()
    dev = init_dist(world, local)
    cfg = CONFIGS["reddit"]
    a = gcn.normalize_adjacency(make_inputs(cfg))  # D^-1/2 (A + I) D^-1/2
    gcfg = gcn.GCNConfig(in_features=602, hidden=256, classes=41)
    if args.gcn_pad > 0:
        gcfg.pad_to = args.gcn_pad
    adj, info = gcn.build_adjacency(a, dev, rank, world, G.ExecOptions(exact=not args.fast))
    h, y = gcn.synthetic_features(a.n_rows, gcfg.in_features, gcfg.classes)
    ht = torch.from_numpy(h[info.lo:info.hi]).to(dev)
    yt = torch.from_numpy(y[info.lo:info.hi]).to(dev)
    model = gcn.GCN(gcfg, dev)
    info_arg = info if world > 1 else None
    for _ in range(args.warmup):
        model.step(ht, yt, adj, info_arg, a.n_rows)
    torch.cuda.synchronize()
    gcn.EXCHANGE_EVENTS = [] if world > 1 else None
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = G.launch_count()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    e0.record(st)
    for _ in range(args.steps):
        loss = model.step(ht, yt, adj, info_arg, a.n_rows)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    flops = gcn.spmm_flops_per_step(a.nnz(), gcfg)
    exchange = None
    if gcn.EXCHANGE_EVENTS:
        ag = sum(s.elapsed_time(e) for s, e in gcn.EXCHANGE_EVENTS)
        t = torch.tensor([ag], dtype=torch.float64, device=dev)
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        exchange = {"allgather_ms_per_step": round(float(t.item()) / args.steps, 3),
                    "allgathers_per_step": len(gcn.EXCHANGE_EVENTS) // args.steps,
                    "note": "per-layer in-place ncclAllGather into the padded buffer (inside "
                            "the step), max over ranks"}
    gcn.EXCHANGE_EVENTS = None
    if rank == 0:
        print(json.dumps({
            "metric": "GCN 2-layer training step (Reddit shape, hidden 256): SpMM GFLOP/s "
                      "(4 SpMMs per step) over the whole step time",
            "value": round(flops * args.steps / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "two-layer GCN, Reddit-shaped power-law graph, features 602, "
                                   "hidden 256, classes 41, full batch, SGD",
                       "parallelism": f"row-shard x{world}, per-layer all-gather"},
            "exchange": exchange,
            "loss": round(float(loss.item()), 6),
            "gpu_launches": G.launch_count() - launches0}), flush=True)
    adj.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def run_propagate(args):
    """Stacked SpMM layers: H_{t+1} = A H_t for --hops hops on
    the Reddit shape (N=128, sum) over nnz-balanced row shards, with the
    per-hop exchange either fused into the SpMM epilogue (`--exchange fused`:
    every rank's kernel stores its rows into every rank's next-hop buffer
    through peer mappings, then one device barrier; dist.fused_propagate's
    loop) or unfused (`--exchange nccl`: local SpMM into the padded slot, then
    one in-place all_gather_into_tensor; dist.nccl_propagate's loop).  A step
    is one hop; value = 2*nnz*N*hops / time, max over ranks; the exchange
    share is timed on the same stream."""
    import torch
    import paper_2007_03179_b200 as G
    from paper_2007_03179_b200 import dist as D

    world, rank, local = dist_env()
    dev = init_dist(world, local)
    cfg = dict(CONFIGS[args.base])
    n = args.n or cfg["n"]
    a = make_inputs(cfg)
    m = a.n_rows
    info = D.ShardInfo(rank, world, D.partition_rows(np.asarray(a.row_ptr), world))
    x0 = torch.from_numpy(G.make_random_dense(m, n, B_SEED).data).to(dev)
    ex = G.ExecOptions(exact=not args.fast)
    st = torch.cuda.current_stream()
    stamps = []  # (hop start, spmm done, exchange done) events

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        return e

    if args.exchange == "fused":
        shard = D.shard_csr(a, info.lo, info.hi)
        plan = G.Plan(G.DeviceCsr.from_host(shard, dev), n, "sum", exec=ex)
        bufs = [D.PeerRows(m, n, info, dev), D.PeerRows(m, n, info, dev)]
        bufs[0].full.copy_(x0)
        dsts = [bf.dsts()[0] for bf in bufs]

        def hop(t, timed):
            src, dst = bufs[t % 2], bufs[(t + 1) % 2]
            e0 = ev() if timed else None
            if info.hi > info.lo:
                plan.execute_gather(src.full, dsts[(t + 1) % 2])
            e1 = ev() if timed else None
            dst.barrier()
            if timed:
                stamps.append((e0, e1, ev()))

        def result(t):
            return bufs[t % 2].full
    else:
        pad = info.max_rows
        shard = D.pad_columns(D.shard_csr(a, info.lo, info.hi), info) if world > 1 else a
        plan = G.Plan(G.DeviceCsr.from_host(shard, dev), n, "sum", exec=ex)
        idx = torch.from_numpy(D.padded_row(info, np.arange(m))).to(dev)
        bufs = [torch.zeros((world * pad, n), dtype=torch.float32, device=dev) for _ in range(2)]
        bufs[0].index_copy_(0, idx, x0)

        def hop(t, timed):
            src, dst = bufs[t % 2], bufs[(t + 1) % 2]
            slot = dst[info.rank * pad:(info.rank + 1) * pad]
            e0 = ev() if timed else None
            if info.rows:
                plan.execute(src, slot[:info.rows])
            e1 = ev() if timed else None
            if world > 1:
                D.allgather_padded(slot, info, out=dst)
            if timed:
                stamps.append((e0, e1, ev()))

        def result(t):
            return bufs[t % 2].index_select(0, idx)

    hops = args.hops
    for t in range(args.warmup * hops):
        hop(t, False)
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    launches0 = G.launch_count()
    base = args.warmup * hops
    for t in range(base, base + args.steps * hops):
        hop(t, True)
    torch.cuda.synchronize()
    total = sum(s.elapsed_time(e) for s, _, e in stamps)
    spmm = sum(s.elapsed_time(m1) for s, m1, _ in stamps)
    launches = G.launch_count() - launches0
    red = torch.tensor([total, spmm], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(red, op=dist.ReduceOp.MAX)
    total, spmm = float(red[0]), float(red[1])
    out = result(base + args.steps * hops)
    chk = int(G.checksum(G.DenseMatrix.of(out.cpu().numpy()))) if args.checksum else None
    nh = args.steps * hops
    if rank == 0:
        print(json.dumps({
            "metric": "stacked SpMM propagation H_{t+1} = A H_t (%s shape, N=%d, sum): "
                      "GFLOP/s per hop incl. the per-hop exchange" % (args.base, n),
            "value": round(2.0 * a.nnz() * n * nh / (total * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
            "n_gpus": world, "steps": nh, "warmup": args.warmup * hops,
            "ms_per_step": round(total / nh, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": DATA_DESC,
            "config": {"workload": cfg["desc"].replace(f"N={cfg['n']}", f"N={n}") + f", {hops} hops",
                       "parallelism": f"row-shard x{world}", "exchange": args.exchange,
                       "backend": os.environ.get("GESPMM_DIST_BACKEND", "nccl") if world > 1 else None},
            "exchange": {"kind": args.exchange,
                         "spmm_ms_per_hop": round(spmm / nh, 4),
                         "exchange_ms_per_hop": round((total - spmm) / nh, 4),
                         "note": "fused: SpMM with replica stores, then the device barrier; "
                                 "nccl: SpMM into the padded slot, then all_gather_into_tensor; "
                                 "max over ranks of each sum"},
            "checksum": chk, "gpu_launches": launches}), flush=True)
    if args.exchange == "fused":
        for bf in bufs:
            bf.check()
            bf.close()
    plan.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def relaunch(args):
    """`bench.py --gpus N` outside torchrun: start N ranks (one process per GPU)
    under torch.distributed.run on this node and return rank 0's exit code.
    Rank 0 prints the JSON line."""
    import socket
    import subprocess
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    log(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}")
    return subprocess.call(cmd)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", choices=sorted(CONFIGS) + ["gcn", "propagate"], default="reddit")
    p.add_argument("--hops", type=int, default=3, help="propagate: SpMM hops per step")
    p.add_argument("--base", choices=["reddit", "pubmed"], default="reddit",
                   help="propagate: the square graph to propagate over")
    p.add_argument("--exchange", choices=["fused", "nccl"], default="fused",
                   help="propagate: per-hop exchange fused into the SpMM epilogue, or NCCL all-gather")
    p.add_argument("--checksum", action="store_true", help="propagate: print the result checksum")
    p.add_argument("--variant", default="tuned", choices=["tuned", "naive", "crc", "crc-cwm"])
    p.add_argument("--cf", type=int, default=2)
    p.add_argument("--hub-threshold", type=int, default=0)
    p.add_argument("--fast", action="store_true", help="FFMA sum (1e-5 tolerance) instead of exact")
    p.add_argument("--l2-persist", type=int, nargs="?", const=1, default=0,
                   help="1: L2 access-policy window on B; 2: persisting set-aside only")
    p.add_argument("--no-hints", action="store_true", help="evict_normal instead of L2 hints")
    p.add_argument("--hints", type=int, default=1,
                   help="L2 hint mode (1: cold B rows evict_first, 2: evict_normal)")
    p.add_argument("--col-slices", type=int, default=0,
                   help="slice-major column traversal: 0 auto, 1 off, S slices")
    p.add_argument("--tuned-cf", type=int, default=0, help="tuned warp kernel merge factor")
    p.add_argument("--rows-per-warp", type=int, default=0,
                   help="rows sharing a warp (float4 lanes, N <= 256): 0 auto")
    p.add_argument("--l2-hot-mb", type=int, default=0,
                   help="hot-column map budget in MB (0 auto, <0 off)")
    p.add_argument("--no-flush", action="store_true", help="skip the L2 flush between steps")
    p.add_argument("--gcn-pad", type=int, default=0,
                   help="GCN: pad the class width to a multiple of this (default GCNConfig.pad_to)")
    p.add_argument("--hot-rows-mb", type=int, default=0,
                   help="relocated hot B rows budget (MB), experimental build; <=0 off")
    p.add_argument("--n", type=int, default=0, help="override the config's dense width N")
    p.add_argument("--op", default="", choices=["", "sum", "mean", "max", "min"],
                   help="override the config's reduce op (max/min carry the arg output)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-ceiling", action="store_true", help="skip the live gather-ceiling probe")
    p.add_argument("--dump-c", default="", help="save each rank's C shard to PATH.rank<r>.npy")
    p.add_argument("--cluster-hot", type=int, default=0,
                   help="N=128: hot B rows in cluster DSMEM, cluster size 2/4/8/16 (0 off)")
    args = p.parse_args()
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.warmup < 3:
        log("[bench] warmup raised to 3 (timing rules)")
        args.warmup = 3
    if args.config == "gcn":
        return run_gcn(args)
    if args.config == "propagate":
        return run_propagate(args)
    cfg = dict(CONFIGS[args.config])
    if args.n or args.op:
        n, op = args.n or cfg["n"], args.op or cfg["op"]
        cfg["desc"] = cfg["desc"].replace(f"N={cfg['n']}, {cfg['op']}", f"N={n}, {op}")
        if op in ("max", "min") and not cfg.get("arg"):
            cfg["desc"] += f" + arg{op}"
        cfg.update(n=n, op=op, arg=cfg.get("arg", False) or op in ("max", "min"))
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())

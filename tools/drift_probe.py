#!/usr/bin/env python
"""Why does the Reddit step time drift up within a bench run (2.83 -> 3.28 ms
after ~20 steps at a constant 1965 MHz SM clock)?  Per-step kernel times over
long runs with/without the L2 flush and with idle gaps between steps, plus
NVML temperature / power / clocks sampled along."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import pynvml

    import bench
    import paper_2007_03179_b200 as G
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    dev = torch.device("cuda", 0)
    a = bench.make_inputs(bench.CONFIGS["reddit"])
    b = torch.from_numpy(G.make_random_dense(a.n_cols, 128, 42).data).to(dev)
    d = G.DeviceCsr.from_host(a, dev)
    c = torch.empty((a.n_rows, 128), device=dev)
    plan = G.Plan(d, 128, "sum")
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device=dev)
    for name, do_flush, gap in (("flush", True, 0.0), ("noflush", False, 0.0),
                                ("flush+2ms idle", True, 0.002), ("flush", True, 0.0)):
        ts, info = [], []
        for i in range(300):
            if do_flush:
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.execute(b, c)
            e1.record()
            if gap:
                torch.cuda.synchronize()
                time.sleep(gap)
            if i % 50 == 49:
                torch.cuda.synchronize()
                info.append((pynvml.nvmlDeviceGetTemperature(h, 0),
                             pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                             pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                             pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                             hex(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))))
            ts.append((e0, e1))
        torch.cuda.synchronize()
        ms = [x.elapsed_time(y) for x, y in ts]
        blocks = [round(statistics.mean(ms[k:k + 25]), 3) for k in range(0, 300, 25)]
        print(f"{name:16s} per-25-step means: {blocks}", flush=True)
        print(f"{'':16s} (temp C, W, sm MHz, mem MHz, reasons) every 50: {info}", flush=True)
        time.sleep(2.0)


if __name__ == "__main__":
    main()

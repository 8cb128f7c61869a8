#!/usr/bin/env python
"""Raw pinned H2D bandwidth: one copy on one stream vs the same bytes split
over 2 or 4 streams (copy engines), and with a concurrent D2H."""
import time
import torch

def main():
    n = 459 * 1024 * 1024 // 4
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    hb = torch.empty(n // 4, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    db = torch.empty(n // 4, dtype=torch.float32, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(4)]
    def run(k, d2h=False):
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            parts = k
            step = n // parts
            for i in range(parts):
                with torch.cuda.stream(streams[i]):
                    d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
            if d2h:
                with torch.cuda.stream(streams[3]):
                    hb.copy_(db, non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return n * 4 / best / 1e9
    for k in (1, 2, 4):
        print(f"H2D {k} stream(s): {run(k):.1f} GB/s")
    print(f"H2D 1 stream + concurrent D2H (115 MB): {run(1, True):.1f} GB/s (H2D bytes only)")
    print(f"H2D 2 streams + concurrent D2H: {run(2, True):.1f} GB/s")

if __name__ == "__main__":
    main()

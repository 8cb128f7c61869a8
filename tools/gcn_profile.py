"""Per-kernel breakdown of the GCN training step (bench.py --config gcn setup):
torch.profiler over a few steps, device time per kernel name and per step.

    python tools/gcn_profile.py [--steps 3] [--fast]
"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.getcwd())

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2007_03179_b200 as G  # noqa: E402
from paper_2007_03179_b200 import gcn  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--fast", action="store_true")
    args = p.parse_args()
    dev = torch.device("cuda", 0)
    a = gcn.normalize_adjacency(bench.make_inputs(bench.CONFIGS["reddit"]))
    gcfg = gcn.GCNConfig(in_features=602, hidden=256, classes=41)
    adj, _ = gcn.build_adjacency(a, dev, 0, 1, G.ExecOptions(exact=not args.fast))
    h, y = gcn.synthetic_features(a.n_rows, gcfg.in_features, gcfg.classes)
    ht, yt = torch.from_numpy(h).to(dev), torch.from_numpy(y).to(dev)
    model = gcn.GCN(gcfg, dev)
    for _ in range(3):
        model.step(ht, yt, adj, None, a.n_rows)
    torch.cuda.synchronize()
    acts = [torch.profiler.ProfilerActivity.CUDA]
    with torch.profiler.profile(activities=acts) as prof:
        for _ in range(args.steps):
            model.step(ht, yt, adj, None, a.n_rows)
        torch.cuda.synchronize()
    tot = collections.Counter()
    cnt = collections.Counter()
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            tot[e.name] += e.device_time_total
            cnt[e.name] += 1
    all_us = sum(tot.values())
    print(f"device time per step {all_us / args.steps / 1e3:.3f} ms (kernels + copies, summed)")
    for name, us in tot.most_common(25):
        print(f"{us / args.steps / 1e3:8.3f} ms/step  x{cnt[name] // args.steps:<3d} {name[:110]}")
    adj.close()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Observability parity: the reference's SIMT simulator (32-byte segment
coalescer, /root/reference/proj/include/spmm/simt.hpp:60-104, metrics
:117-162) against B200's measured L1 sector counts for the paper's Algorithms
1-3 (kernels_faithful.cu), on the same inputs.  Reproduces the paper's Table IV
/ V style numbers (gld transactions, gld_efficiency, CRC and CWM reductions,
PAPER.md:439-509) on real hardware.

    # on the GPU box: one launch per (case, variant) under ncu
    ncu --metrics <METRICS> --csv --log-file gpurun_out/sectors.csv \\
        python tools/sector_parity.py run
    # here (needs oracle/_ref): simulator counts + comparison table
    python tools/sector_parity.py report gpurun_out/sectors.csv [--out profiles/...]

Mapping: simulator gld_transactions  <->  l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum
         simulator gst_transactions  <->  l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum
         simulator gld_efficiency    <->  smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,"
           "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,"
           "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,"
           "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct,"
           "gpu__time_duration.sum")

# (name, rows, nnz, n): the paper's Table IV random-graph shape (degree 10,
# N=512) at 16K rows, a ragged N, and the Pubmed shape at N=64.
CASES = [("paper16k_n512", 16384, 163840, 512),
         ("ragged_n48", 4096, 40960, 48),
         ("pubmed_n64", 19717, 88648, 64)]
VARIANTS = [("naive", 1), ("crc", 1), ("crc-cwm", 2), ("crc-cwm", 4), ("crc-cwm", 8)]
SMALL_CASES = [("small_n100", 700, 5000, 100), ("small_n512", 300, 4000, 512)]


def cases():
    return SMALL_CASES if os.environ.get("GESPMM_SECTOR_CASES") == "small" else CASES


def inputs(rows, nnz, n, seed=1):
    import paper_2007_03179_b200 as G
    a = G.gen_uniform_random(G.GraphGenSpec(rows, nnz, seed))
    G.randomize_values(a, seed + 1)
    b = G.make_random_dense(rows, n, 42)
    return a, b


def run():
    import torch
    import paper_2007_03179_b200 as G
    dev = torch.device("cuda", 0)
    for name, rows, nnz, n in cases():
        a, b = inputs(rows, nnz, n)
        d = G.DeviceCsr.from_host(a, dev)
        bt = torch.from_numpy(b.data).to(dev)
        for v, cf in VARIANTS:
            var = G.variant_by_name(v, cf)
            c, _ = G.spmm(d, bt, "sum", variant=var)
            torch.cuda.synchronize()
            print(f"{name} {v} cf={cf} launched", flush=True)


def _ncu_rows(path):
    """ncu --csv: one row per (launch, metric); returns launches in order."""
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    launches = {}
    for r in rows:
        key = int(r["ID"])
        launches.setdefault(key, {"kernel": r["Kernel Name"]})
        val = r["Metric Value"].replace(",", "")
        try:
            launches[key][r["Metric Name"]] = float(val)
        except ValueError:
            launches[key][r["Metric Name"]] = val
    return [launches[k] for k in sorted(launches)]


def report(ncu_csv, out_prefix):
    import oracle as O
    launches = [x for x in _ncu_rows(ncu_csv) if "k_naive" in x["kernel"] or "k_crc" in x["kernel"]]
    expected = len(cases()) * len(VARIANTS)
    if len(launches) != expected:
        raise SystemExit(f"expected {expected} faithful launches in {ncu_csv}, got {len(launches)}")
    table = []
    i = 0
    for name, rows, nnz, n in cases():
        a, b = inputs(rows, nnz, n)
        for v, cf in VARIANTS:
            sim = O.ref_sim_metrics(a.n_rows, a.n_cols, a.row_ptr, a.col_ind, a.vals, b.data,
                                    "sum", v, cf)
            hw = launches[i]
            i += 1
            ld = int(hw["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"])
            st = int(hw["l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum"])
            eff_hw = hw["smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct"] / 100.0
            eff_sim = sim["requested_load_bytes"] / max(sim["transferred_load_bytes"], 1)
            table.append({
                "case": name, "rows": rows, "nnz": int(a.nnz()), "n": n,
                "variant": v if v != "crc-cwm" else f"crc-cwm{cf}", "kernel": hw["kernel"],
                "sim_gld_transactions": sim["gld_transactions"], "b200_ld_sectors": ld,
                "ld_match": ld == sim["gld_transactions"],
                "sim_gst_transactions": sim["gst_transactions"], "b200_st_sectors": st,
                "st_match": st == sim["gst_transactions"],
                "sim_gld_efficiency": round(eff_sim, 4), "b200_gld_efficiency": round(eff_hw, 4),
                "sim_sparse_ld": sim["ld_col_ind"] + sim["ld_val"],
            })
    with open(out_prefix + ".json", "w") as f:
        json.dump(table, f, indent=1)
    hdr = ("| case | variant | sim gld trans. | B200 ld sectors | match | sim gst | B200 st "
           "sectors | match | sim gld_eff | B200 gld_eff |")
    lines = [hdr, "|" + "---|" * 10]
    for r in table:
        lines.append(f"| {r['case']} | {r['variant']} | {r['sim_gld_transactions']:,} | "
                     f"{r['b200_ld_sectors']:,} | {'yes' if r['ld_match'] else 'NO'} | "
                     f"{r['sim_gst_transactions']:,} | {r['b200_st_sectors']:,} | "
                     f"{'yes' if r['st_match'] else 'NO'} | {r['sim_gld_efficiency']:.2%} | "
                     f"{r['b200_gld_efficiency']:.2%} |")
    # Table IV / V style ratios
    lines.append("")
    for name, *_ in cases():
        rs = {r["variant"]: r for r in table if r["case"] == name}
        nv, cr = rs["naive"], rs["crc"]
        lines.append(f"{name}: naive/crc load sectors B200 {nv['b200_ld_sectors'] / cr['b200_ld_sectors']:.3f} "
                     f"(sim {nv['sim_gld_transactions'] / cr['sim_gld_transactions']:.3f}); "
                     "CWM sweep sectors " + " / ".join(
                         f"{rs[k]['b200_ld_sectors']:,}" for k in ("crc", "crc-cwm2", "crc-cwm4", "crc-cwm8")))
    text = "\n".join(lines) + "\n"
    with open(out_prefix + ".md", "w") as f:
        f.write(text)
    print(text)
    return table


def main():
    p = argparse.ArgumentParser()
    p.add_argument("mode", choices=["run", "report"])
    p.add_argument("csv", nargs="?")
    p.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_sector_parity"))
    args = p.parse_args()
    if args.mode == "run":
        run()
    else:
        report(args.csv, args.out)


if __name__ == "__main__":
    main()

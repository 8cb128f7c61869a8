"""The reference CLI's result records (JSON lines + CSV) for runs on the B200.

The reference's `spmm_cli bench` / `sweep` emit one JSON object per (matrix,
N, variant) run and a flat CSV with the same values
(/root/reference/proj/tools/spmm_cli.cpp:108-219, 566-611, 715-740).  Tools
that consume those files (plots, the acceptance scripts) keep working when the
runs come from this library: the records carry the same keys, with the
device timing under "b200" next to where the reference puts "native" (its
host-thread backend) or "sim" (its SIMT simulator's transaction counts).

* base record: tool, version, timestamp, input (generator spec or path), m, k,
  n, nnz, backend, variant, cf, op, warp_size, warps_per_block, b_seed
  (spmm_cli.cpp:139-165);
* per-backend object: workers, repeats, elapsed_s (median), elapsed_mean_s,
  flops (2 nnz N), gflops, checksum (16 hex digits of the FNV-1a checksum,
  dense.hpp:62-72) — the reference's "native" object (spmm_cli.cpp:595-601);
* verification: "none" or "bitwise" (checksum and memcmp equal to the CPU
  oracle), error: the spmm::Error text when the run failed.

The CSV header is the reference's, column for column (spmm_cli.cpp:168-172);
the device rows fill the native columns (workers = 1 device) and leave the
simulator's transaction columns empty, as the reference does for native rows.
"""
from __future__ import annotations

import dataclasses
import datetime
import json
from typing import Callable, Dict, List, Optional

TOOL_NAME = "spmm-lab"          # common.hpp:9 (records stay consumable by the same tools)
TOOL_VERSION = "0.1.0"          # common.hpp:10
BACKEND = "b200"

CSV_HEADER = (
    "matrix,backend,variant,cf,op,m,k,n,nnz,warp_size,warps_per_block,b_seed,"
    "gld_transactions,gst_transactions,requested_load_bytes,transferred_load_bytes,"
    "gld_efficiency,shared_loads,shared_stores,rowptr_load_tx,colind_load_tx,val_load_tx,"
    "b_load_tx,c_store_tx,workers,repeats,elapsed_s,gflops,checksum,verification,error")


@dataclasses.dataclass
class RunSettings:
    """spmm_cli.cpp:86-106 (RunSettings), for one device run."""
    input_descriptor: str = ""
    generator: Optional[Dict] = None      # {"rows", "nnz", "seed", "self_loops"}
    m: int = 0
    k: int = 0
    n: int = 0
    nnz: int = 0
    backend: str = BACKEND
    variant: str = "tuned"
    cf: int = 1
    op: str = "sum"
    warp_size: int = 32
    warps_per_block: int = 4
    b_seed: int = 42
    workers: int = 1
    repeats: int = 0
    verification: str = "none"
    error: str = ""


def iso_timestamp() -> str:
    return datetime.datetime.now(datetime.timezone.utc).strftime("%Y-%m-%dT%H:%M:%SZ")


def hex_checksum(v: int) -> str:
    return f"{int(v) & 0xffffffffffffffff:016x}"


def fmt_double(x: float) -> str:
    """std::ostream default formatting of a double (6 significant digits)."""
    return f"{x:.6g}"


def base_record(s: RunSettings) -> Dict:
    rec = {"tool": TOOL_NAME, "version": TOOL_VERSION, "timestamp": iso_timestamp()}
    if s.generator is not None:
        rec["input"] = {"generator": dict(s.generator)}
    else:
        rec["input"] = {"path": s.input_descriptor}
    rec.update(m=s.m, k=s.k, n=s.n, nnz=s.nnz, backend=s.backend, variant=s.variant, cf=s.cf,
               op=s.op, warp_size=s.warp_size, warps_per_block=s.warps_per_block,
               b_seed=s.b_seed)
    return rec


def backend_object(rep, workers: int) -> Dict:
    """The per-backend timing object (spmm_cli.cpp:595-601) from a ThroughputReport."""
    return {"workers": workers, "repeats": rep.repeats, "elapsed_s": rep.elapsed_s,
            "elapsed_mean_s": rep.elapsed_mean_s, "flops": rep.flops, "gflops": rep.gflops,
            "checksum": hex_checksum(rep.output_checksum)}


def csv_field(s: str) -> str:
    """RFC-4180 quoting for fields with commas, quotes or newlines (spmm_cli.cpp:183-193)."""
    if not any(c in s for c in ',"\n'):
        return s
    return '"' + s.replace('"', '""') + '"'


def csv_line(s: RunSettings, rep=None) -> str:
    head = [csv_field(s.input_descriptor), s.backend, s.variant, str(s.cf), s.op, str(s.m),
            str(s.k), str(s.n), str(s.nnz), str(s.warp_size), str(s.warps_per_block),
            str(s.b_seed)]
    sim = [""] * 12  # no simulator counts for device runs
    if rep is not None:
        nat = [str(s.workers), str(s.repeats), fmt_double(rep.elapsed_s), fmt_double(rep.gflops),
               hex_checksum(rep.output_checksum)]
    else:
        nat = [""] * 5
    return ",".join(head + sim + nat + [s.verification, csv_field(s.error)])


def variant_fields(v) -> tuple:
    """(name, cf_effective) as KernelVariant::name() / cf_effective() (kernel.hpp:44-68)."""
    return v.name(), v.cf_effective()


def bench_records(a, descriptor: str, n_list: List[int], variants, op: str = "sum",
                  repeats: int = 9, b_seed: int = 42, generator: Optional[Dict] = None,
                  reference: Optional[Callable] = None):
    """cmd_bench (spmm_cli.cpp:566-611) on the B200: for each N and variant, time
    the native_spmm-shaped host call with api.bench and yield (record, csv_row).
    reference(a, b, op) -> expected C (a CPU checker supplied by the caller,
    e.g. the test oracle): each output is then compared bitwise and the record
    says "bitwise" or "mismatch"."""
    import numpy as np
    from . import api
    op_obj = api.reduce_op_by_name(op)
    for n in n_list:
        b = api.make_random_dense(a.n_cols, n, b_seed)
        want = reference(a, b, op) if reference is not None else None
        baseline = None
        for v in variants:
            name, cf = variant_fields(v)
            s = RunSettings(input_descriptor=descriptor, generator=generator, m=a.n_rows,
                            k=a.n_cols, n=n, nnz=a.nnz(), variant=name, cf=cf, op=op,
                            b_seed=b_seed, repeats=repeats)
            rep = None
            try:
                rep = api.bench(a, b, v, op_obj, 0, repeats)
                if want is not None:
                    got = api.native_spmm(a, b, v, op_obj)
                    same = np.array_equal(np.ascontiguousarray(got.data).view(np.uint32),
                                          np.ascontiguousarray(want).view(np.uint32))
                    s.verification = "bitwise" if same else "mismatch"
            except api.Error as e:
                s.error = str(e)
            rec = base_record(s)
            if rep is not None:
                rec[BACKEND] = backend_object(rep, s.workers)
                if baseline is None:
                    baseline = rep.elapsed_s
                elif rep.elapsed_s > 0:
                    rec[BACKEND]["speedup_vs_first"] = baseline / rep.elapsed_s
            rec["verification"] = s.verification
            if s.error:
                rec["error"] = s.error
            yield rec, csv_line(s, rep)


def dumps(rec: Dict) -> str:
    """One JSON line (compact, like nlohmann::json::dump())."""
    return json.dumps(rec, separators=(",", ":"))

"""Generate the committed golden fixtures from the UNMODIFIED reference.

Run in the dev container (needs oracle/_ref/libspmmref.so, built from
/root/reference by oracle/Makefile):

    python tests/golden/make_golden.py

Writes tests/golden/golden.json (specs + reference checksums) and
tests/golden/small_cases.npz (full inputs/outputs for the hand cases and the
first corpus cases).  Every expected output below is produced by the
reference's own functions through the shim:

  native_spmm          proj/include/spmm/native.hpp:101-143
  gen_uniform_random   proj/include/spmm/generate.hpp:39-69
  randomize_values     proj/include/spmm/generate.hpp:73-80
  make_random_dense    proj/include/spmm/dense.hpp:51-59
  checksum             proj/include/spmm/dense.hpp:62-72
  validate             proj/include/spmm/csr.hpp:112-153
  from_coo             proj/include/spmm/csr.hpp:58-93

The case lists restate the reference's own tests:
  hand cases           proj/tests/test_kernels.cpp:26-116, test_native.cpp:12-25,
                       test_oracle.cpp:14-41
  random corpus        proj/tests/test_kernels.cpp:118-137 (seed 404 shape) and
                       proj/tests/acceptance.cpp:73-116 (seed 20260810 shape)
  validation errors    proj/tests/test_simt.cpp:249-258, test_csr.cpp
  configs              BASELINE.json configs[0..1] on the reference's uniform
                       generator (seed 1, values seed 2, B seed 42)
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402

MASK64 = (1 << 64) - 1


class MT64:
    """std::mt19937_64 (the reference's seeding RNG for its test drivers)."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & MASK64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & MASK64
        self.idx = 312

    def __call__(self):
        if self.idx >= 312:
            for i in range(312):
                x = (self.mt[i] & 0xFFFFFFFF80000000) | (self.mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                self.mt[i] = self.mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & MASK64


def fnv_arrays(*arrays):
    h = 1469598103934665603
    for a in arrays:
        for byte in np.ascontiguousarray(a).tobytes():
            h ^= byte
            h = (h * 1099511628211) & MASK64
    return h


def coo(rows, cols, entries):
    r = np.array([e[0] for e in entries], np.uint32)
    c = np.array([e[1] for e in entries], np.uint32)
    v = np.array([e[2] for e in entries], np.float32)
    return O.ref_from_coo(rows, cols, r, c, v)


def hand_cases():
    cases = []

    def add(name, m, k, csr, b, op, variant="crc", cf=2):
        rp, ci, v = csr
        b = np.asarray(b, np.float32)
        want = O.ref_native_spmm(m, k, rp, ci, v, b, op, variant, cf, 1)
        cases.append(dict(name=name, m=m, k=k, row_ptr=rp, col_ind=ci, vals=v, b=b, op=op,
                          want=want))

    eye = coo(3, 3, [(0, 0, 1.0), (1, 1, 1.0), (2, 2, 1.0)])
    add("identity_reproduces_b", 3, 3, eye, O.ref_make_random_dense(3, 4, 11), "sum")
    b = np.zeros((2, 2), np.float32)
    b[0, 0] = b[1, 1] = 1.0
    add("single_row_2_3", 1, 2, coo(1, 2, [(0, 0, 2.0), (0, 1, 3.0)]), b, "sum", "naive")
    add("two_rows_times_ones", 2, 3, coo(2, 3, [(0, 0, 1.0), (0, 2, 2.0), (1, 1, 3.0)]),
        np.ones((3, 2), np.float32), "sum")
    empty = (np.zeros(4, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.float32))
    add("empty_rows_sum_seed", 3, 3, empty, O.ref_make_random_dense(3, 5, 3), "sum")
    add("empty_rows_max_seed", 3, 3, empty, O.ref_make_random_dense(3, 5, 3), "max")
    bm = np.zeros((3, 1), np.float32)
    bm[1, 0], bm[2, 0] = 5.0, 3.0
    add("max_pool_neighbors", 3, 3, coo(3, 3, [(0, 1, 1.0), (0, 2, 1.0)]), bm, "max")
    add("upper_triangular_times_identity", 2, 2,
        coo(2, 2, [(0, 0, 1.0), (0, 1, 2.0), (1, 1, 3.0)]), b, "sum")
    add("short_row_partial_tile", 1, 8, coo(1, 8, [(0, c, 1.0) for c in range(5)]),
        O.ref_make_random_dense(8, 8, 5), "sum")
    add("long_row_three_tiles", 1, 100, coo(1, 100, [(0, c, 1.0) for c in range(70)]),
        O.ref_make_random_dense(100, 8, 5), "sum")
    b64 = np.arange(1, 65, dtype=np.float32).reshape(1, 64)
    add("cwm_lane_owns_strided_columns", 1, 1, coo(1, 1, [(0, 0, 2.0)]), b64, "sum",
        "crc-cwm", 2)
    add("cwm_ragged_boundary_n48", 1, 1, coo(1, 1, [(0, 0, 1.0)]),
        O.ref_make_random_dense(1, 48, 9), "sum", "crc-cwm", 2)
    return cases


def random_corpus():
    """Spec + reference checksum for two seeded corpora shaped like the reference's own."""
    out = []
    rng = MT64(404)  # test_kernels.cpp:118-137
    n_choices = [1, 5, 16, 33, 48, 64, 500]
    for it in range(25):
        rows = 1 + rng() % 200
        nnz = rng() % (rows * (rows - 1) // 2 + 1)
        gen_seed = rng()
        loops = (rng() & 1) != 0
        val_seed = rng()
        n = n_choices[rng() % len(n_choices)]
        b_seed = rng()
        op = "max" if it & 1 else "sum"
        out.append(dict(corpus="kernels404", rows=rows, nnz=nnz, gen_seed=gen_seed,
                        loops=loops, val_seed=val_seed, n=n, b_seed=b_seed, op=op))
    rng = MT64(20260810)  # acceptance.cpp:73-116
    n_choices = [1, 5, 16, 32, 33, 64, 500, 512]
    for case in range(200):
        rows = 1 + rng() % 1024
        loops = (rng() & 1) != 0
        degree = rng() % 17
        cap = rows * rows if loops else rows * (rows - 1)
        nnz = min(degree * rows, cap)
        gen_seed = rng()
        val_seed = rng()
        n = n_choices[rng() % 8]
        b_seed = rng()
        op = "max" if case & 1 else "sum"
        rng()  # cf choice draw (variant-only, result is variant-independent)
        out.append(dict(corpus="acceptance20260810", rows=rows, nnz=nnz, gen_seed=gen_seed,
                        loops=loops, val_seed=val_seed, n=n, b_seed=b_seed, op=op))
    for spec in out:
        rp, ci, v = O.ref_gen_uniform(spec["rows"], spec["nnz"], spec["gen_seed"], spec["loops"])
        v = O.ref_randomize_values(v, spec["val_seed"])
        b = O.ref_make_random_dense(spec["rows"], spec["n"], spec["b_seed"])
        c = O.ref_native_spmm(spec["rows"], spec["rows"], rp, ci, v, b, spec["op"], "crc-cwm",
                              2, 4)
        spec["csr_fnv"] = fnv_arrays(rp, ci, v)
        spec["b_checksum"] = O.ref_checksum(b)
        spec["checksum"] = O.ref_checksum(c)
    return out


def configs():
    out = []
    for name, rows, nnz, ns in (("cora", 2708, 10556, [16]),
                                ("pubmed", 19717, 88648, [32, 64, 128])):
        rp, ci, v = O.ref_gen_uniform(rows, nnz, 1, False)
        v = O.ref_randomize_values(v, 2)
        for n in ns:
            b = O.ref_make_random_dense(rows, n, 42)
            for op in ("sum", "max"):
                variant, cf = O.ref_select_variant(n)
                c = O.ref_native_spmm(rows, rows, rp, ci, v, b, op, variant, cf, 0)
                out.append(dict(config=name, rows=rows, nnz=nnz, gen_seed=1, val_seed=2,
                                b_seed=42, n=n, op=op, csr_fnv=fnv_arrays(rp, ci, v),
                                checksum=O.ref_checksum(c)))
    return out


def validation_cases():
    """Invalid inputs and the exact spmm::Error text the reference raises."""
    cases = []

    def add(name, m, k, rp, ci, v, b_rows=None, n=2):
        rp = np.asarray(rp, np.uint32)
        ci = np.asarray(ci, np.uint32)
        v = np.asarray(v, np.float32)
        b_rows = k if b_rows is None else b_rows
        b = np.zeros((b_rows, n), np.float32)
        msg = O.ref_native_spmm_error(m, k, rp, ci, v, b, b_rows, n)
        cnt, first = O.ref_validate(m, k, rp, ci, v)
        cases.append(dict(name=name, m=m, k=k, row_ptr=rp.tolist(), col_ind=ci.tolist(),
                          vals=v.tolist(), b_rows=b_rows, n=n, error=msg,
                          violations=cnt, first_violation=first))

    add("dimension_mismatch", 2, 3, [0, 1, 2], [0, 1], [1, 1], b_rows=4)
    add("row_ptr_not_starting_at_zero", 2, 3, [1, 1, 2], [0, 1], [1, 1])
    add("row_ptr_decreasing", 3, 3, [0, 2, 1, 2], [0, 1], [1, 1])
    add("row_ptr_end_not_nnz", 2, 3, [0, 1, 1], [0, 1], [1, 1])
    add("column_out_of_bounds", 2, 3, [0, 1, 2], [0, 3], [1, 1])
    add("columns_not_increasing", 1, 3, [0, 2], [2, 1], [1, 1])
    add("duplicate_column", 1, 3, [0, 2], [1, 1], [1, 1])
    add("oob_and_unsorted_same_row", 1, 4, [0, 3], [2, 9, 1], [1, 1, 1])
    add("col_vals_length_mismatch", 1, 3, [0, 1], [1], [1, 1])
    add("row_ptr_wrong_length", 3, 3, [0, 1], [0], [1])
    add("valid_ok", 2, 3, [0, 1, 2], [0, 1], [1, 1])
    add("zero_n", 2, 3, [0, 1, 2], [0, 1], [1, 1], n=0)
    return cases


def generator_pins():
    pins = []
    for rows, nnz, seed, loops in ((4, 8, 7, False), (100, 900, 12345, False), (4, 16, 0, True),
                                   (65536, 655360, 1, False), (2708, 10556, 1, False)):
        rp, ci, v = O.ref_gen_uniform(rows, nnz, seed, loops)
        pins.append(dict(kind="gen_uniform", rows=rows, nnz=nnz, seed=seed, loops=loops,
                         fnv=fnv_arrays(rp, ci, v)))
    for nnz, seed in ((1, 2), (1000, 2), (12345, 99)):
        v = O.ref_randomize_values(np.ones(nnz, np.float32), seed)
        pins.append(dict(kind="randomize_values", nnz=nnz, seed=seed, fnv=fnv_arrays(v)))
    for rows, cols, seed in ((3, 4, 11), (257, 65, 3), (1000, 128, 42)):
        d = O.ref_make_random_dense(rows, cols, seed)
        pins.append(dict(kind="make_random_dense", rows=rows, cols=cols, seed=seed,
                         checksum=O.ref_checksum(d)))
    return pins


def main():
    hc = hand_cases()
    corpus = random_corpus()
    npz = {}
    for i, c in enumerate(hc):
        for key in ("row_ptr", "col_ind", "vals", "b", "want"):
            npz[f"hand{i}_{key}"] = c[key]
    small = [s for s in corpus if s["rows"] <= 64 and s["n"] <= 64][:12]
    for i, s in enumerate(small):
        rp, ci, v = O.ref_gen_uniform(s["rows"], s["nnz"], s["gen_seed"], s["loops"])
        v = O.ref_randomize_values(v, s["val_seed"])
        b = O.ref_make_random_dense(s["rows"], s["n"], s["b_seed"])
        c = O.ref_native_spmm(s["rows"], s["rows"], rp, ci, v, b, s["op"], "crc", 2, 1)
        for key, arr in (("row_ptr", rp), ("col_ind", ci), ("vals", v), ("b", b), ("want", c)):
            npz[f"small{i}_{key}"] = arr
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **npz)
    doc = {
        "generated_by": "tests/golden/make_golden.py (reference via oracle/_ref/libspmmref.so)",
        "hand_cases": [dict(name=c["name"], m=c["m"], k=c["k"], n=int(c["b"].shape[1]),
                            op=c["op"], checksum=O.ref_checksum(c["want"]), npz_index=i)
                       for i, c in enumerate(hc)],
        "small_cases": [dict(s, npz_index=i) for i, s in enumerate(small)],
        "random_corpus": corpus,
        "configs": configs(),
        "validation": validation_cases(),
        "generator": generator_pins(),
    }
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(doc, f, indent=1)
    print(f"wrote {len(hc)} hand cases, {len(corpus)} corpus specs, "
          f"{len(doc['configs'])} config checksums, {len(doc['validation'])} validation cases")


if __name__ == "__main__":
    main()
